/*
 * oracle/na_oracle.c — plain, slow, obviously correct fp64 neighborhood
 * attention (forward and backward).  TEST INFRASTRUCTURE ONLY; see the
 * header for who may use it and for the definition it follows.
 *
 * Nothing here is blocked, fused or reordered beyond the definition:
 * the forward enumerates N(x) axis by axis, takes a max, a sum of exps, a
 * log and a weighted sum; the backward is the textbook softmax-attention
 * gradient written out per (x, y) pair.  Parallelism is only across
 * independent (b, h) slices or independent sampled tokens.
 */
#include "na_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ---------- exact upcasts of the input element types ---------- */

static double half_bits_to_double(uint16_t h) {
  /* IEEE 754 binary16: 1 sign, 5 exponent (bias 15), 10 fraction bits. */
  int sign = (h >> 15) & 1;
  int e = (h >> 10) & 0x1f;
  int f = h & 0x3ff;
  double v;
  if (e == 0) v = ldexp((double)f, -24);                 /* subnormal: f * 2^-24 */
  else if (e == 31) v = f ? NAN : INFINITY;
  else v = ldexp((double)(f + 1024), e - 25);            /* (1024+f) * 2^(e-15-10) */
  return sign ? -v : v;
}

static double bf16_bits_to_double(uint16_t b) {
  /* bfloat16 is the upper half of an IEEE binary32. */
  uint32_t u = (uint32_t)b << 16;
  float f;
  memcpy(&f, &u, 4);
  return (double)f;
}

static double load(int dtype, const void* base, int64_t i) {
  switch (dtype) {
    case NAR_F64: return ((const double*)base)[i];
    case NAR_F32: return (double)((const float*)base)[i];
    case NAR_F16: return half_bits_to_double(((const uint16_t*)base)[i]);
    case NAR_BF16: return bf16_bits_to_double(((const uint16_t*)base)[i]);
  }
  return NAN;
}

/* ---------- problem geometry ---------- */

int nar_check(const nar_problem* p) {
  if (p->rank < 1 || p->rank > 3) return 1;
  if (p->batch < 1 || p->heads < 1 || p->head_dim < 1) return 2;
  for (int a = 0; a < p->rank; ++a) {
    if (p->extent[a] < 1) return 2;
    if (p->kernel_size[a] < 1) return 3;
    if (!p->is_causal[a] && p->kernel_size[a] % 2 == 0) return 4;
    if (p->dilation[a] < 1) return 5;
    if ((int64_t)p->kernel_size[a] * p->dilation[a] > p->extent[a]) return 6;
  }
  return 0;
}

static double scale_of(const nar_problem* p) {
  return p->scale > 0 ? p->scale : 1.0 / sqrt((double)p->head_dim);
}

static int64_t tokens_per_slice(const nar_problem* p) {
  int64_t n = 1;
  for (int a = 0; a < p->rank; ++a) n *= p->extent[a];
  return n;
}

/* flat spatial index -> per-axis coordinates (row-major, axis 0 outermost) */
static void unflatten(const nar_problem* p, int64_t x, int c[3]) {
  for (int a = p->rank - 1; a >= 0; --a) {
    c[a] = (int)(x % p->extent[a]);
    x /= p->extent[a];
  }
}

static int64_t flatten(const nar_problem* p, const int c[3]) {
  int64_t x = 0;
  for (int a = 0; a < p->rank; ++a) x = x * p->extent[a] + c[a];
  return x;
}

int nar_axis_window(int L, int k, int dil, int causal, int x, int* first, int* last) {
  int r = x % dil;                       /* residue class of x      */
  int xc = x / dil;                      /* compacted coordinate in the class    */
  int Lr = (L - r + dil - 1) / dil;      /* size of the class: ceil((L-r)/dil)   */
  int lo, hi;
  if (causal) {                          /* no larger coordinates     */
    lo = xc - k + 1;
    if (lo < 0) lo = 0;
    hi = xc;
  } else {                               /* Fig. 2: window shifts inward at edges */
    lo = xc - k / 2;
    if (lo > Lr - k) lo = Lr - k;
    if (lo < 0) lo = 0;
    hi = lo + k - 1;
  }
  *first = r + dil * lo;
  *last = r + dil * hi;
  return hi - lo + 1;
}

int nar_contains(const nar_problem* p, int64_t x, int64_t y) {
  int cx[3], cy[3];
  unflatten(p, x, cx);
  unflatten(p, y, cy);
  for (int a = 0; a < p->rank; ++a) {
    int first, last;
    nar_axis_window(p->extent[a], p->kernel_size[a], p->dilation[a], p->is_causal[a], cx[a],
                    &first, &last);
    if (cy[a] < first || cy[a] > last) return 0;
    if ((cy[a] - first) % p->dilation[a] != 0) return 0;
  }
  return 1;
}

/* Enumerate N(x) (flat spatial key indices) in lexicographic axis order.
 * keys must hold prod(k) entries; returns the count. */
static int neighborhood(const nar_problem* p, int64_t x, int64_t* keys) {
  int cx[3], first[3], cnt[3] = {1, 1, 1};
  unflatten(p, x, cx);
  for (int a = 0; a < p->rank; ++a) {
    int last;
    cnt[a] = nar_axis_window(p->extent[a], p->kernel_size[a], p->dilation[a], p->is_causal[a],
                             cx[a], &first[a], &last);
  }
  int n = 0, c[3] = {0, 0, 0};
  for (int i0 = 0; i0 < cnt[0]; ++i0)
    for (int i1 = 0; i1 < (p->rank > 1 ? cnt[1] : 1); ++i1)
      for (int i2 = 0; i2 < (p->rank > 2 ? cnt[2] : 1); ++i2) {
        int ii[3] = {i0, i1, i2};
        for (int a = 0; a < p->rank; ++a) c[a] = first[a] + p->dilation[a] * ii[a];
        keys[n++] = flatten(p, c);
      }
  return n;
}

static int64_t max_window(const nar_problem* p) {
  int64_t l = 1;
  for (int a = 0; a < p->rank; ++a) l *= p->kernel_size[a];
  return l;
}

/* Forward for one query x of slice `bh`.  keys/prob are scratch of size
 * prod(k).  Writes O_x (D doubles) and returns LSE_x; also leaves the key list
 * in keys, P_xy in prob and the count in *nk. */
static double forward_row(const nar_problem* p, int dtype, const void* q, const void* k,
                          const void* v, int64_t bh, int64_t x, int64_t* keys, double* prob,
                          int* nk, double* o_row) {
  const int64_t N = tokens_per_slice(p);
  const int D = p->head_dim;
  const double scale = scale_of(p);
  const int64_t qoff = (bh * N + x) * D;
  int n = neighborhood(p, x, keys);
  double m = -INFINITY;
  for (int j = 0; j < n; ++j) {                              /* s_xy = scale <q_x, k_y> */
    const int64_t koff = (bh * N + keys[j]) * D;
    double s = 0.0;
    for (int d = 0; d < D; ++d) s += load(dtype, q, qoff + d) * load(dtype, k, koff + d);
    prob[j] = scale * s;
    if (prob[j] > m) m = prob[j];
  }
  double l = 0.0;
  for (int j = 0; j < n; ++j) l += exp(prob[j] - m);
  const double lse = m + log(l);
  for (int j = 0; j < n; ++j) prob[j] = exp(prob[j] - lse); /* P_xy */
  for (int d = 0; d < D; ++d) o_row[d] = 0.0;
  for (int j = 0; j < n; ++j) {
    const int64_t voff = (bh * N + keys[j]) * D;
    for (int d = 0; d < D; ++d) o_row[d] += prob[j] * load(dtype, v, voff + d);
  }
  *nk = n;
  return lse;
}

int nar_fwd(const nar_problem* p, int dtype, const void* q, const void* k, const void* v,
            double* o, double* lse) {
  int rc = nar_check(p);
  if (rc) return rc;
  const int64_t N = tokens_per_slice(p), BH = (int64_t)p->batch * p->heads;
  const int D = p->head_dim;
  const int64_t L = max_window(p);
#pragma omp parallel for schedule(dynamic)
  for (int64_t bh = 0; bh < BH; ++bh) {
    int64_t* keys = (int64_t*)malloc(sizeof(int64_t) * L);
    double* prob = (double*)malloc(sizeof(double) * L);
    for (int64_t x = 0; x < N; ++x) {
      int nk;
      lse[bh * N + x] = forward_row(p, dtype, q, k, v, bh, x, keys, prob, &nk, o + (bh * N + x) * D);
    }
    free(keys);
    free(prob);
  }
  return 0;
}

int nar_fwd_tokens(const nar_problem* p, int dtype, const void* q, const void* k, const void* v,
                   int64_t n, const int64_t* tokens, double* o, double* lse) {
  int rc = nar_check(p);
  if (rc) return rc;
  const int64_t N = tokens_per_slice(p);
  const int D = p->head_dim;
  const int64_t L = max_window(p);
#pragma omp parallel for schedule(dynamic)
  for (int64_t i = 0; i < n; ++i) {
    int64_t* keys = (int64_t*)malloc(sizeof(int64_t) * L);
    double* prob = (double*)malloc(sizeof(double) * L);
    int nk;
    lse[i] = forward_row(p, dtype, q, k, v, tokens[i] / N, tokens[i] % N, keys, prob, &nk, o + i * D);
    free(keys);
    free(prob);
  }
  return 0;
}

/* O as the method stores it (reading R12: D_x uses the stored output O, in
 * the inputs' 16-bit dtype): the fp64 value rounded to fp32 (the kernel's
 * accumulator) and then to o_dtype, round-to-nearest-even.  NAR_F64 = exact. */
static double stored(int o_dtype, double x) {
  if (o_dtype == NAR_F64) return x;
  float f = (float)x;
  if (o_dtype == NAR_F16) return (double)(_Float16)f;
  if (o_dtype == NAR_BF16) {
    uint32_t u;
    memcpy(&u, &f, 4);
    if ((u & 0x7f800000u) != 0x7f800000u) u += 0x7fffu + ((u >> 16) & 1u);
    u &= 0xffff0000u;
    memcpy(&f, &u, 4);
  }
  return (double)f;
}

int nar_bwd(const nar_problem* p, int dtype, int o_dtype, const void* q, const void* k,
            const void* v, const void* d_o, double* dq, double* dk, double* dv) {
  int rc = nar_check(p);
  if (rc) return rc;
  const int64_t N = tokens_per_slice(p), BH = (int64_t)p->batch * p->heads;
  const int D = p->head_dim;
  const int64_t L = max_window(p);
  const double scale = scale_of(p);
  memset(dq, 0, sizeof(double) * BH * N * D);
  memset(dk, 0, sizeof(double) * BH * N * D);
  memset(dv, 0, sizeof(double) * BH * N * D);
#pragma omp parallel for schedule(dynamic)
  for (int64_t bh = 0; bh < BH; ++bh) {       /* slices are independent: no atomics */
    int64_t* keys = (int64_t*)malloc(sizeof(int64_t) * L);
    double* prob = (double*)malloc(sizeof(double) * L);
    double* o_row = (double*)malloc(sizeof(double) * D);
    for (int64_t x = 0; x < N; ++x) {
      int nk;
      forward_row(p, dtype, q, k, v, bh, x, keys, prob, &nk, o_row);
      const int64_t xo = (bh * N + x) * D;
      double Dx = 0.0;                          /* D_x = <dO_x, O_x> */
      for (int d = 0; d < D; ++d) Dx += load(dtype, d_o, xo + d) * stored(o_dtype, o_row[d]);
      for (int j = 0; j < nk; ++j) {
        const int64_t yo = (bh * N + keys[j]) * D;
        double dP = 0.0;                        /* dP_xy = <dO_x, v_y> */
        for (int d = 0; d < D; ++d) dP += load(dtype, d_o, xo + d) * load(dtype, v, yo + d);
        const double dS = prob[j] * (dP - Dx);  /* dS_xy = P_xy (dP_xy - D_x) */
        for (int d = 0; d < D; ++d) {
          dq[xo + d] += scale * dS * load(dtype, k, yo + d);
          dk[yo + d] += scale * dS * load(dtype, q, xo + d);
          dv[yo + d] += prob[j] * load(dtype, d_o, xo + d);
        }
      }
    }
    free(keys);
    free(prob);
    free(o_row);
  }
  return 0;
}

int nar_bwd_tokens(const nar_problem* p, int dtype, int o_dtype, const void* q, const void* k,
                   const void* v, const void* d_o, int64_t n, const int64_t* tokens, double* dq,
                   double* dk, double* dv) {
  int rc = nar_check(p);
  if (rc) return rc;
  const int64_t N = tokens_per_slice(p);
  const int D = p->head_dim;
  const int64_t L = max_window(p);
  const double scale = scale_of(p);
#pragma omp parallel for schedule(dynamic)
  for (int64_t i = 0; i < n; ++i) {
    int64_t* keys = (int64_t*)malloc(sizeof(int64_t) * L);
    double* prob = (double*)malloc(sizeof(double) * L);
    double* o_row = (double*)malloc(sizeof(double) * D);
    const int64_t bh = tokens[i] / N, t = tokens[i] % N;
    double* dqi = dq + i * D;
    double* dki = dk + i * D;
    double* dvi = dv + i * D;
    for (int d = 0; d < D; ++d) dqi[d] = dki[d] = dvi[d] = 0.0;

    /* dQ_t: t as the query. */
    int nk;
    forward_row(p, dtype, q, k, v, bh, t, keys, prob, &nk, o_row);
    {
      const int64_t xo = (bh * N + t) * D;
      double Dx = 0.0;
      for (int d = 0; d < D; ++d) Dx += load(dtype, d_o, xo + d) * stored(o_dtype, o_row[d]);
      for (int j = 0; j < nk; ++j) {
        const int64_t yo = (bh * N + keys[j]) * D;
        double dP = 0.0;
        for (int d = 0; d < D; ++d) dP += load(dtype, d_o, xo + d) * load(dtype, v, yo + d);
        const double dS = prob[j] * (dP - Dx);
        for (int d = 0; d < D; ++d) dqi[d] += scale * dS * load(dtype, k, yo + d);
      }
    }

    /* dK_t, dV_t: t as the key.  Every query x with t in N(x) lies within
     * (k-1)*dil of t on each axis (x and t share a window of k members of
     * the same residue class), so scanning that box and testing membership
     * with the forward rule enumerates {x : t in N(x)} exactly. */
    int ct[3], lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
    unflatten(p, t, ct);
    for (int a = 0; a < p->rank; ++a) {
      const int reach = (p->kernel_size[a] - 1) * p->dilation[a];
      lo[a] = ct[a] - reach < 0 ? 0 : ct[a] - reach;
      hi[a] = ct[a] + reach > p->extent[a] - 1 ? p->extent[a] - 1 : ct[a] + reach;
    }
    int c[3] = {0, 0, 0};
    for (c[0] = lo[0]; c[0] <= hi[0]; ++c[0])
      for (c[1] = lo[1]; c[1] <= hi[1]; ++c[1])
        for (c[2] = lo[2]; c[2] <= hi[2]; ++c[2]) {
          const int64_t x = flatten(p, c);
          if (!nar_contains(p, x, t)) continue;
          forward_row(p, dtype, q, k, v, bh, x, keys, prob, &nk, o_row);
          int jt = -1;
          for (int j = 0; j < nk; ++j)
            if (keys[j] == t) jt = j;
          const int64_t xo = (bh * N + x) * D, to = (bh * N + t) * D;
          double Dx = 0.0, dP = 0.0;
          for (int d = 0; d < D; ++d) {
            Dx += load(dtype, d_o, xo + d) * stored(o_dtype, o_row[d]);
            dP += load(dtype, d_o, xo + d) * load(dtype, v, to + d);
          }
          const double dS = prob[jt] * (dP - Dx);
          for (int d = 0; d < D; ++d) {
            dki[d] += scale * dS * load(dtype, q, xo + d);
            dvi[d] += prob[jt] * load(dtype, d_o, xo + d);
          }
        }
    free(keys);
    free(prob);
    free(o_row);
  }
  return 0;
}

int nar_bwd_gather(const nar_problem* p, int dtype, int o_dtype, const void* q, const void* k,
                   const void* v, const void* d_o, double* dq, double* dk, double* dv) {
  int rc = nar_check(p);
  if (rc) return rc;
  const int64_t N = tokens_per_slice(p), BH = (int64_t)p->batch * p->heads;
  const int D = p->head_dim;
  const int64_t L = max_window(p);
  const double scale = scale_of(p);
  double* lse = (double*)malloc(sizeof(double) * N);
  double* Dvec = (double*)malloc(sizeof(double) * N);
  for (int64_t bh = 0; bh < BH; ++bh) {
    /* queries: LSE_x, D_x = <dO_x, O_x>, dQ_x = scale sum_y P_xy (dP_xy - D_x) k_y */
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t x = 0; x < N; ++x) {
      int64_t* keys = (int64_t*)malloc(sizeof(int64_t) * L);
      double* prob = (double*)malloc(sizeof(double) * L);
      double* o_row = (double*)malloc(sizeof(double) * D);
      int nk;
      lse[x] = forward_row(p, dtype, q, k, v, bh, x, keys, prob, &nk, o_row);
      const int64_t xo = (bh * N + x) * D;
      double Dx = 0.0;
      for (int d = 0; d < D; ++d) Dx += load(dtype, d_o, xo + d) * stored(o_dtype, o_row[d]);
      Dvec[x] = Dx;
      for (int d = 0; d < D; ++d) dq[xo + d] = 0.0;
      for (int j = 0; j < nk; ++j) {
        const int64_t yo = (bh * N + keys[j]) * D;
        double dP = 0.0;
        for (int d = 0; d < D; ++d) dP += load(dtype, d_o, xo + d) * load(dtype, v, yo + d);
        const double dS = prob[j] * (dP - Dx);
        for (int d = 0; d < D; ++d) dq[xo + d] += scale * dS * load(dtype, k, yo + d);
      }
      free(keys);
      free(prob);
      free(o_row);
    }
    /* keys: dK_t = scale sum_{x: t in N(x)} dS_xt q_x, dV_t = sum P_xt dO_x.
     * The queries with t in N(x) lie within (k-1)*dil of t on each axis
     * (see nar_bwd_tokens); membership is tested with the forward rule. */
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t t = 0; t < N; ++t) {
      const int64_t to = (bh * N + t) * D;
      for (int d = 0; d < D; ++d) dk[to + d] = dv[to + d] = 0.0;
      int ct[3], lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
      unflatten(p, t, ct);
      for (int a = 0; a < p->rank; ++a) {
        const int reach = (p->kernel_size[a] - 1) * p->dilation[a];
        lo[a] = ct[a] - reach < 0 ? 0 : ct[a] - reach;
        hi[a] = ct[a] + reach > p->extent[a] - 1 ? p->extent[a] - 1 : ct[a] + reach;
      }
      int c[3] = {0, 0, 0};
      for (c[0] = lo[0]; c[0] <= hi[0]; ++c[0])
        for (c[1] = lo[1]; c[1] <= hi[1]; ++c[1])
          for (c[2] = lo[2]; c[2] <= hi[2]; ++c[2]) {
            const int64_t x = flatten(p, c);
            if (!nar_contains(p, x, t)) continue;
            const int64_t xo = (bh * N + x) * D;
            double s = 0.0, dP = 0.0;
            for (int d = 0; d < D; ++d) {
              s += load(dtype, q, xo + d) * load(dtype, k, to + d);
              dP += load(dtype, d_o, xo + d) * load(dtype, v, to + d);
            }
            const double P = exp(scale * s - lse[x]);      /* P_xt */
            const double dS = P * (dP - Dvec[x]);            /* dS_xt */
            for (int d = 0; d < D; ++d) {
              dk[to + d] += scale * dS * load(dtype, q, xo + d);
              dv[to + d] += P * load(dtype, d_o, xo + d);
            }
          }
    }
  }
  free(lse);
  free(Dvec);
  return 0;
}

int nar_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
