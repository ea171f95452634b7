// fna_simt.cu — CUDA-core (fp32 FFMA) fused neighborhood attention kernels.
//
// The fp32 path of the library (TF32 off, so fp32 problems meet the 1e-4
// tolerance) and the path for any problem the tcgen05 kernels do not cover.
// One warp per output row: the 32 lanes split head_dim, the warp walks the
// row's neighborhood key by key with an online softmax (Milakov-Gimelshein,
// P:152-156) so attention weights never leave registers (fused, §3.3).
//
//   fna_fwd_simt    : O_x, LSE_x for every query x         (Eq. 1)
//   fna_bwd_pre     : D_x = <dO_x, O_x>                      (softmax Jacobian)
//   fna_dq_simt     : dQ_x = scale sum_y P(dP - D_x) k_y     (NN on dA)
//   fna_dkdv_simt   : dK_y, dV_y over the inverse window     (IN)
#include <cuda_bf16.h>
#include <type_traits>
#include <cuda_fp16.h>

#include "na_geom.cuh"
#include "na_kernels.h"
#include "tc_plan.h"

namespace na {
namespace {

template <typename T> __device__ __forceinline__ float ld(const T* p);
template <> __device__ __forceinline__ float ld<float>(const float* p) { return __ldg(p); }
template <> __device__ __forceinline__ float ld<__half>(const __half* p) { return __half2float(__ldg(p)); }
template <> __device__ __forceinline__ float ld<__nv_bfloat16>(const __nv_bfloat16* p) {
  return __bfloat162float(__ldg(p));
}
template <typename T> __device__ __forceinline__ T cvt(float x);
template <> __device__ __forceinline__ float cvt<float>(float x) { return x; }
template <> __device__ __forceinline__ __half cvt<__half>(float x) { return __float2half_rn(x); }
template <> __device__ __forceinline__ __nv_bfloat16 cvt<__nv_bfloat16>(float x) {
  return __float2bfloat16_rn(x);
}

__device__ __forceinline__ float ld_val(__half x) { return __half2float(x); }
__device__ __forceinline__ float ld_val(__nv_bfloat16 x) { return __bfloat162float(x); }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Per-axis compacted coordinate, residue and class size of flat token x.
struct Coord {
  int c[3], r[3], Lr[3];
};

__device__ __forceinline__ Coord decode(const Geom& g, int x) {
  Coord o;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    int v = a < g.rank ? (x / g.tstride[a]) % g.L[a] : 0;
    int dil = g.dil[a];
    o.r[a] = v % dil;
    o.c[a] = v / dil;
    o.Lr[a] = a < g.rank ? class_size(g.L[a], dil, o.r[a]) : 1;
  }
  return o;
}

__device__ __forceinline__ int token_of(const Geom& g, const Coord& co, const int cc[3]) {
  int t = 0;
#pragma unroll
  for (int a = 0; a < 3; ++a)
    if (a < g.rank) t += (co.r[a] + g.dil[a] * cc[a]) * g.tstride[a];
  return t;
}

// Element offset, inside its (b, h) slice, of the token at compacted
// coordinates cc of co's residue class (Geom::sX strides; contiguous:
// token_of * D).
__device__ __forceinline__ long long elem_of(const Geom& g, const Layout& ly, const Coord& co,
                                             const int cc[3]) {
  long long e = 0;
#pragma unroll
  for (int a = 0; a < 3; ++a)
    if (a < g.rank) e += (long long)(co.r[a] + g.dil[a] * cc[a]) * ly.sX[a];
  return e;
}

// ------------------------------------------------------------------ forward
template <typename T, int DPL>
__global__ void __launch_bounds__(256) fna_fwd_simt(Geom g, Layout ly, const T* __restrict__ q,
                                                    const T* __restrict__ k,
                                                    const T* __restrict__ v, T* __restrict__ o,
                                                    float* __restrict__ lse) {
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= (int64_t)g.BH * g.N) return;
  const int bh = (int)(row / g.N), x = (int)(row % g.N);
  const int64_t base = (int64_t)bh * ly.sBH;
  const Coord co = decode(g, x);
  const int64_t xe = base + elem_of(g, ly, co, co.c);  // this query's row
  float qr[DPL], acc[DPL];
#pragma unroll
  for (int i = 0; i < DPL; ++i) {
    int d = lane + 32 * i;
    qr[i] = d < g.D ? ld(q + xe + d) * g.scale_log2 : 0.f;
    acc[i] = 0.f;
  }
  int lo[3], hi[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    lo[a] = a < g.rank ? win_start(co.c[a], co.Lr[a], g.k[a], g.causal[a]) : 0;
    hi[a] = a < g.rank ? win_end(co.c[a], co.Lr[a], g.k[a], g.causal[a]) : 0;
  }
  float m = -INFINITY, l = 0.f;
  int cc[3];
  for (cc[0] = lo[0]; cc[0] <= hi[0]; ++cc[0])
    for (cc[1] = lo[1]; cc[1] <= hi[1]; ++cc[1])
      for (cc[2] = lo[2]; cc[2] <= hi[2]; ++cc[2]) {
        const int64_t y = base + elem_of(g, ly, co, cc);
        float s = 0.f;
#pragma unroll
        for (int i = 0; i < DPL; ++i) {
          int d = lane + 32 * i;
          if (d < g.D) s = fmaf(qr[i], ld(k + y + d), s);
        }
        s = warp_sum(s);                       // log2-domain logit
        const float mn = fmaxf(m, s);
        const float corr = exp2f(m - mn);      // 0 when m = -inf
        const float p = exp2f(s - mn);
        l = l * corr + p;
#pragma unroll
        for (int i = 0; i < DPL; ++i) {
          int d = lane + 32 * i;
          acc[i] = acc[i] * corr + (d < g.D ? p * ld(v + y + d) : 0.f);
        }
        m = mn;
      }
  const float inv = 1.f / l;
#pragma unroll
  for (int i = 0; i < DPL; ++i) {
    int d = lane + 32 * i;
    if (d < g.D) o[xe + d] = cvt<T>(acc[i] * inv);
  }
  if (lse && lane == 0) lse[row] = (m + log2f(l)) * 0.69314718055994531f;
}

// ------------------------------------------------------------- bwd: D_x
template <typename T>
__global__ void __launch_bounds__(256) fna_bwd_pre(Geom g, Layout ly, const T* __restrict__ o,
                                                   const T* __restrict__ d_o,
                                                   float* __restrict__ Dvec) {
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= (int64_t)g.BH * g.N) return;
  float s = 0.f;
  const int64_t re = elem_of_token(g, ly, (int)(row / g.N), (int)(row % g.N));
  for (int d = lane; d < g.D; d += 32) s = fmaf(ld(o + re + d), ld(d_o + re + d), s);
  s = warp_sum(s);
  if (lane == 0) Dvec[row] = s;
}

// D_x for 16-bit rows: each thread reads 16 bytes (8 elements) of O and dO,
// D/8 consecutive threads own a row and reduce with shuffles (fully
// coalesced 16-byte loads; the kernel is HBM-bound).
// Row-vector mode (lse != nullptr, tensor-core path): instead of D_x at the
// token's index, writes the pair (-LSE_x * log2(e), D_x) into the two planes
// of the class-compacted layout (na_geom.cuh, Geom::rv_*), so the backward
// kernels fetch a chunk's partner values with one TMA box.
// Divisors of the token -> (b*h, residue class, compacted coordinate) map
// as multiply-high magic numbers (the integer divisions dominated this
// HBM-bound kernel for multi-dimensional problems).
struct RvDiv {
  FastDiv n, l[3], dil[3];
};

// Element offset of row `row` (= bh * N + token) in a Q/K/V/O-type tensor
// (Geom::sBH / sX strides), with the same fast divisions.
__device__ __forceinline__ long long row_elem(const Geom& g, const Layout& ly, const RvDiv& f, long long row) {
  const uint32_t r32 = (uint32_t)row;
  const uint32_t bh = fdiv(r32, f.n);
  uint32_t n = r32 - bh * f.n.d;
  long long off = (long long)bh * ly.sBH;
#pragma unroll
  for (int a = 2; a >= 0; --a) {
    if (a < g.rank) {
      const uint32_t rest = fdiv(n, f.l[a]);
      off += (long long)(n - rest * f.l[a].d) * ly.sX[a];
      n = rest;
    }
  }
  return off;
}

__device__ __forceinline__ long long rv_index(const Geom& g, const RvDiv& f, long long row) {
  // B*H*N < 2^31 for any problem whose tensors fit in memory (validated).
  const uint32_t r32 = (uint32_t)row;
  const uint32_t bh = fdiv(r32, f.n);
  uint32_t n = r32 - bh * f.n.d;
  int res = 0, mul = 1;
  long long off = 0;
#pragma unroll
  for (int a = 2; a >= 0; --a) {  // innermost axis first
    if (a < g.rank) {
      const uint32_t rest = fdiv(n, f.l[a]);
      const uint32_t x = n - rest * f.l[a].d;
      n = rest;
      const uint32_t c = fdiv(x, f.dil[a]);
      res += (int)(x - c * f.dil[a].d) * mul;
      mul *= g.dil[a];
      off += (long long)c * g.rv_cs[a];
    }
  }
  return rv_base(g, (int)bh, res) + off;
}

template <typename T, int kPreRows>
__global__ void __launch_bounds__(256) fna_bwd_pre_vec(Geom g, Layout ly, const T* __restrict__ o,
                                                       const T* __restrict__ d_o,
                                                       float* __restrict__ Dvec,
                                                       const float* __restrict__ lse, RvDiv f) {
  // D/8 threads per row; only the tensor-core path (D in {16, 32, 64, 128})
  // launches this kernel, so tpr is a power of two: shift/mask, no 64-bit division.
  // Each thread covers kPreRows rows (one per 256/tpr-row slab of the block),
  // all loads issued before any arithmetic: more bytes in flight per thread
  // (2 for rank 1; the multi-dimensional slot arithmetic prefers 1).
  const int tpr = g.D / 8;
  const int shift = __ffs(tpr) - 1;
  const int64_t slab = 256 >> shift;  // rows per slab
  const int64_t row0 = (int64_t)blockIdx.x * kPreRows * slab + (threadIdx.x >> shift);
  const int part = (int)(threadIdx.x & (tpr - 1));
  const int64_t rows = (int64_t)g.BH * g.N;
  uint4 a[kPreRows], b[kPreRows];
  float l[kPreRows];
  long long i[kPreRows];
#pragma unroll
  for (int k = 0; k < kPreRows; ++k) {
    const int64_t row = row0 + k * slab;
    const bool valid = row < rows;
    // Row-vector mode: LSE and the destination index first, so their latency
    // overlaps the O/dO loads (one HBM round trip per warp, not two).
    l[k] = 0.f;
    i[k] = 0;
    if (lse && part == 0 && valid) {
      l[k] = lse[row];
      i[k] = rv_index(g, f, row);
    }
    const long long re = ly.contig ? row * g.D : (valid ? row_elem(g, ly, f, row) : 0);
    a[k] = valid ? __ldg(reinterpret_cast<const uint4*>(o + re) + part) : make_uint4(0, 0, 0, 0);
    b[k] = valid ? __ldg(reinterpret_cast<const uint4*>(d_o + re) + part) : make_uint4(0, 0, 0, 0);
  }
#pragma unroll
  for (int k = 0; k < kPreRows; ++k) {
    const int64_t row = row0 + k * slab;
    const T* ea = reinterpret_cast<const T*>(&a[k]);
    const T* eb = reinterpret_cast<const T*>(&b[k]);
    float s = 0.f;
#pragma unroll
    for (int e = 0; e < 8; ++e) s = fmaf(ld_val(ea[e]), ld_val(eb[e]), s);
    for (int off = 1; off < tpr; off <<= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (part == 0 && row < rows) {
      if (lse) {
        Dvec[i[k]] = -l[k] * 1.4426950408889634f;
        Dvec[i[k] + g.rv_plane] = s;
      } else {
        Dvec[row] = s;
      }
    }
  }
}

// ------------------------------------------------------------- bwd: dQ
template <typename T, int DPL>
__global__ void __launch_bounds__(256) fna_dq_simt(Geom g, Layout ly, const T* __restrict__ q,
                                                   const T* __restrict__ k,
                                                   const T* __restrict__ v,
                                                   const T* __restrict__ d_o,
                                                   const float* __restrict__ lse,
                                                   float* __restrict__ Dvec,
                                                   T* __restrict__ dq) {
  // 16-bit inputs: D_x read from Dvec is <dO_x, O_x> with the stored
  // (rounded) O, an estimate; c = sum_y P_xy (dP_xy - Dt_x) = D_x - Dt_x and
  // PK = sum_y P_xy k_y are accumulated alongside, dQ = scale (acc - c PK) is
  // the gradient with D_x = sum_y P_xy dP_xy, and Dt_x + c is written back
  // for the dK/dV kernel, which runs after this one (R12).
  constexpr bool kCorr = !std::is_same<T, float>::value;
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= (int64_t)g.BH * g.N) return;
  const int bh = (int)(row / g.N), x = (int)(row % g.N);
  const int64_t base = (int64_t)bh * ly.sBH;
  const Coord co = decode(g, x);
  const int64_t xe = base + elem_of(g, ly, co, co.c);  // this query's row
  float qr[DPL], dor[DPL], acc[DPL], pk[DPL];
  float csum = 0.f;
#pragma unroll
  for (int i = 0; i < DPL; ++i) {
    int d = lane + 32 * i;
    qr[i] = d < g.D ? ld(q + xe + d) : 0.f;
    dor[i] = d < g.D ? ld(d_o + xe + d) : 0.f;
    acc[i] = pk[i] = 0.f;
  }
  const float lse_x = lse[row], D_x = Dvec[row];
  int lo[3], hi[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    lo[a] = a < g.rank ? win_start(co.c[a], co.Lr[a], g.k[a], g.causal[a]) : 0;
    hi[a] = a < g.rank ? win_end(co.c[a], co.Lr[a], g.k[a], g.causal[a]) : 0;
  }
  int cc[3];
  for (cc[0] = lo[0]; cc[0] <= hi[0]; ++cc[0])
    for (cc[1] = lo[1]; cc[1] <= hi[1]; ++cc[1])
      for (cc[2] = lo[2]; cc[2] <= hi[2]; ++cc[2]) {
        const int64_t y = base + elem_of(g, ly, co, cc);
        float s = 0.f, dp = 0.f;
#pragma unroll
        for (int i = 0; i < DPL; ++i) {
          int d = lane + 32 * i;
          if (d < g.D) {
            s = fmaf(qr[i], ld(k + y + d), s);
            dp = fmaf(dor[i], ld(v + y + d), dp);
          }
        }
        s = warp_sum(s);
        dp = warp_sum(dp);
        const float p = __expf(s * g.scale - lse_x);
        const float ds = p * (dp - D_x);
        if constexpr (kCorr) csum += ds;
#pragma unroll
        for (int i = 0; i < DPL; ++i) {
          int d = lane + 32 * i;
          if (d < g.D) {
            const float kv = ld(k + y + d);
            acc[i] = fmaf(ds, kv, acc[i]);
            if constexpr (kCorr) pk[i] = fmaf(p, kv, pk[i]);
          }
        }
      }
#pragma unroll
  for (int i = 0; i < DPL; ++i) {
    int d = lane + 32 * i;
    if (d < g.D) dq[xe + d] = cvt<T>((acc[i] - csum * pk[i]) * g.scale);
  }
  if (kCorr && lane == 0) Dvec[row] = D_x + csum;
}

// ------------------------------------------------------------- bwd: dK, dV
template <typename T, int DPL>
__global__ void __launch_bounds__(256) fna_dkdv_simt(Geom g, Layout ly, const T* __restrict__ q,
                                                     const T* __restrict__ k,
                                                     const T* __restrict__ v,
                                                     const T* __restrict__ d_o,
                                                     const float* __restrict__ lse,
                                                     const float* __restrict__ Dvec,
                                                     T* __restrict__ dk, T* __restrict__ dv) {
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= (int64_t)g.BH * g.N) return;
  const int bh = (int)(row / g.N), y = (int)(row % g.N);
  const int64_t base = (int64_t)bh * ly.sBH;
  const Coord co = decode(g, y);
  const int64_t ye = base + elem_of(g, ly, co, co.c);  // this key's row
  float kr[DPL], vr[DPL], ak[DPL], av[DPL];
#pragma unroll
  for (int i = 0; i < DPL; ++i) {
    int d = lane + 32 * i;
    kr[i] = d < g.D ? ld(k + ye + d) : 0.f;
    vr[i] = d < g.D ? ld(v + ye + d) : 0.f;
    ak[i] = av[i] = 0.f;
  }
  int lo[3], hi[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {   // inverse neighborhood: exact per-axis intervals
    lo[a] = a < g.rank ? inv_start(co.c[a], co.Lr[a], g.k[a], g.causal[a]) : 0;
    hi[a] = a < g.rank ? inv_end(co.c[a], co.Lr[a], g.k[a], g.causal[a]) : 0;
  }
  int cc[3];
  for (cc[0] = lo[0]; cc[0] <= hi[0]; ++cc[0])
    for (cc[1] = lo[1]; cc[1] <= hi[1]; ++cc[1])
      for (cc[2] = lo[2]; cc[2] <= hi[2]; ++cc[2]) {
        const int xt = token_of(g, co, cc);
        const int64_t xo = base + elem_of(g, ly, co, cc);
        float s = 0.f, dp = 0.f;
#pragma unroll
        for (int i = 0; i < DPL; ++i) {
          int d = lane + 32 * i;
          if (d < g.D) {
            s = fmaf(ld(q + xo + d), kr[i], s);
            dp = fmaf(ld(d_o + xo + d), vr[i], dp);
          }
        }
        s = warp_sum(s);
        dp = warp_sum(dp);
        const int64_t xr = (int64_t)bh * g.N + xt;
        const float p = __expf(s * g.scale - lse[xr]);
        const float ds = p * (dp - Dvec[xr]);
#pragma unroll
        for (int i = 0; i < DPL; ++i) {
          int d = lane + 32 * i;
          if (d < g.D) {
            ak[i] = fmaf(ds, ld(q + xo + d), ak[i]);
            av[i] = fmaf(p, ld(d_o + xo + d), av[i]);
          }
        }
      }
#pragma unroll
  for (int i = 0; i < DPL; ++i) {
    int d = lane + 32 * i;
    if (d < g.D) {
      dk[ye + d] = cvt<T>(ak[i] * g.scale);
      dv[ye + d] = cvt<T>(av[i]);
    }
  }
}

template <typename T, int DPL>
cudaError_t launch_fwd(const Geom& g, const Layout& ly, const void* q, const void* k, const void* v, void* o,
                       float* lse, cudaStream_t st) {
  const int64_t rows = (int64_t)g.BH * g.N;
  prof_begin(KID_FWD_SIMT, st);
  fna_fwd_simt<T, DPL><<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(
      g, ly, (const T*)q, (const T*)k, (const T*)v, (T*)o, lse);
  prof_end(st);
  return cudaGetLastError();
}

template <typename T, int DPL>
cudaError_t launch_bwd(const Geom& g, const Layout& ly, const void* q, const void* k, const void* v, const void* o,
                       const void* d_o, const float* lse, void* dq, void* dk, void* dv,
                       float* Dvec, cudaStream_t st) {
  const int64_t rows = (int64_t)g.BH * g.N;
  const unsigned grid = (unsigned)((rows + 7) / 8);
  prof_begin(KID_BWD_PRE, st);
  fna_bwd_pre<T><<<grid, 256, 0, st>>>(g, ly, (const T*)o, (const T*)d_o, Dvec);
  prof_end(st);
  // dQ first: for 16-bit inputs it corrects D_x in Dvec for dK/dV
  prof_begin(KID_DQ_SIMT, st);
  fna_dq_simt<T, DPL><<<grid, 256, 0, st>>>(g, ly, (const T*)q, (const T*)k, (const T*)v,
                                            (const T*)d_o, lse, Dvec, (T*)dq);
  prof_end(st);
  prof_begin(KID_DKDV_SIMT, st);
  fna_dkdv_simt<T, DPL><<<grid, 256, 0, st>>>(g, ly, (const T*)q, (const T*)k, (const T*)v,
                                              (const T*)d_o, lse, Dvec, (T*)dk, (T*)dv);
  prof_end(st);
  return cudaGetLastError();
}

template <typename T>
cudaError_t fwd_by_dim(const Geom& g, const Layout& ly, const void* q, const void* k, const void* v, void* o,
                       float* lse, cudaStream_t st) {
  if (g.D <= 32) return launch_fwd<T, 1>(g, ly, q, k, v, o, lse, st);
  if (g.D <= 64) return launch_fwd<T, 2>(g, ly, q, k, v, o, lse, st);
  if (g.D <= 128) return launch_fwd<T, 4>(g, ly, q, k, v, o, lse, st);
  return launch_fwd<T, 8>(g, ly, q, k, v, o, lse, st);
}

template <typename T>
cudaError_t bwd_by_dim(const Geom& g, const Layout& ly, const void* q, const void* k, const void* v, const void* o,
                       const void* d_o, const float* lse, void* dq, void* dk, void* dv,
                       float* Dvec, cudaStream_t st) {
  if (g.D <= 32) return launch_bwd<T, 1>(g, ly, q, k, v, o, d_o, lse, dq, dk, dv, Dvec, st);
  if (g.D <= 64) return launch_bwd<T, 2>(g, ly, q, k, v, o, d_o, lse, dq, dk, dv, Dvec, st);
  if (g.D <= 128) return launch_bwd<T, 4>(g, ly, q, k, v, o, d_o, lse, dq, dk, dv, Dvec, st);
  return launch_bwd<T, 8>(g, ly, q, k, v, o, d_o, lse, dq, dk, dv, Dvec, st);
}

}  // namespace

cudaError_t simt_fwd(int dtype, const Geom& g, const Layout& ly, const void* q, const void* k, const void* v,
                     void* o, float* lse, cudaStream_t st) {
  switch (dtype) {
    case 0: return fwd_by_dim<float>(g, ly, q, k, v, o, lse, st);
    case 1: return fwd_by_dim<__half>(g, ly, q, k, v, o, lse, st);
    default: return fwd_by_dim<__nv_bfloat16>(g, ly, q, k, v, o, lse, st);
  }
}

cudaError_t rv_clear_padding(const Geom& g, float* Dvec, cudaStream_t st) {
  bool ragged = g.rv_lc[g.rank - 1] * g.dil[g.rank - 1] != g.L[g.rank - 1];
  for (int a = 0; a + 1 < g.rank; ++a) ragged = ragged || g.L[a] % g.dil[a] != 0;
  if (!ragged) return cudaSuccess;
  return cudaMemsetAsync(Dvec, 0, (size_t)g.BH * g.nres * 2 * g.rv_plane * sizeof(float), st);
}

cudaError_t bwd_preprocess(int dtype, const Geom& g, const Layout& ly, const void* o, const void* d_o, const float* lse,
                           float* Dvec, cudaStream_t st) {
  const int64_t rows = (int64_t)g.BH * g.N;
  const unsigned grid = (unsigned)((rows + 7) / 8);
  if (lse) {  // row-vector layout: slots no token maps to (ragged classes) must read as 0
    bool ragged = g.rv_lc[g.rank - 1] * g.dil[g.rank - 1] != g.L[g.rank - 1];
    for (int a = 0; a + 1 < g.rank; ++a) ragged = ragged || g.L[a] % g.dil[a] != 0;
    if (ragged) {
      cudaError_t e = cudaMemsetAsync(Dvec, 0, (size_t)g.BH * g.nres * 2 * g.rv_plane * sizeof(float), st);
      if (e != cudaSuccess) return e;
    }
  }
  RvDiv f;
  f.n = make_fastdiv((uint32_t)g.N);
  for (int a = 0; a < 3; ++a) {
    f.l[a] = make_fastdiv((uint32_t)(a < g.rank ? g.L[a] : 1));
    f.dil[a] = make_fastdiv((uint32_t)(a < g.rank ? g.dil[a] : 1));
  }
  prof_begin(KID_BWD_PRE, st);
  const int rpt = g.rank == 1 ? 2 : 1;  // rows per thread
  const unsigned vgrid = (unsigned)((rows * (g.D / 8) + 256 * rpt - 1) / (256 * rpt));
  switch (dtype) {
    case 0: fna_bwd_pre<float><<<grid, 256, 0, st>>>(g, ly, (const float*)o, (const float*)d_o, Dvec); break;
    case 1:
      if (rpt == 2) fna_bwd_pre_vec<__half, 2><<<vgrid, 256, 0, st>>>(g, ly, (const __half*)o, (const __half*)d_o, Dvec, lse, f);
      else fna_bwd_pre_vec<__half, 1><<<vgrid, 256, 0, st>>>(g, ly, (const __half*)o, (const __half*)d_o, Dvec, lse, f);
      break;
    default:
      if (rpt == 2)
        fna_bwd_pre_vec<__nv_bfloat16, 2><<<vgrid, 256, 0, st>>>(g, ly, (const __nv_bfloat16*)o,
                                                                 (const __nv_bfloat16*)d_o, Dvec, lse, f);
      else
        fna_bwd_pre_vec<__nv_bfloat16, 1><<<vgrid, 256, 0, st>>>(g, ly, (const __nv_bfloat16*)o,
                                                                 (const __nv_bfloat16*)d_o, Dvec, lse, f);
  }
  prof_end(st);
  return cudaGetLastError();
}

cudaError_t simt_bwd(int dtype, const Geom& g, const Layout& ly, const void* q, const void* k, const void* v,
                     const void* o, const void* d_o, const float* lse, void* dq, void* dk,
                     void* dv, float* Dvec, cudaStream_t st) {
  switch (dtype) {
    case 0: return bwd_by_dim<float>(g, ly, q, k, v, o, d_o, lse, dq, dk, dv, Dvec, st);
    case 1: return bwd_by_dim<__half>(g, ly, q, k, v, o, d_o, lse, dq, dk, dv, Dvec, st);
    default: return bwd_by_dim<__nv_bfloat16>(g, ly, q, k, v, o, d_o, lse, dq, dk, dv, Dvec, st);
  }
}

}  // namespace na
