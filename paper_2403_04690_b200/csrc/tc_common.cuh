// tc_common.cuh — tile / row bookkeeping shared by the tcgen05 kernels, and
// the host helpers that build their plan and TMA tensor maps.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <type_traits>

#include "na_geom.cuh"
#include "tc_plan.h"
#include "tc_ptx.cuh"

namespace na {

// Host side (tc_host.cpp).
// `pick`: which of the kTopPlans cheapest candidates of the cost model
// (0 = cheapest); *ncand (if given) = how many exist (1 for rank 1).
TcPlan make_plan(const Geom& g, int tile_rows, int pick = 0, int* ncand = nullptr);
// (plan_choice / set_plan_choice: na_kernels.h)
int num_sms();  // SMs of the current device (cached per device)
cudaError_t make_map(CUtensorMap* map, int dtype, const Geom& g, const Layout& ly, const void* base,
                     const int box[3], int box_x);

template <bool BF16>
__device__ __forceinline__ uint32_t pack2(float a, float b) {
  if constexpr (BF16) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
  } else {
    __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
  }
}

template <bool BF16>
__device__ __forceinline__ float2 unpack2(uint32_t w) {
  if constexpr (BF16) {
    return __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w));
  } else {
    return __half22float2(*reinterpret_cast<const __half2*>(&w));
  }
}

// acc + the two bf16 halves of w, each in fp32 (one mixed-precision
// add.f32.bf16 per half, FHADD.BF16 with a half selector in SASS; no unpack).
__device__ __forceinline__ float2 add_bf16x2(float2 acc, uint32_t w) {
  float2 r;
  asm("{\n\t.reg .b16 l, h;\n\tmov.b32 {l, h}, %2;\n\t"
      "add.rn.f32.bf16 %0, l, %3;\n\tadd.rn.f32.bf16 %1, h, %4;\n\t}"
      : "=f"(r.x), "=f"(r.y)
      : "r"(w), "f"(acc.x), "f"(acc.y));
  return r;
}

// 2^x for a pair of values on the FMA pipe (the MUFU ex2 unit is the
// scarcest resource of the softmax): Cody-Waite split x = n + f with
// n = rint(x), f in [-0.5, 0.5]; 2^f by a degree-3 polynomial with c0 = 1
// exactly (relative error 1.1e-4, below half an fp16 ulp; P is rounded to
// 16 bits before the PV MMA); 2^n is added to the exponent field.  x is
// clamped to >= -127 so a masked logit (-inf) yields +0 (n = -127, f = 0).
__device__ __forceinline__ float2 exp2_poly2(float2 x) {
  constexpr float kC1 = 0.6933686137f, kC2 = 0.2422178388f, kC3 = 0.0545928255f;
  x.x = fmaxf(x.x, -127.f);
  x.y = fmaxf(x.y, -127.f);
  const float2 t = __fadd2_rn(x, make_float2(12582912.f, 12582912.f));  // 1.5*2^23: rint in low bits
  const float2 n = __fadd2_rn(t, make_float2(-12582912.f, -12582912.f));
  const float2 f = __fadd2_rn(x, make_float2(-n.x, -n.y));
  float2 p = __ffma2_rn(f, make_float2(kC3, kC3), make_float2(kC2, kC2));
  p = __ffma2_rn(p, f, make_float2(kC1, kC1));
  p = __ffma2_rn(p, f, make_float2(1.f, 1.f));
  const int ex = (__float_as_int(t.x) - 0x4B400000) << 23;
  const int ey = (__float_as_int(t.y) - 0x4B400000) << 23;
  return make_float2(__int_as_float(__float_as_int(p.x) + ex), __int_as_float(__float_as_int(p.y) + ey));
}

// Which exponentials go to the FMA-pipe polynomial: at column c of a
// 4-column step (c = 0, 4, ..., 28 within a 32-column group) the step's
// second pair.  Mode 0: none; 1: steps with c & 4 (25 % of the elements);
// 2: every step (50 %); 3: c & 12 == 4 (12.5 %).  The polynomial costs ~6
// issue slots per element against ~1 for MUFU, so the best share depends
// on how MUFU- vs issue-bound a kernel is: measured per kernel and rank
// (round 2, session 3) -- forward rank 1: 1, rank
// 2/3: 0; dK/dV rank 1/2: 0, rank 3: 1; dQ: 1, head_dim <= 32: 3.
// NA_POLY_MODE (build flag) overrides every kernel's choice.
template <int MODE>
__device__ __forceinline__ constexpr bool use_poly(int c) {
#ifdef NA_POLY_MODE
  constexpr int m = NA_POLY_MODE;
#else
  constexpr int m = MODE;
#endif
  return m == 2 ? true : m == 1 ? (c & 4) != 0 : m == 3 ? (c & 12) == 4 : false;
}

// Which (b*h, residue class, tile) a CTA owns, and the tile's halo.
// `tile` = the 128-token box this CTA is stationary on (queries in the
// forward and dQ kernels, keys in the dK/dV kernel); `inverse` selects
// whether its streamed partner range is the forward halo
// [start(lo), end(hi)] or the inverse halo [inv_start(lo), inv_end(hi)].
template <int RANK>
struct TileCtx {
  int bh;
  int res;        // flat residue class (r[0] * dil[1] + r[1]) * dil[2] + r[2]
  int r[3];       // residue per axis
  int Lr[3];      // class size per axis
  int q_origin[3];
  int qv[3];      // valid extent of the tile per axis
  int lo[3];      // halo low corner
  int nch[3];     // chunks per axis
  int nchunks;

  __device__ __forceinline__ bool init(const Geom& g, const TcPlan& pl, unsigned block,
                                       bool inverse = false) {
    const uint32_t rest = fdiv(block, pl.f_tiles);
    uint32_t tile = block - rest * pl.f_tiles.d;
    const uint32_t bhq = fdiv(rest, pl.f_nres);
    uint32_t res = rest - bhq * pl.f_nres.d;
    bh = (int)bhq;
    this->res = (int)res;
    nchunks = 1;
#pragma unroll
    for (int a = 2; a >= 0; --a) {
      if (a >= RANK) {
        r[a] = 0; Lr[a] = 1; q_origin[a] = 0; qv[a] = 1; lo[a] = 0; nch[a] = 1;
        continue;
      }
      const uint32_t rq = fdiv(res, pl.f_dil[a]);
      r[a] = (int)(res - rq * pl.f_dil[a].d);
      res = rq;
      const uint32_t tq_ = fdiv(tile, pl.f_ntile[a]);
      const int ti = (int)(tile - tq_ * pl.f_ntile[a].d);
      tile = tq_;
      Lr[a] = (int)fdiv((uint32_t)(g.L[a] - r[a] + g.dil[a] - 1), pl.f_dil[a]);
      q_origin[a] = ti * pl.tq[a];
      qv[a] = min(pl.tq[a], Lr[a] - q_origin[a]);
      int hi;
      if (!inverse) {
        lo[a] = win_start(q_origin[a], Lr[a], g.k[a], g.causal[a]);
        hi = win_end(q_origin[a] + qv[a] - 1, Lr[a], g.k[a], g.causal[a]);
      } else {
        lo[a] = inv_start(q_origin[a], Lr[a], g.k[a], g.causal[a]);
        hi = inv_end(q_origin[a] + qv[a] - 1, Lr[a], g.k[a], g.causal[a]);
      }
      nch[a] = (int)fdiv((uint32_t)(hi - lo[a] + pl.ckv[a]), pl.f_ckv[a]);
      nchunks *= nch[a];
    }
#pragma unroll
    for (int a = 0; a < RANK; ++a)
      if (qv[a] <= 0) return false;
    return true;
  }

  __device__ __forceinline__ void chunk_origin(const TcPlan& pl, int j, int org[3]) const {
    int rem = j;
#pragma unroll
    for (int a = 2; a >= 0; --a) {
      if (a >= RANK) { org[a] = 0; continue; }
      if (a == 0) {  // outermost axis: rem < nch[0] already
        org[a] = lo[a] + rem * pl.ckv[a];
      } else {
        org[a] = lo[a] + (rem % nch[a]) * pl.ckv[a];
        rem /= nch[a];
      }
    }
  }

  // Odometer step from chunk j's origin to chunk j+1's (innermost axis
  // fastest, the order of chunk_origin) without divisions.
  __device__ __forceinline__ void next_origin(const TcPlan& pl, int org[3]) const {
#pragma unroll
    for (int a = RANK - 1; a >= 0; --a) {
      org[a] += pl.ckv[a];
      if (a == 0 || org[a] < lo[a] + nch[a] * pl.ckv[a]) break;
      org[a] = lo[a];
    }
  }

  // TMA load of a box whose compacted corner is `org` (+x_off on the
  // innermost axis).  Coordinates are original-tensor element coordinates
  // r + dil * c; the tensor map's elementStrides = dil walks the class.
  // c0: first head_dim column (64 for the second half of a 128-wide row).
  template <int R>
  __device__ __forceinline__ void load_box(const CUtensorMap* m, void* dst, uint64_t* bar,
                                           const int org[3], int x_off, const Geom& g, int c0 = 0) const {
    if constexpr (R == 1) {
      ptx::tma_load_3d_w(dst, m, bar, c0, r[0] + g.dil[0] * (org[0] + x_off), bh);
    } else if constexpr (R == 2) {
      ptx::tma_load_4d_w(dst, m, bar, c0, r[1] + g.dil[1] * (org[1] + x_off),
                       r[0] + g.dil[0] * org[0], bh);
    } else {
      ptx::tma_load_5d_w(dst, m, bar, c0, r[2] + g.dil[2] * (org[2] + x_off),
                       r[1] + g.dil[1] * org[1], r[0] + g.dil[0] * org[0], bh);
    }
  }

  // TMA store of the stationary tile's box (one thread issues).
  template <int R>
  __device__ __forceinline__ void store_box(const CUtensorMap* m, const void* src, int x_off,
                                            const Geom& g, int c0 = 0) const {
    if constexpr (R == 1) {
      ptx::tma_store_3d(m, src, c0, r[0] + g.dil[0] * (q_origin[0] + x_off), bh);
    } else if constexpr (R == 2) {
      ptx::tma_store_4d(m, src, c0, r[1] + g.dil[1] * (q_origin[1] + x_off), r[0] + g.dil[0] * q_origin[0],
                        bh);
    } else {
      ptx::tma_store_5d(m, src, c0, r[2] + g.dil[2] * (q_origin[2] + x_off), r[1] + g.dil[1] * q_origin[1],
                        r[0] + g.dil[0] * q_origin[0], bh);
    }
  }
};

// First tile >= `tile` (stepping by gridDim.x) whose context is valid; fills
// `t` and returns it, or returns num_tiles when the CTA has none left.
template <int RANK, bool INVERSE>
__device__ __forceinline__ unsigned seek_tile(const Geom& g, const TcPlan& pl, unsigned tile, unsigned num_tiles,
                                              TileCtx<RANK>& t) {
  for (; tile < num_tiles; tile += gridDim.x)
    if (t.init(g, pl, tile, INVERSE)) break;
  return tile;
}

// Bits [lo - 32*w0, hi - 32*w0] (inclusive, clipped) of 32-bit words w0, w0+1, ...
// OR-ed into mw[0..NW); branch-free (64-bit shifts handle the 32-bit edge).
template <int NW>
__device__ __forceinline__ void set_range_w(uint32_t* mw, int lo, int hi, int w0) {
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    const int off = 32 * (w0 + w);
    const int a = min(max(lo - off, 0), 32);
    const int b = min(max(hi - off + 1, a), 32);
    mw[w] |= (uint32_t)(((1ull << b) - 1ull) ^ ((1ull << a) - 1ull));
  }
}
__device__ __forceinline__ void set_range(uint32_t mw[4], int lo, int hi) { set_range_w<4>(mw, lo, hi, 0); }

// 2^n - 1 for n in [0, 64] (n >= 64: all ones).
__device__ __forceinline__ unsigned long long lowbits64(int n) {
  return n >= 64 ? ~0ull : (n <= 0 ? 0ull : (1ull << n) - 1ull);
}
// OR bits [a, b] (a <= b, within [0, 128)) into the 128-bit value (lo, hi).
__device__ __forceinline__ void range128(int a, int b, unsigned long long& lo, unsigned long long& hi) {
  lo |= lowbits64(b + 1) & ~lowbits64(a);
  hi |= lowbits64(b + 1 - 64) & ~lowbits64(a - 64);
}

// One row (= one TMEM lane = one thread) of a stationary tile.
template <int RANK>
struct RowCtx {
  int c[3];         // compacted coordinate of this row's token
  int wlo[3], whi[3];  // partner interval per axis (window or inverse window)
  bool valid;

  __device__ __forceinline__ void init(const Geom& g, const TcPlan& pl, const TileCtx<RANK>& t,
                                       int row, bool inverse = false) {
    valid = true;
    int rem = row;
#pragma unroll
    for (int a = 2; a >= 0; --a) {
      if (a >= RANK) { c[a] = 0; wlo[a] = 0; whi[a] = 0; continue; }
      const int off = rem & (pl.tq[a] - 1);  // tile extents are powers of two
      rem >>= pl.tq_shift[a];
      c[a] = t.q_origin[a] + off;
      valid = valid && off < t.qv[a];
      if (!inverse) {
        wlo[a] = win_start(c[a], t.Lr[a], g.k[a], g.causal[a]);
        whi[a] = win_end(c[a], t.Lr[a], g.k[a], g.causal[a]);
      } else {
        wlo[a] = inv_start(c[a], t.Lr[a], g.k[a], g.causal[a]);
        whi[a] = inv_end(c[a], t.Lr[a], g.k[a], g.causal[a]);
      }
    }
    if (!valid) {
#pragma unroll
      for (int a = 0; a < 3; ++a) { wlo[a] = 1; whi[a] = 0; }
    }
  }

  // Index of this row's token in a [BH, N] row vector (LSE).
  __device__ __forceinline__ long long token_index(const Geom& g, const TileCtx<RANK>& t) const {
    long long tok = 0;
#pragma unroll
    for (int a = 0; a < RANK; ++a) tok += (long long)(t.r[a] + g.dil[a] * c[a]) * g.tstride[a];
    return (long long)t.bh * g.N + tok;
  }
  // Element offset of this row's token in a [BH, N, D] tensor.
  __device__ __forceinline__ long long out_offset(const Geom& g, const TileCtx<RANK>& t) const {
    return token_index(g, t) * g.D;
  }

  // Validity bitmask of the <=128 chunk columns for this row: column
  // (lt*ckv1 + ly)*ckv2 + lx is the key at org + (lt, ly, lx).
  // Validity bits of the 64 columns [64h, 64h + 64) of the chunk at `org`.
  __device__ __forceinline__ void sub_mask(const TcPlan& pl, const int org[3], int h, uint32_t w[2]) const {
    if constexpr (RANK == 1) {
      w[0] = w[1] = 0u;
      const int lo = max(wlo[0] - org[0], 0), hi = min(whi[0] - org[0], pl.ckv[0] - 1);
      set_range_w<2>(w, lo, hi, 2 * h);
    } else {
      uint32_t mw[4];
      chunk_mask(pl, org, mw);
      w[0] = h ? mw[2] : mw[0];
      w[1] = h ? mw[3] : mw[1];
    }
  }

  __device__ __forceinline__ void chunk_mask(const TcPlan& pl, const int org[3], uint32_t mw[4]) const {
    if constexpr (RANK == 1) {
      mw[0] = mw[1] = mw[2] = mw[3] = 0u;
      int lo = wlo[0] - org[0], hi = whi[0] - org[0];
      lo = lo < 0 ? 0 : lo;
      hi = hi > pl.ckv[0] - 1 ? pl.ckv[0] - 1 : hi;
      set_range(mw, lo, hi);
    } else {
      // window on the innermost axis, replicated on every chunk row by one
      // multiplication, then AND-ed with the rows whose outer coordinates are
      // inside the window (an interval of rows per outermost index).
      constexpr int ax = RANK - 1;
      const int cx = pl.ckv[ax];
      const int xlo = max(wlo[ax] - org[ax], 0), xhi = min(whi[ax] - org[ax], cx - 1);
      const int ylo = max(wlo[ax - 1] - org[ax - 1], 0), yhi = min(whi[ax - 1] - org[ax - 1], pl.ckv[ax - 1] - 1);
      unsigned long long rlo = 0ull, rhi = 0ull;
      if (cx > 64) {  // then the chunk is a single row of the innermost axis
        bool ok = xlo <= xhi && ylo <= yhi;
        if constexpr (RANK == 3) ok = ok && wlo[0] <= org[0] && org[0] <= whi[0];
        if (ok) range128(xlo, xhi, rlo, rhi);
      } else if (xlo <= xhi && ylo <= yhi) {
        const unsigned long long xm = lowbits64(xhi + 1) & ~lowbits64(xlo);  // cx <= 64 when rows > 1
        const unsigned long long rep_lo = xm * pl.rep_lo;
        const unsigned long long rep_hi = xm * pl.rep_hi | (pl.rep_sh ? xm >> pl.rep_sh : 0ull);
        if constexpr (RANK == 2) {
          range128(ylo * cx, (yhi + 1) * cx - 1, rlo, rhi);
          rlo &= rep_lo;
          rhi &= rep_hi;
        } else {
          const int c1 = pl.ckv[1];
          const int tlo = max(wlo[0] - org[0], 0), thi = min(whi[0] - org[0], pl.ckv[0] - 1);
          if (pl.ckv[0] == 1) {  // one outermost slice: the rank-2 pattern if it is inside
            if (tlo <= thi) range128(ylo * cx, (yhi + 1) * cx - 1, rlo, rhi);
            rlo &= rep_lo;
            rhi &= rep_hi;
          } else if (tlo <= thi) {
            // one slice's (y, x) pattern, then replicated over the slices
            const int S = c1 * cx;
            const unsigned long long slice =
                (xm * pl.rep1) & lowbits64((yhi + 1) * cx) & ~lowbits64(ylo * cx);
            const unsigned long long f_lo = slice * pl.rep2_lo;
            const unsigned long long f_hi = slice * pl.rep2_hi | (pl.rep2_sh ? slice >> pl.rep2_sh : 0ull);
            range128(tlo * S, (thi + 1) * S - 1, rlo, rhi);
            rlo &= f_lo;
            rhi &= f_hi;
          }
        }
      }
      mw[0] = (uint32_t)rlo;
      mw[1] = (uint32_t)(rlo >> 32);
      mw[2] = (uint32_t)rhi;
      mw[3] = (uint32_t)(rhi >> 32);
    }
  }
};

}  // namespace na
