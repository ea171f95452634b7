// tc_bwd.cu — fused neighborhood attention backward on sm_100a tensor cores.
//
// The backward is the paper's operator composition (§3.1) fused
// FlashAttention-style, recomputing the attention weights from the saved LSE
// instead of storing them:
//   dP = PN(dO, V)          dS = P o (dP - D),  D_x = <dO_x, O_x>
//   dQ = scale NN(dS, K)    dK = scale IN(dS, Q)    dV = IN(P, dO)
// Two kernels, each output element has exactly one writer (no atomics):
//   fna_dkdv_tc  key-stationary: a CTA owns 128 keys of one residue class and
//                streams the query chunks of the tile's INVERSE halo
//                [inv_start(y_lo), inv_end(y_hi)] (the IN gather pattern,
//                P:253-258).  Per 64-query sub-chunk: S^T = K Q^T and
//                dP^T = V dO^T (SS MMAs), P^T = exp(scale S^T - LSE_q) and
//                dS^T = P^T (dP^T - D_q) by the compute warps (written back to
//                TMEM as 16-bit), then dV += P^T dO and dK += dS^T Q (TS MMAs).
//   fna_dq_tc    query-stationary over the forward halo: S = Q K^T, dP = dO V^T,
//                dS = P (dP - D), dQ += dS K.
// Warp roles (320 threads, 1 CTA per SM): warp 0 TMA producer, warp 1 TMEM
// owner + single-thread MMA issuer, warps 2..9 two compute warpgroups
// (thread = TMEM lane = stationary row).  Sub-chunk u lives in TMEM buffer
// u%2 and is processed by warpgroup u%2, so the tensor core computes
// sub-chunk u+1 while warpgroup u%2 works on u (ping-pong):
//   MMA order: ST_0, ST_1, [P_0] OUT_0, ST_2, [P_1] OUT_1, ST_3, ...
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "na_geom.cuh"
#include "na_kernels.h"
#include "tc_common.cuh"
#include "tc_plan.h"
#include "tc_ptx.cuh"

namespace na {
namespace {

constexpr int kStages = 2;
constexpr int kThreads = 320;
constexpr float kLog2e = 1.4426950408889634f;

template <int D>
struct BwdSmem {
  static constexpr int kRowBytes = D * 2;
  static constexpr int kTile = 128 * kRowBytes;
  static constexpr int kA0 = 0;                       // stationary tile 0 (K | Q)
  static constexpr int kA1 = kA0 + kTile;             // stationary tile 1 (V | dO)
  static constexpr int kB0 = kA1 + kTile;             // streamed [kStages] (Q | K)
  static constexpr int kB1 = kB0 + kStages * kTile;   // streamed [kStages] (dO | V)
  static constexpr int kVec = kB1 + kStages * kTile;  // [group][slot][LSE2 x64 | D x64] fp32
  static constexpr int kBar = kVec + 2 * 2 * 128 * 4;
  static constexpr int kBytes = kBar + 256;
};

// TMEM columns: [0,128) two 64-column S-like buffers, [128,256) two dP-like
// buffers, [256, 256+D) first output, [256+D, 256+2D) second output.
constexpr uint32_t kColS = 0, kColP = 128, kColOut = 256;

enum : int {
  B_A = 0,                  // stationary tiles loaded
  B_B = 1,                  // streamed stage full [kStages]
  B_E = B_B + kStages,      // streamed stage empty [kStages]
  B_S = B_E + kStages,      // S and dP of a sub-chunk ready [2]
  B_P = B_S + 2,            // packed operands of a sub-chunk written [2] (128 arrivals)
  B_O = B_P + 2,            // outputs final
  B_COUNT = B_O + 1
};

template <int RANK, int D, bool BF16, bool KV_STATIONARY>
__device__ __forceinline__ void bwd_body(const CUtensorMap& map_a0, const CUtensorMap& map_a1,
                                         const CUtensorMap& map_b0, const CUtensorMap& map_b1,
                                         const Geom& g, const TcPlan& pl, const float* __restrict__ lse,
                                         const float* __restrict__ dvec, void* __restrict__ out0,
                                         void* __restrict__ out1) {
  using S = BwdSmem<D>;
  using T = typename std::conditional<BF16, __nv_bfloat16, __half>::type;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + S::kBar);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + B_COUNT);
  float* vec = reinterpret_cast<float*>(smem + S::kVec);

  TileCtx<RANK> t;
  if (!t.init(g, pl, blockIdx.x, /*inverse=*/KV_STATIONARY)) return;
  const int nchunks = t.nchunks;
  const int ns = pl.n_kv > 64 ? 2 : 1;
  const int nsub = nchunks * ns;
  const uint32_t warp = ptx::warp_id(), lane = ptx::lane_id();

  if (threadIdx.x == 0) {
    ptx::mbar_init(bar + B_A, 1);
    for (int s = 0; s < kStages; ++s) {
      ptx::mbar_init(bar + B_B + s, 1);
      ptx::mbar_init(bar + B_E + s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(bar + B_S + b, 1);
      ptx::mbar_init(bar + B_P + b, 128);
    }
    ptx::mbar_init(bar + B_O, 1);
    ptx::fence_barrier_init();
  }
  if (pl.rows_kv < 128) {  // rows no TMA box writes must be finite (zero)
    const int nz = (128 - pl.rows_kv) * S::kRowBytes / 16;
    for (int i = threadIdx.x; i < 2 * kStages * nz; i += kThreads) {
      const int buf = i / nz, off = i % nz;
      uint4* base = reinterpret_cast<uint4*>(smem + S::kB0 + buf * S::kTile + pl.rows_kv * S::kRowBytes);
      base[off] = make_uint4(0, 0, 0, 0);
    }
    ptx::fence_proxy_async();
  }
  if (warp == 1) ptx::tmem_alloc<512>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ===================== TMA producer (whole warp, one lane issues) =====================
    {
      ptx::tma_prefetch(&map_a0);
      ptx::tma_prefetch(&map_a1);
      ptx::tma_prefetch(&map_b0);
      ptx::tma_prefetch(&map_b1);
      ptx::mbar_expect_tx_w(bar + B_A, 2 * 128 * S::kRowBytes);
      for (int i = 0; i < pl.q_issues; ++i) {
        t.template load_box<RANK>(&map_a0, smem + S::kA0 + i * pl.q_box_x * S::kRowBytes, bar + B_A,
                                  t.q_origin, i * pl.q_box_x, g);
        t.template load_box<RANK>(&map_a1, smem + S::kA1 + i * pl.q_box_x * S::kRowBytes, bar + B_A,
                                  t.q_origin, i * pl.q_box_x, g);
      }
      const uint32_t bytes = 2 * pl.rows_kv * S::kRowBytes;
      for (int j = 0; j < nchunks; ++j) {
        const int s = j % kStages;
        if (j >= kStages) ptx::mbar_wait(bar + B_E + s, ((j / kStages) - 1) & 1);
        int org[3];
        t.chunk_origin(pl, j, org);
        ptx::mbar_expect_tx_w(bar + B_B + s, bytes);
        for (int i = 0; i < pl.kv_issues; ++i) {
          t.template load_box<RANK>(&map_b0, smem + S::kB0 + s * S::kTile + i * pl.kv_box_x * S::kRowBytes,
                                    bar + B_B + s, org, i * pl.kv_box_x, g);
          t.template load_box<RANK>(&map_b1, smem + S::kB1 + s * S::kTile + i * pl.kv_box_x * S::kRowBytes,
                                    bar + B_B + s, org, i * pl.kv_box_x, g);
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (whole warp, one lane issues) =====================
    {
      constexpr uint32_t kSw = D == 64 ? 2u : 4u;
      constexpr uint32_t kSbo = 8 * S::kRowBytes;
      const int n1 = pl.n_kv - 64;
      const uint32_t idesc_s0 = ptx::make_idesc(128, ns == 2 ? 64 : pl.n_kv, BF16, false);
      const uint32_t idesc_s1 = ptx::make_idesc(128, ns == 2 ? n1 : 16, BF16, false);
      constexpr uint32_t idesc_o = ptx::make_idesc(128, D, BF16, true);
      const uint32_t a0 = ptx::smem_u32(smem + S::kA0), a1 = ptx::smem_u32(smem + S::kA1);
      auto issue_st = [&](int u) {
        const int j = u / ns, h = u % ns, s = j % kStages;
        if (h == 0) {
          ptx::mbar_wait(bar + B_B + s, (j / kStages) & 1);
          ptx::tc_fence_after();
        }
        const uint32_t off = h * 64 * S::kRowBytes;
        const uint32_t b0 = ptx::smem_u32(smem + S::kB0 + s * S::kTile) + off;
        const uint32_t b1 = ptx::smem_u32(smem + S::kB1 + s * S::kTile) + off;
        const uint32_t id = h ? idesc_s1 : idesc_s0;
        const uint32_t buf = (u & 1) * 64;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          // KV-stationary: S^T = K Q^T, dP^T = V dO^T.  Q-stationary: S = Q K^T, dP = dO V^T.
          ptx::mma_ss_w(tmem + kColS + buf, ptx::make_sdesc(a0 + kk * 32, 16, kSbo, kSw),
                      ptx::make_sdesc(b0 + kk * 32, 16, kSbo, kSw), id, kk > 0);
          ptx::mma_ss_w(tmem + kColP + buf, ptx::make_sdesc(a1 + kk * 32, 16, kSbo, kSw),
                      ptx::make_sdesc(b1 + kk * 32, 16, kSbo, kSw), id, kk > 0);
        }
        ptx::mma_commit_w(bar + B_S + (u & 1));
      };
      ptx::mbar_wait(bar + B_A, 0);
      issue_st(0);
      if (nsub > 1) issue_st(1);
      for (int u = 0; u < nsub; ++u) {
        const int j = u / ns, h = u % ns, s = j % kStages;
        const int width = h ? n1 : (ns == 2 ? 64 : pl.n_kv);
        const uint32_t off = h * 64 * S::kRowBytes;
        const uint32_t b0 = ptx::smem_u32(smem + S::kB0 + s * S::kTile) + off;
        const uint32_t b1 = ptx::smem_u32(smem + S::kB1 + s * S::kTile) + off;
        const uint32_t buf = (u & 1) * 64;
        ptx::mbar_wait(bar + B_P + (u & 1), (u >> 1) & 1);
        ptx::tc_fence_after();
        for (int kk = 0; kk < width / 16; ++kk) {
          const uint32_t boff = kk * 16 * S::kRowBytes;
          const uint32_t acc = (u > 0 || kk > 0) ? 1u : 0u;
          if constexpr (KV_STATIONARY) {
            // dV += P^T dO ; dK += dS^T Q   (B operands MN-major)
            ptx::mma_ts_w(tmem + kColOut + D, tmem + kColS + buf + kk * 8,
                        ptx::make_sdesc(b1 + boff, 128 * S::kRowBytes, kSbo, kSw), idesc_o, acc);
            ptx::mma_ts_w(tmem + kColOut, tmem + kColP + buf + kk * 8,
                        ptx::make_sdesc(b0 + boff, 128 * S::kRowBytes, kSbo, kSw), idesc_o, acc);
          } else {
            // dQ += dS K
            ptx::mma_ts_w(tmem + kColOut, tmem + kColS + buf + kk * 8,
                        ptx::make_sdesc(b0 + boff, 128 * S::kRowBytes, kSbo, kSw), idesc_o, acc);
          }
        }
        if (h == ns - 1) ptx::mma_commit_w(bar + B_E + s);
        if (u + 2 < nsub) issue_st(u + 2);
      }
      ptx::mma_commit_w(bar + B_O);
    }
  } else {
    // ===================== compute warpgroups (2 x 128 threads) =====================
    const int grp = (warp - 2) >> 2;     // processes sub-chunks u with u % 2 == grp
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const int gtid = ((warp - 2) & 3) * 32 + lane;  // 0..127 within the group
    const uint32_t trow = tmem + ((uint32_t)(quarter * 32) << 16);
    RowCtx<RANK> r;
    r.init(g, pl, t, row, /*inverse=*/KV_STATIONARY);
    const float sl2 = g.scale_log2;
    float row_lse2 = 0.f, row_d = 0.f;
    if constexpr (!KV_STATIONARY) {
      if (r.valid) {
        const long long tok = r.out_offset(g, t) / g.D;
        row_lse2 = lse[tok] * kLog2e;
        row_d = dvec[tok];
      }
    }
    uint32_t mw[4] = {0u, 0u, 0u, 0u};
    int it = 0;
    for (int u = grp; u < nsub; u += 2, ++it) {
      const int j = u / ns, h = u % ns;
      int org[3];
      t.chunk_origin(pl, j, org);
      r.chunk_mask(pl, org, mw);
      const uint32_t w0 = h ? mw[2] : mw[0], w1 = h ? mw[3] : mw[1];
      float* cv = vec + (grp * 2 + (it & 1)) * 128;  // [LSE2 x64 | D x64] of this sub-chunk's columns
      if constexpr (KV_STATIONARY) {
        // stage the partner (query) LSE and D values of this sub-chunk's columns
        const int col = gtid & 63, which = gtid >> 6;
        const int ccol = h * 64 + col;  // column within the chunk
        float val = 0.f;
        if (ccol < pl.rows_kv) {
          int rem = ccol;
          bool ok = true;
          long long tok = 0;
#pragma unroll
          for (int a = 2; a >= 0; --a) {
            if (a >= RANK) continue;
            const int cc = org[a] + rem % pl.ckv[a];
            rem /= pl.ckv[a];
            ok = ok && cc < t.Lr[a];
            tok += (long long)(t.r[a] + g.dil[a] * cc) * g.tstride[a];
          }
          if (ok) {
            tok += (long long)t.bh * g.N;
            val = which == 0 ? lse[tok] * kLog2e : dvec[tok];
          }
        }
        cv[which * 64 + col] = val;
        ptx::named_bar_sync(1 + grp, 128);
      }
      const uint32_t buf = (u & 1) * 64;
      ptx::mbar_wait(bar + B_S + (u & 1), (u >> 1) & 1);
      ptx::tc_fence_after();
      uint32_t pk_p[32], pk_s[32];
#pragma unroll
      for (int gq = 0; gq < 2; ++gq) {
        const uint32_t w = gq ? w1 : w0;
        if (!__any_sync(0xffffffffu, w != 0u)) {
#pragma unroll
          for (int c = 0; c < 16; ++c) pk_p[16 * gq + c] = pk_s[16 * gq + c] = 0u;
          continue;
        }
        const bool full = __all_sync(0xffffffffu, w == 0xffffffffu);
        uint32_t sv[32], pv[32];
        NA_TMEM_LD32(trow + kColS + buf + 32 * gq, sv);
        NA_TMEM_LD32(trow + kColP + buf + 32 * gq, pv);
        ptx::tmem_ld_wait();
#pragma unroll
        for (int c = 0; c < 32; c += 2) {
          float2 nl, dd;
          if constexpr (KV_STATIONARY) {
            nl = make_float2(-cv[32 * gq + c], -cv[32 * gq + c + 1]);
            dd = make_float2(cv[64 + 32 * gq + c], cv[64 + 32 * gq + c + 1]);
          } else {
            nl = make_float2(-row_lse2, -row_lse2);
            dd = make_float2(row_d, row_d);
          }
          float2 x = __ffma2_rn(make_float2(__uint_as_float(sv[c]), __uint_as_float(sv[c + 1])),
                                make_float2(sl2, sl2), nl);
          if (!full) {
            x.x = (w >> c) & 1u ? x.x : -INFINITY;
            x.y = (w >> (c + 1)) & 1u ? x.y : -INFINITY;
          }
          const float2 p = make_float2(ptx::ex2(x.x), ptx::ex2(x.y));
          const float2 ds = __fmul2_rn(p, __fadd2_rn(make_float2(__uint_as_float(pv[c]),
                                                                 __uint_as_float(pv[c + 1])),
                                                     make_float2(-dd.x, -dd.y)));
          pk_p[16 * gq + (c >> 1)] = pack2<BF16>(p.x, p.y);
          pk_s[16 * gq + (c >> 1)] = pack2<BF16>(ds.x, ds.y);
        }
      }
      if constexpr (KV_STATIONARY) {
        NA_TMEM_ST32(trow + kColS + buf, pk_p);  // P^T  -> A of dV += P^T dO
        NA_TMEM_ST32(trow + kColP + buf, pk_s);  // dS^T -> A of dK += dS^T Q
      } else {
        NA_TMEM_ST32(trow + kColS + buf, pk_s);  // dS -> A of dQ += dS K
      }
      ptx::tmem_st_wait();
      ptx::tc_fence_before();
      ptx::mbar_arrive(bar + B_P + (u & 1));
    }
    // ---- epilogue ----
    ptx::mbar_wait(bar + B_O, 0);
    ptx::tc_fence_after();
    // KV-stationary: group 0 writes dK (x scale), group 1 writes dV.
    // Q-stationary: the two groups split dQ's D columns.
    const long long off = r.out_offset(g, t);
    constexpr int kCols = KV_STATIONARY ? D : D / 2;
    const uint32_t src = KV_STATIONARY ? kColOut + grp * D : kColOut + grp * (D / 2);
    T* dst = reinterpret_cast<T*>(KV_STATIONARY && grp ? out1 : out0) + off +
             (KV_STATIONARY ? 0 : grp * (D / 2));
    const float mul = (KV_STATIONARY && grp) ? 1.f : g.scale;
#pragma unroll
    for (int c0 = 0; c0 < kCols; c0 += 16) {
      uint32_t ov[16];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(ov[0]), "=r"(ov[1]), "=r"(ov[2]), "=r"(ov[3]), "=r"(ov[4]), "=r"(ov[5]), "=r"(ov[6]),
            "=r"(ov[7]), "=r"(ov[8]), "=r"(ov[9]), "=r"(ov[10]), "=r"(ov[11]), "=r"(ov[12]),
            "=r"(ov[13]), "=r"(ov[14]), "=r"(ov[15])
          : "r"(trow + src + c0));
      ptx::tmem_ld_wait();
      if (r.valid) {
        uint32_t pk[8];
#pragma unroll
        for (int c = 0; c < 16; c += 2)
          pk[c >> 1] = pack2<BF16>(__uint_as_float(ov[c]) * mul, __uint_as_float(ov[c + 1]) * mul);
        uint4* d4 = reinterpret_cast<uint4*>(dst + c0);
        d4[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        d4[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem);
  }
}

// dK, dV: key-stationary over the inverse halo.
template <int RANK, int D, bool BF16>
__global__ void __launch_bounds__(kThreads, 1)
    fna_dkdv_tc(const __grid_constant__ CUtensorMap map_k, const __grid_constant__ CUtensorMap map_v,
                const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_do,
                Geom g, TcPlan pl, const float* __restrict__ lse, const float* __restrict__ dvec,
                void* __restrict__ dk, void* __restrict__ dv) {
  bwd_body<RANK, D, BF16, true>(map_k, map_v, map_q, map_do, g, pl, lse, dvec, dk, dv);
}

// dQ: query-stationary over the forward halo.
template <int RANK, int D, bool BF16>
__global__ void __launch_bounds__(kThreads, 1)
    fna_dq_tc(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_do,
              const __grid_constant__ CUtensorMap map_k, const __grid_constant__ CUtensorMap map_v,
              Geom g, TcPlan pl, const float* __restrict__ lse, const float* __restrict__ dvec,
              void* __restrict__ dq) {
  bwd_body<RANK, D, BF16, false>(map_q, map_do, map_k, map_v, g, pl, lse, dvec, dq, nullptr);
}

template <int RANK, int D, bool BF16>
cudaError_t launch_both(const Geom& g, const TcPlan& pl, const CUtensorMap* m, const float* lse,
                        const float* dvec, void* dq, void* dk, void* dv, cudaStream_t st) {
  // m: [0] Q tile, [1] K tile, [2] V tile, [3] dO tile, [4] Q chunk, [5] K chunk,
  //    [6] V chunk, [7] dO chunk
  const int smem = BwdSmem<D>::kBytes + 1024;
  auto kdkdv = fna_dkdv_tc<RANK, D, BF16>;
  auto kdq = fna_dq_tc<RANK, D, BF16>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kdkdv, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(kdq, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const long long grid = (long long)g.BH * pl.nres * pl.tiles;
  if (grid > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
  prof_begin(KID_DKDV_TC, st);
  kdkdv<<<(unsigned)grid, kThreads, smem, st>>>(m[1], m[2], m[4], m[7], g, pl, lse, dvec, dk, dv);
  prof_end(st);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  prof_begin(KID_DQ_TC, st);
  kdq<<<(unsigned)grid, kThreads, smem, st>>>(m[0], m[3], m[5], m[6], g, pl, lse, dvec, dq);
  prof_end(st);
  return cudaGetLastError();
}

template <int RANK>
cudaError_t by_type(int dtype, const Geom& g, const TcPlan& pl, const CUtensorMap* m,
                    const float* lse, const float* dvec, void* dq, void* dk, void* dv,
                    cudaStream_t st) {
  const bool bf = dtype == 2;
  if (g.D == 64)
    return bf ? launch_both<RANK, 64, true>(g, pl, m, lse, dvec, dq, dk, dv, st)
              : launch_both<RANK, 64, false>(g, pl, m, lse, dvec, dq, dk, dv, st);
  return bf ? launch_both<RANK, 32, true>(g, pl, m, lse, dvec, dq, dk, dv, st)
            : launch_both<RANK, 32, false>(g, pl, m, lse, dvec, dq, dk, dv, st);
}

}  // namespace

cudaError_t tc_bwd(int dtype, const Geom& g, const void* q, const void* k, const void* v,
                   const void* o, const void* d_o, const float* lse, void* dq, void* dk, void* dv,
                   float* Dvec, cudaStream_t st, int* launches) {
  const char* why;
  if (!tc_supported(dtype, g, &why)) return cudaErrorNotSupported;
  cudaError_t e = bwd_preprocess(dtype, g, o, d_o, Dvec, st);
  if (e != cudaSuccess) return e;
  TcPlan pl = make_plan(g, 128);
  CUtensorMap m[8];
  const void* ptrs[4] = {q, k, v, d_o};
  for (int i = 0; i < 4; ++i) {
    if ((e = make_map(&m[i], dtype, g, ptrs[i], pl.tq, pl.q_box_x)) != cudaSuccess) return e;
    if ((e = make_map(&m[4 + i], dtype, g, ptrs[i], pl.ckv, pl.kv_box_x)) != cudaSuccess) return e;
  }
  *launches = 3;
  switch (g.rank) {
    case 1: return by_type<1>(dtype, g, pl, m, lse, Dvec, dq, dk, dv, st);
    case 2: return by_type<2>(dtype, g, pl, m, lse, Dvec, dq, dk, dv, st);
    default: return by_type<3>(dtype, g, pl, m, lse, Dvec, dq, dk, dv, st);
  }
}

}  // namespace na
