// tc_fwd.cu — fused neighborhood attention forward on sm_100a tensor cores.
//
// One CTA = one 128-query multi-dimensional tile of one residue class of one
// (b, h) (§3.3 fused NA, Fig. 4; dilation as extra CTAs P:329-331).
// Warp roles (192 threads, 2 CTAs per SM):
//   warp 0      TMA producer: Q box once, then K and V boxes of every KV chunk
//               of the tile's halo (a 2-stage mbarrier ring).
//   warp 1      TMEM owner + single-thread tcgen05.mma issuer:
//                 S = Q K^T  (SS, fp32 accumulate in TMEM cols [0,128))
//                 O += P V   (TS: P read from TMEM cols [0,64), V MN-major)
//   warps 2..5  softmax: thread = query row = TMEM lane.  tcgen05.ld its S
//               row, applies the neighborhood mask (per-row window bitmask,
//               P:295), online softmax in the log2 domain with lazy
//               O rescaling, writes P (16-bit) back into TMEM,
//               and finally normalizes O and stores O and LSE.
// Only chunks of the tile's halo box [start(q_lo), end(q_hi)] are visited
// (tile skipping: every other KV tile has no key in any row's window).
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
constexpr int kThreads = 192;

template <int D>
struct FwdSmem {
  static constexpr int kRowBytes = D * 2;
  static constexpr int kTile = 128 * kRowBytes;  // Q tile, or one K/V stage
  static constexpr int kQ = 0;
  static constexpr int kK = kQ + kTile;
  static constexpr int kV = kK + kStages * kTile;
  static constexpr int kBar = kV + kStages * kTile;
  static constexpr int kBytes = kBar + 256;
};

template <int RANK, int D, bool BF16>
__global__ void __launch_bounds__(kThreads, 2)
    fna_fwd_tc(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_k,
               const __grid_constant__ CUtensorMap map_v, Geom g, TcPlan pl, void* __restrict__ o_ptr,
               float* __restrict__ lse) {
  using S = FwdSmem<D>;
  using T = typename std::conditional<BF16, __nv_bfloat16, __half>::type;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S::kBar);
  uint64_t* bar_q = bars + 0;
  uint64_t* bar_k = bars + 1;                 // [kStages]
  uint64_t* bar_v = bars + 1 + kStages;       // [kStages]
  uint64_t* bar_e = bars + 1 + 2 * kStages;   // kv stage empty [kStages]
  uint64_t* bar_s = bars + 1 + 3 * kStages;   // S ready in TMEM
  uint64_t* bar_p = bar_s + 1;                // P written to TMEM (128 arrivals)
  uint64_t* bar_o = bar_s + 2;                // final O ready
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar_s + 3);

  // ---- which tile is this CTA -------------------------------------------
  TileCtx<RANK> t;
  if (!t.init(g, pl, blockIdx.x)) return;  // tile beyond a ragged class: no work
  const int nchunks = t.nchunks;

  const uint32_t warp = ptx::warp_id(), lane = ptx::lane_id();
  if (threadIdx.x == 0) {
    ptx::mbar_init(bar_q, 1);
    for (int s = 0; s < kStages; ++s) {
      ptx::mbar_init(bar_k + s, 1);
      ptx::mbar_init(bar_v + s, 1);
      ptx::mbar_init(bar_e + s, 1);
    }
    ptx::mbar_init(bar_s, 1);
    ptx::mbar_init(bar_p, 128);
    ptx::mbar_init(bar_o, 1);
    ptx::fence_barrier_init();
  }
  // Zero the K/V rows no TMA box writes (rows_kv..127): the MMA reads up to
  // n_kv rows and 0 * garbage could be NaN.
  if (pl.rows_kv < 128) {
    const int nz = (128 - pl.rows_kv) * S::kRowBytes / 16;
    for (int i = threadIdx.x; i < 2 * kStages * nz; i += kThreads) {
      const int buf = i / nz, off = i % nz;
      uint4* base = reinterpret_cast<uint4*>(smem + S::kK + buf * S::kTile + pl.rows_kv * S::kRowBytes);
      base[off] = make_uint4(0, 0, 0, 0);
    }
    ptx::fence_proxy_async();
  }
  if (warp == 1) ptx::tmem_alloc<256>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  constexpr uint32_t kColS = 0, kColO = 128;

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      ptx::tma_prefetch(&map_q);
      ptx::tma_prefetch(&map_k);
      ptx::tma_prefetch(&map_v);
      ptx::mbar_expect_tx(bar_q, 128 * S::kRowBytes);
      for (int i = 0; i < pl.q_issues; ++i)
        t.template load_box<RANK>(&map_q, smem + S::kQ + i * pl.q_box_x * S::kRowBytes, bar_q,
                                  t.q_origin, i * pl.q_box_x, g);
      const uint32_t kv_bytes = pl.rows_kv * S::kRowBytes;
      for (int j = 0; j < nchunks; ++j) {
        const int s = j % kStages;
        if (j >= kStages) ptx::mbar_wait(bar_e + s, ((j / kStages) - 1) & 1);
        int org[3];
        t.chunk_origin(pl, j, org);
        uint8_t* kd = smem + S::kK + s * S::kTile;
        uint8_t* vd = smem + S::kV + s * S::kTile;
        ptx::mbar_expect_tx(bar_k + s, kv_bytes);
        for (int i = 0; i < pl.kv_issues; ++i)
          t.template load_box<RANK>(&map_k, kd + i * pl.kv_box_x * S::kRowBytes, bar_k + s, org,
                                    i * pl.kv_box_x, g);
        ptx::mbar_expect_tx(bar_v + s, kv_bytes);
        for (int i = 0; i < pl.kv_issues; ++i)
          t.template load_box<RANK>(&map_v, vd + i * pl.kv_box_x * S::kRowBytes, bar_v + s, org,
                                    i * pl.kv_box_x, g);
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    if (lane == 0) {
      constexpr uint32_t kSw = D == 64 ? 2u : 4u;               // SW128 : SW64
      constexpr uint32_t kSbo = 8 * S::kRowBytes;               // 8-row core-matrix group
      const uint32_t idesc_s = ptx::make_idesc(128, pl.n_kv, BF16, false);
      constexpr uint32_t idesc_o = ptx::make_idesc(128, D, BF16, true);
      const uint32_t q_addr = ptx::smem_u32(smem + S::kQ);
      ptx::mbar_wait(bar_q, 0);
      for (int j = 0; j < nchunks; ++j) {
        const int s = j % kStages;
        const uint32_t ph = (j / kStages) & 1;
        const uint32_t k_addr = ptx::smem_u32(smem + S::kK + s * S::kTile);
        const uint32_t v_addr = ptx::smem_u32(smem + S::kV + s * S::kTile);
        ptx::mbar_wait(bar_k + s, ph);
        ptx::tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)  // S = Q K^T, K-dim = head_dim
          ptx::mma_ss(tmem + kColS, ptx::make_sdesc(q_addr + kk * 32, 16, kSbo, kSw),
                      ptx::make_sdesc(k_addr + kk * 32, 16, kSbo, kSw), idesc_s, kk > 0);
        ptx::mma_commit(bar_s);
        ptx::mbar_wait(bar_p, j & 1);  // softmax wrote P_j (and rescaled O)
        ptx::mbar_wait(bar_v + s, ph);
        ptx::tc_fence_after();
        for (int kk = 0; kk < pl.n_kv / 16; ++kk)  // O += P V, K-dim = keys
          ptx::mma_ts(tmem + kColO, tmem + kColS + kk * 8,
                      ptx::make_sdesc(v_addr + kk * 16 * S::kRowBytes, 128 * S::kRowBytes, kSbo, kSw),
                      idesc_o, (j > 0 || kk > 0) ? 1u : 0u);
        ptx::mma_commit(bar_e + s);  // K/V stage s free once these MMAs finish
      }
      ptx::mma_commit(bar_o);
    }
  } else {
    // ===================== softmax / epilogue (128 threads) =====================
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t trow = tmem + ((uint32_t)(quarter * 32) << 16);
    RowCtx<RANK> r;
    r.init(g, pl, t, row);
    const float sl2 = g.scale_log2;
    float m_ref = -INFINITY, l = 0.f;
    for (int j = 0; j < nchunks; ++j) {
      uint32_t mw[4];
      int org[3];
      t.chunk_origin(pl, j, org);
      r.chunk_mask(pl, org, mw);
      ptx::mbar_wait(bar_s, j & 1);
      ptx::tc_fence_after();
      uint32_t sv[128];
      NA_TMEM_LD32(trow + kColS + 0, (sv + 0));
      NA_TMEM_LD32(trow + kColS + 32, (sv + 32));
      NA_TMEM_LD32(trow + kColS + 64, (sv + 64));
      NA_TMEM_LD32(trow + kColS + 96, (sv + 96));
      ptx::tmem_ld_wait();
      float mx = -INFINITY;
#pragma unroll
      for (int c = 0; c < 128; ++c) {
        const float f = (mw[c >> 5] >> (c & 31)) & 1u ? __uint_as_float(sv[c]) * sl2 : -INFINITY;
        sv[c] = __float_as_uint(f);
        mx = fmaxf(mx, f);
      }
      // lazy rescaling: move the reference max only when it grows by > 8
      // (factor 256); P stays <= 2^8, exact after the final normalization.
      const bool need = mx > m_ref + 8.f;
      if (__any_sync(0xffffffffu, need && m_ref != -INFINITY && j > 0)) {
        const float f = need && m_ref != -INFINITY ? ptx::ex2(m_ref - mx) : 1.f;
#pragma unroll
        for (int c0 = 0; c0 < D; c0 += 32) {
          uint32_t ov[32];
          NA_TMEM_LD32(trow + kColO + c0, ov);
          ptx::tmem_ld_wait();
#pragma unroll
          for (int c = 0; c < 32; ++c) ov[c] = __float_as_uint(__uint_as_float(ov[c]) * f);
          NA_TMEM_ST32(trow + kColO + c0, ov);
        }
        l *= f;
      } else if (need) {
        l *= m_ref != -INFINITY ? ptx::ex2(m_ref - mx) : 0.f;
      }
      if (need) m_ref = mx;
      const float mu = m_ref == -INFINITY ? 0.f : m_ref;
      float sum = 0.f;
#pragma unroll
      for (int c = 0; c < 128; c += 2) {
        const float p0 = ptx::ex2(__uint_as_float(sv[c]) - mu);
        const float p1 = ptx::ex2(__uint_as_float(sv[c + 1]) - mu);
        sum += p0 + p1;
        sv[c >> 1] = pack2<BF16>(p0, p1);
      }
      l += sum;
      NA_TMEM_ST32(trow + kColS + 0, (sv + 0));
      NA_TMEM_ST32(trow + kColS + 32, (sv + 32));
      ptx::tmem_st_wait();
      ptx::tc_fence_before();
      ptx::mbar_arrive(bar_p);
    }
    // ---- epilogue: O / l, LSE ----
    ptx::mbar_wait(bar_o, 0);
    ptx::tc_fence_after();
    const float inv = l > 0.f ? 1.f / l : 0.f;
    T* orow = reinterpret_cast<T*>(o_ptr) + r.out_offset(g, t);
#pragma unroll
    for (int c0 = 0; c0 < D; c0 += 32) {
      uint32_t ov[32];
      NA_TMEM_LD32(trow + kColO + c0, ov);
      ptx::tmem_ld_wait();
      if (r.valid) {
        uint32_t pk[16];
#pragma unroll
        for (int c = 0; c < 32; c += 2)
          pk[c >> 1] = pack2<BF16>(__uint_as_float(ov[c]) * inv, __uint_as_float(ov[c + 1]) * inv);
        uint4* dst = reinterpret_cast<uint4*>(orow + c0);
#pragma unroll
        for (int c = 0; c < 4; ++c) dst[c] = make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
      }
    }
    if (lse && r.valid) lse[r.out_offset(g, t) / g.D] = (m_ref + __log2f(l)) * 0.69314718055994531f;
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<256>(tmem);
  }
}

template <int RANK, int D, bool BF16>
cudaError_t launch(const Geom& g, const TcPlan& pl, const CUtensorMap& mq, const CUtensorMap& mk,
                   const CUtensorMap& mv, void* o, float* lse, cudaStream_t st) {
  auto kern = fna_fwd_tc<RANK, D, BF16>;
  const int smem = FwdSmem<D>::kBytes + 1024;
  static bool attr = false;  // benign race: idempotent
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const long long grid = (long long)g.BH * pl.nres * pl.tiles;
  if (grid > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
  prof_begin(KID_FWD_TC, st);
  kern<<<(unsigned)grid, kThreads, smem, st>>>(mq, mk, mv, g, pl, o, lse);
  prof_end(st);
  return cudaGetLastError();
}

template <int RANK>
cudaError_t by_type(int dtype, const Geom& g, const TcPlan& pl, const CUtensorMap& mq,
                    const CUtensorMap& mk, const CUtensorMap& mv, void* o, float* lse,
                    cudaStream_t st) {
  const bool bf = dtype == 2;
  if (g.D == 64) return bf ? launch<RANK, 64, true>(g, pl, mq, mk, mv, o, lse, st)
                           : launch<RANK, 64, false>(g, pl, mq, mk, mv, o, lse, st);
  return bf ? launch<RANK, 32, true>(g, pl, mq, mk, mv, o, lse, st)
            : launch<RANK, 32, false>(g, pl, mq, mk, mv, o, lse, st);
}

}  // namespace

cudaError_t tc_fwd(int dtype, const Geom& g, const void* q, const void* k, const void* v, void* o,
                   float* lse, cudaStream_t st, int* launches) {
  const char* why;
  if (!tc_supported(dtype, g, &why)) return cudaErrorNotSupported;
  TcPlan pl = make_plan(g, /*q_tile_rows=*/128);
  CUtensorMap mq, mk, mv;
  cudaError_t e;
  if ((e = make_map(&mq, dtype, g, q, pl.tq, pl.q_box_x)) != cudaSuccess) return e;
  if ((e = make_map(&mk, dtype, g, k, pl.ckv, pl.kv_box_x)) != cudaSuccess) return e;
  if ((e = make_map(&mv, dtype, g, v, pl.ckv, pl.kv_box_x)) != cudaSuccess) return e;
  *launches = 1;
  switch (g.rank) {
    case 1: return by_type<1>(dtype, g, pl, mq, mk, mv, o, lse, st);
    case 2: return by_type<2>(dtype, g, pl, mq, mk, mv, o, lse, st);
    default: return by_type<3>(dtype, g, pl, mq, mk, mv, o, lse, st);
  }
}

}  // namespace na
