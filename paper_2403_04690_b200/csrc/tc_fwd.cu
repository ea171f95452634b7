// tc_fwd.cu — fused neighborhood attention forward on sm_100a tensor cores.
//
// One CTA handles 128-query multi-dimensional tiles, each of one residue
// class of one (b, h) (§3.3 fused NA, Fig. 4; dilation as extra
// tiles P:329-331).  Persistent: 2 CTAs per SM walk the tile list
// blockIdx.x, blockIdx.x + gridDim.x, ...  Warp roles (256 threads = two
// warpgroups; the single-lane roles take the highest warp ids, which the
// scheduler favours; warpgroup 1 hands most of its registers to warpgroup 0
// with setmaxnreg):
//   warps 0..3  softmax + epilogue: thread = query row = TMEM lane; the
//               epilogue stages O in the tile's (dead) Q buffer and thread 0
//               writes it with a TMA bulk-tensor store.
//   warp 6      TMA producer: Q box per tile (double-buffered), then K and V
//               boxes of every KV chunk of the tile's halo (2-stage rings; a
//               K stage is released as soon as its S MMA is done, a V stage
//               after its PV MMA).
//   warp 7      TMEM owner + MMA issuer (whole warp, one elected lane).
// Each KV chunk (<= 128 keys, one TMA box) is one softmax round: one
// S = Q K^T MMA of N = n_kv (<= 128) columns into the TMEM S buffer; the
// softmax warps load it and release the buffer at once (B_SF), so the next
// round's S MMA runs under this round's exponentials; P goes to its own TMEM
// buffer, then O += P V.  MMA issue order:
//   S_0, [SF_0] S_1, [P_0] PV_0, [SF_1] S_2, [P_1] PV_1, ...
// The softmax warps wait for PV_{kv-1} (B_PF) only before overwriting P or
// rescaling O, i.e. never in steady state: they run back to back, the
// tensor core fills the gaps, and the second CTA on the SM shares the pipes.
// O is single-buffered: the next tile's PV_0 needs that tile's P_0, which the
// softmax warps write only after their epilogue has read O.
// Softmax per round (the whole round's logits of a row in registers):
// tcgen05.ld the row's logits, neighborhood mask (per-row window bitmask)
// applied only to 32-column groups that are partially valid for the warp,
// groups with no valid key skipped, online softmax in the log2 domain with
// lazy O rescaling, P written back to TMEM as 16-bit (A operand
// of PV).  The exponentials are split between the MUFU unit (ex2.approx) and
// a Cody-Waite polynomial on the FMA pipe (packed FFMA2), since MUFU
// throughput bounds this kernel.  Only chunks of the tile's halo box
// [start(q_lo), end(q_hi)] are visited.
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

constexpr int kMaxStages = 2;  // K/V ring depth bound (barrier slots); FwdSmem<D>::kStages is the depth
constexpr int kThreads = 256;
constexpr int kSoftmax = 128;    // softmax threads (warps 0..3)
// The warp scheduler favours the highest warp id among eligible warps, so the
// latency-critical single-lane roles take the highest ids.
constexpr int kProducerWarp = 6;
constexpr int kMmaWarp = 7;
// Registers after setmaxnreg: warpgroup 1 (producer, MMA, two idle warps)
// gives its share to the softmax warpgroup, which holds a whole 128-column
// round of logits in registers.  128 * (kRegsSoftmax + kRegsOther) = the
// 2-CTA/SM budget of 256 threads x 128.
constexpr uint32_t kRegsSoftmax = 200;
constexpr uint32_t kRegsOther = 56;
// Small-tile variant (SMALL: head_dim <= 32 and KV chunks of <= 64 keys,
// e.g. 2-D 56x56 k=7 with dilation 8, one 7x7 class per tile): a tile is
// one or two short rounds, so per-tile latency dominates and more tiles
// must be in flight per SM.  S 64 + P 32 + O 32 TMEM columns -> 128 per
// CTA, 3 CTAs per SM; registers 3 x 256 x 80 = 61440 split 120 / 40.
// (4 CTAs per SM would leave 96 / 32 registers: ~650 bytes of spills.)
constexpr uint32_t kRegsSoftmaxSmall = 120;
constexpr uint32_t kRegsOtherSmall = 40;
// TMEM columns (256 per CTA, two CTAs per SM): S [0, 128) fp32 logits of the
// current round; P [128, 192) the previous round's probabilities as packed
// 16-bit pairs (A operand of PV); O [192, 192 + D) the fp32 accumulator.
constexpr uint32_t kColS = 0, kColP = 128, kColO = 192;
constexpr uint32_t kColPSmall = 64, kColOSmall = 96;
// head_dim 128 (KV chunks <= 64 keys): S [0, 64), P [64, 96), O [128, 256).
template <bool SMALL, bool WIDE = false>
struct FwdCfg {
  static constexpr int kCtas = SMALL ? 3 : 2;            // CTAs per SM
  static constexpr uint32_t kTmemCols = SMALL ? 128 : 256;
  static constexpr uint32_t kColP_ = SMALL ? kColPSmall : WIDE ? 64 : kColP;
  static constexpr uint32_t kColO_ = SMALL ? kColOSmall : WIDE ? 128 : kColO;
  static constexpr int kGroups = (SMALL || WIDE) ? 2 : 4;  // 32-column groups of a round
  static constexpr uint32_t kRegsS = SMALL ? kRegsSoftmaxSmall : kRegsSoftmax;
  static constexpr uint32_t kRegsO = SMALL ? kRegsOtherSmall : kRegsOther;
};

// head_dim 128 ("wide"): a 256-byte row exceeds the 128-byte swizzle span,
// so every tile is stored as two 64-column halves [half][rows][128 B], each
// a SW128 operand (TMA loads / stores one half per issue, c0 = 0 / 64); the
// S MMA's K-steps 4..7 read the second halves, and V (the MN-major B of PV)
// has its two 64-column atoms LBO = one half apart.  KV chunks hold <= 64
// keys (planner) and the ring has one stage, so Q x 2 + K + V = 96 KB and
// two CTAs still fit an SM.
template <int D>
struct FwdSmem {
  static constexpr bool kWide = D > 64;
  static constexpr int kHalves = kWide ? 2 : 1;
  static constexpr int kRowBytes = (kWide ? 64 : D) * 2;  // one swizzled row (of one half)
  static constexpr int kKvRows = kWide ? 64 : 128;        // K / V rows per stage
  static constexpr int kStages = kWide ? 1 : 2;           // K / V ring depth
  static constexpr int kQHalf = 128 * kRowBytes;
  static constexpr int kTile = kHalves * kQHalf;          // Q tile (also the O staging tile)
  static constexpr int kKvHalf = kKvRows * kRowBytes;
  static constexpr int kKvTile = kHalves * kKvHalf;       // one K or V stage
  static constexpr int kQ = 0;                            // [2] (double-buffered across tiles)
  static constexpr int kK = kQ + 2 * kTile;
  static constexpr int kV = kK + kStages * kKvTile;
  static constexpr int kBar = kV + kStages * kKvTile;
  static constexpr int kBytes = kBar + 256;
};

// Barrier slots.
enum : int {
  B_QF = 0,                 // Q buffer full [2]
  B_QE = B_QF + 2,          // Q buffer empty [2]
  B_K = B_QE + 2,           // K stage full [kMaxStages]
  B_V = B_K + kMaxStages,      // V stage full [kMaxStages]
  B_KE = B_V + kMaxStages,     // K stage free (its S MMA is done) [kMaxStages]
  B_VE = B_KE + kMaxStages,    // V stage free (its PV MMA is done) [kMaxStages]
  B_S = B_VE + kMaxStages,     // S of a round ready
  B_SF = B_S + 1,           // S loaded by the softmax warps: buffer free (128 arrivals)
  B_P = B_SF + 1,           // P of a round written (128 arrivals)
  B_PF = B_P + 1,           // PV of a round done: P buffer free, O stable
  B_OF = B_PF + 1,          // O of a tile final
  B_COUNT = B_OF + 1
};

// Tensor maps: Q tiles, K and V chunks, and O tiles (TMA store, Q's box).
struct FwdMaps {
  CUtensorMap q, k, v, o;
};

// PRECISE (bf16 only, bf16_precise()): O normalised by the sum of the
// bf16-rounded P (R13).
template <int RANK, int D, bool BF16, bool PRECISE, bool SMALL>
__global__ void __launch_bounds__(kThreads, FwdCfg<SMALL>::kCtas)
    fna_fwd_tc(const __grid_constant__ FwdMaps maps, Geom g, TcPlan pl, float* __restrict__ lse,
               unsigned num_tiles) {
  const CUtensorMap& map_q = maps.q;
  const CUtensorMap& map_k = maps.k;
  const CUtensorMap& map_v = maps.v;
  const CUtensorMap& map_o = maps.o;
  using S = FwdSmem<D>;
  constexpr bool kSumRounded = BF16 && PRECISE;
  using C = FwdCfg<SMALL, (D > 64)>;
  constexpr int kStages = S::kStages;
  constexpr uint32_t kColP = C::kColP_, kColO = C::kColO_;
  constexpr int kG = C::kGroups;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte aligned by pointer arithmetic on the __shared__ array, so the
  // compiler keeps the shared address space (LDS/STS, not generic LD/ST).
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + S::kBar);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + B_COUNT);

  const uint32_t warp = ptx::warp_id(), lane = ptx::lane_id();
  if (threadIdx.x == 0) {
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(bar + B_QF + b, 1);
      ptx::mbar_init(bar + B_QE + b, 1);
    }
    ptx::mbar_init(bar + B_OF, 1);
    ptx::mbar_init(bar + B_SF, kSoftmax);
    ptx::mbar_init(bar + B_PF, 1);
    for (int s = 0; s < kMaxStages; ++s) {
      ptx::mbar_init(bar + B_K + s, 1);
      ptx::mbar_init(bar + B_V + s, 1);
      ptx::mbar_init(bar + B_KE + s, 1);
      ptx::mbar_init(bar + B_VE + s, 1);
    }
    ptx::mbar_init(bar + B_S, 1);
    ptx::mbar_init(bar + B_P, kSoftmax);
    ptx::fence_barrier_init();
  }
  // Zero the K/V rows no TMA box writes (rows_kv..127): the MMA reads up to
  // n_kv rows and 0 * garbage could be NaN.
  if (pl.rows_kv < S::kKvRows) {
    const int nz = (S::kKvRows - pl.rows_kv) * S::kRowBytes / 16;
    for (int i = threadIdx.x; i < 2 * kStages * S::kHalves * nz; i += kThreads) {
      const int buf = i / nz, off = i % nz;  // buf = (K or V stage) x half
      uint4* base = reinterpret_cast<uint4*>(smem + S::kK + buf * S::kKvHalf + pl.rows_kv * S::kRowBytes);
      base[off] = make_uint4(0, 0, 0, 0);
    }
    ptx::fence_proxy_async();
  }
  if (warp == kMmaWarp) ptx::tmem_alloc<C::kTmemCols>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp >= 4) {
  ptx::setmaxnreg_dec<C::kRegsO>();
  if (warp == kProducerWarp) {
    // ===================== TMA producer (whole warp, one lane issues) =====================
    ptx::tma_prefetch(&map_q);
    ptx::tma_prefetch(&map_k);
    ptx::tma_prefetch(&map_v);
    const uint32_t kv_bytes = pl.rows_kv * S::kRowBytes * S::kHalves;
    uint32_t kv_it = 0, ti = 0;
    int tr = 0;
    for (unsigned tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      TileCtx<RANK> t;
      if (!t.init(g, pl, tile)) continue;
      const int qb = ti & 1;
      if (ti >= 2) ptx::mbar_wait(bar + B_QE + qb, ((ti >> 1) - 1) & 1);
      ptx::mbar_expect_tx_w(bar + B_QF + qb, S::kTile);
      for (int h = 0; h < S::kHalves; ++h)
        for (int i = 0; i < pl.q_issues; ++i)
          t.template load_box<RANK>(&map_q, smem + S::kQ + qb * S::kTile + h * S::kQHalf + i * pl.q_box_x * S::kRowBytes,
                                    bar + B_QF + qb, t.q_origin, i * pl.q_box_x, g, 64 * h);
      int org[3] = {t.lo[0], t.lo[1], t.lo[2]};
      for (int j = 0; j < t.nchunks; ++j, ++kv_it, t.next_origin(pl, org)) {
        const int s = kv_it % kStages;
        const uint32_t ph = ((kv_it / kStages) - 1) & 1;
        uint8_t* kd = smem + S::kK + s * S::kKvTile;
        uint8_t* vd = smem + S::kV + s * S::kKvTile;
        if (kv_it >= kStages) ptx::mbar_wait(bar + B_KE + s, ph);
        ptx::mbar_expect_tx_w(bar + B_K + s, kv_bytes);
        for (int h = 0; h < S::kHalves; ++h)
          for (int i = 0; i < pl.kv_issues; ++i)
            t.template load_box<RANK>(&map_k, kd + h * S::kKvHalf + i * pl.kv_box_x * S::kRowBytes, bar + B_K + s,
                                      org, i * pl.kv_box_x, g, 64 * h);
        if (kv_it >= kStages) ptx::mbar_wait(bar + B_VE + s, ph);
        ptx::mbar_expect_tx_w(bar + B_V + s, kv_bytes);
        for (int h = 0; h < S::kHalves; ++h)
          for (int i = 0; i < pl.kv_issues; ++i)
            t.template load_box<RANK>(&map_v, vd + h * S::kKvHalf + i * pl.kv_box_x * S::kRowBytes, bar + B_V + s,
                                      org, i * pl.kv_box_x, g, 64 * h);
        NA_TRACE_EV(0, tr, 1);
      }
      ++ti;
    }
  } else if (warp == kMmaWarp) {
    // ===================== MMA issuer (whole warp, one elected lane) =====================
    // Issue order S_0, [SF_0] S_1, [P_0] PV_0, [SF_1] S_2, [P_1] PV_1, ...:
    // S_{kv+1} starts as soon as the softmax warps have LOADED S_kv, so it
    // overlaps their exponentials; PV_kv reads P from its own buffer.
    constexpr uint32_t kSw = ptx::sw_layout(D);  // SW128 / SW64 / SW32
    constexpr uint32_t kSbo = 8 * S::kRowBytes;  // 8-row core-matrix group
    const uint32_t idesc_s = ptx::make_idesc(128, pl.n_kv, BF16, false);
    constexpr uint32_t idesc_o = ptx::make_idesc(128, D, BF16, true);
    const int kblocks = pl.n_kv / 16;
    int tr = 0;
    // S = Q K_kv^T (K-dim = head_dim); kv = global chunk index
    auto issue_s = [&](uint32_t kv, uint32_t q_addr) {
      const int s = kv % kStages;
      ptx::mbar_wait(bar + B_K + s, (kv / kStages) & 1);
      ptx::tc_fence_after();
      NA_TRACE_EV(1, tr, 10);
      const uint32_t k_addr = ptx::smem_u32(smem + S::kK + s * S::kKvTile);
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {  // K-steps 4..7 (head_dim 128): second halves
        const uint32_t hq = (kk >> 2) * S::kQHalf, hk = (kk >> 2) * S::kKvHalf, ko = (kk & 3) * 32;
        ptx::mma_ss_w(tmem + kColS, ptx::make_sdesc(q_addr + hq + ko, 16, kSbo, kSw),
                      ptx::make_sdesc(k_addr + hk + ko, 16, kSbo, kSw), idesc_s, kk > 0);
      }
      ptx::mma_commit_w(bar + B_S);
      ptx::mma_commit_w(bar + B_KE + s);
    };
    auto q_addr_of = [&](uint32_t ti) { return ptx::smem_u32(smem + S::kQ + (ti & 1) * S::kTile); };
    TileCtx<RANK> t;
    unsigned tile = seek_tile<RANK, false>(g, pl, blockIdx.x, num_tiles, t);
    uint32_t kv = 0, ti = 0;
    if (tile < num_tiles) {
      ptx::mbar_wait(bar + B_QF + 0, 0);
      issue_s(0, q_addr_of(0));
    }
    while (tile < num_tiles) {
      const int nch = t.nchunks;
      TileCtx<RANK> tn;
      unsigned tile_n = num_tiles;
      for (int j = 0; j < nch; ++j, ++kv) {
        const int s = kv % kStages;
        // next S as soon as the softmax warps have read this one
        ptx::mbar_wait(bar + B_SF, kv & 1);
        if (j + 1 < nch) {
          issue_s(kv + 1, q_addr_of(ti));
        } else {
          tile_n = seek_tile<RANK, false>(g, pl, tile + gridDim.x, num_tiles, tn);
          if (tile_n < num_tiles) {  // first S of the next tile
            ptx::mbar_wait(bar + B_QF + ((ti + 1) & 1), ((ti + 1) >> 1) & 1);
            issue_s(kv + 1, q_addr_of(ti + 1));
          }
        }
        ptx::mbar_wait(bar + B_P, kv & 1);  // softmax wrote P_kv (and rescaled O)
        NA_TRACE_EV(1, tr, 11);
        ptx::mbar_wait(bar + B_V + s, (kv / kStages) & 1);
        ptx::tc_fence_after();
        const uint32_t v_addr = ptx::smem_u32(smem + S::kV + s * S::kKvTile);
        for (int kk = 0; kk < kblocks; ++kk)  // O += P V, K-dim = keys
          ptx::mma_ts_w(tmem + kColO, tmem + kColP + kk * 8,
                        ptx::make_sdesc(v_addr + kk * 16 * S::kRowBytes, S::kKvHalf, kSbo, kSw),
                        idesc_o, (j > 0 || kk > 0) ? 1u : 0u);
        ptx::mma_commit_w(bar + B_VE + s);  // V stage free after these MMAs
        ptx::mma_commit_w(bar + B_PF);      // P buffer free, O stable
        if (j == nch - 1) ptx::mma_commit_w(bar + B_OF);
        NA_TRACE_EV(1, tr, 12);
      }
      tile = tile_n;
      t = tn;
      ++ti;
    }
  }
  } else {
    ptx::setmaxnreg_inc<C::kRegsS>();
    // ===================== softmax / epilogue (128 threads) =====================
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t trow = tmem + ((uint32_t)(quarter * 32) << 16);
    const float sl2 = g.scale_log2;
    const bool wide = !SMALL && pl.n_kv > 64;  // P needs TMEM columns [32, 64) too
    uint32_t kv = 0, ti = 0;
    int tr = 0;
    const bool tracer = warp == 2;
    for (unsigned tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      TileCtx<RANK> t;
      if (!t.init(g, pl, tile)) continue;
      RowCtx<RANK> r;
      r.init(g, pl, t, row);
      // l: sum of the fp32 probabilities (-> LSE); lr (bf16 only): sum of the
      // values the PV MMA actually multiplies, bf16(P) -> O normalisation
      // (R13).
      float m_ref = -INFINITY, l = 0.f, lr = 0.f;
      int org[3] = {t.lo[0], t.lo[1], t.lo[2]};  // chunk origin (odometer)
      uint32_t mw[4];                             // this row's mask of the chunk
      r.chunk_mask(pl, org, mw);
      for (int j = 0; j < t.nchunks; ++j, ++kv) {
        // warp-uniform group flags before the wait (they depend on the mask only)
        bool live[kG], full[kG];
#pragma unroll
        for (int gq = 0; gq < kG; ++gq) {
          live[gq] = __any_sync(0xffffffffu, mw[gq] != 0u);
          full[gq] = __all_sync(0xffffffffu, mw[gq] == 0xffffffffu);
        }
        ptx::mbar_wait(bar + B_S, kv & 1);
        ptx::tc_fence_after();
        if (tracer) NA_TRACE_EV(2, tr, 20);
        // The whole round (<= 128 logits of this row) in registers: one
        // tcgen05.wait for all loads, independent chains across the groups.
        uint32_t sv[32 * kG];
#pragma unroll
        for (int gq = 0; gq < kG; ++gq)
          if (live[gq]) NA_TMEM_LD32(trow + kColS + 32 * gq, (sv + 32 * gq));
        // the next chunk's mask, in the shadow of the TMEM load latency
        uint32_t mwn[4] = {0u, 0u, 0u, 0u};
        if (j + 1 < t.nchunks) {
          t.next_origin(pl, org);
          r.chunk_mask(pl, org, mwn);
        }
        ptx::tmem_ld_wait();
        if (tracer) NA_TRACE_EV(2, tr, 24);
        ptx::tc_fence_before();
        ptx::mbar_arrive(bar + B_SF);  // S buffer free: the next S MMA overlaps this round
        // mask (only partially valid groups) and row max of the raw logits
        float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
        for (int gq = 0; gq < kG; ++gq) {
          if (!live[gq]) continue;
          const uint32_t w = mw[gq];
          if (!full[gq]) {
#pragma unroll
            for (int c = 0; c < 32; ++c)
              sv[32 * gq + c] = (w >> c) & 1u ? sv[32 * gq + c] : __float_as_uint(-INFINITY);
          }
#pragma unroll
          for (int c = 0; c < 32; c += 8)  // independent partial maxima: short chains
#pragma unroll
            for (int i = 0; i < 4; ++i)
              m4[i] = fmaxf(m4[i], fmaxf(__uint_as_float(sv[32 * gq + c + i]),
                                         __uint_as_float(sv[32 * gq + c + 4 + i])));
        }
        const float mx = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
        if (tracer) NA_TRACE_EV(2, tr, 25);
        const float mx2 = mx * sl2;  // log2-domain max (-inf stays -inf)
        // lazy rescaling: move the reference max only when it grows by > 8
        // (factor 256); P stays <= 2^8 and the result is exact after the
        // final normalisation.
        const bool need = mx2 > m_ref + 8.f;
        if (__any_sync(0xffffffffu, need && m_ref != -INFINITY)) {
          if (kv > 0) ptx::mbar_wait(bar + B_PF, (kv - 1) & 1);  // O holds PV_{kv-1}
          ptx::tc_fence_after();
          const float f = need && m_ref != -INFINITY ? ptx::ex2(m_ref - mx2) : 1.f;
#pragma unroll 1
          for (int c0 = 0; c0 < D; c0 += 16) {
            uint32_t ov[16];
            NA_TMEM_LD16(trow + kColO + c0, ov);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int c = 0; c < 16; ++c) ov[c] = __float_as_uint(__uint_as_float(ov[c]) * f);
            NA_TMEM_ST16(trow + kColO + c0, ov);
          }
          l *= f;
          if constexpr (kSumRounded) lr *= f;
        } else if (need) {
          l = 0.f;  // no valid key seen yet on this row
          lr = 0.f;
        }
        if (need) m_ref = mx2;
        const float nmu = m_ref == -INFINITY ? 0.f : -m_ref;
        float2 acc0 = make_float2(0.f, 0.f), acc1 = make_float2(0.f, 0.f);
        float2 accr0 = make_float2(0.f, 0.f), accr1 = make_float2(0.f, 0.f);
        // exponentials; P packed as 16-bit pairs IN PLACE: the pair of
        // columns (2i, 2i+1) goes to sv[i], whose logit was already consumed
#pragma unroll
        for (int gq = 0; gq < kG; ++gq) {
          if (!live[gq]) {
#pragma unroll
            for (int c = 0; c < 16; ++c) sv[16 * gq + c] = 0u;
            continue;
          }
#pragma unroll
          for (int c = 0; c < 32; c += 4) {
            const uint32_t* s4 = sv + 32 * gq + c;
            const float2 x0 = __ffma2_rn(make_float2(__uint_as_float(s4[0]), __uint_as_float(s4[1])),
                                         make_float2(sl2, sl2), make_float2(nmu, nmu));
            const float2 x1 = __ffma2_rn(make_float2(__uint_as_float(s4[2]), __uint_as_float(s4[3])),
                                         make_float2(sl2, sl2), make_float2(nmu, nmu));
            const float2 p0 = make_float2(ptx::ex2(x0.x), ptx::ex2(x0.y));  // MUFU
            const float2 p1 = use_poly<RANK == 1 ? 1 : 0>(c) ? exp2_poly2(x1)                   // FMA pipe
                                          : make_float2(ptx::ex2(x1.x), ptx::ex2(x1.y));
            acc0 = __fadd2_rn(acc0, p0);
            acc1 = __fadd2_rn(acc1, p1);
            sv[16 * gq + (c >> 1)] = pack2<BF16>(p0.x, p0.y);
            sv[16 * gq + (c >> 1) + 1] = pack2<BF16>(p1.x, p1.y);
            if constexpr (kSumRounded) {
              accr0 = add_bf16x2(accr0, sv[16 * gq + (c >> 1)]);
              accr1 = add_bf16x2(accr1, sv[16 * gq + (c >> 1) + 1]);
            }
          }
        }
        l += (acc0.x + acc0.y) + (acc1.x + acc1.y);
        if constexpr (kSumRounded) lr += (accr0.x + accr0.y) + (accr1.x + accr1.y);
        if (tracer) NA_TRACE_EV(2, tr, 26);
        // P into its buffer once PV_{kv-1} has read the previous P
        if (kv > 0) ptx::mbar_wait(bar + B_PF, (kv - 1) & 1);
        if (tracer) NA_TRACE_EV(2, tr, 27);
        ptx::tc_fence_after();
        NA_TMEM_ST32(trow + kColP, sv);
        if (wide) NA_TMEM_ST32(trow + kColP + 32, (sv + 32));
        ptx::tmem_st_wait();
        ptx::tc_fence_before();
        ptx::mbar_arrive(bar + B_P);
        if (tracer) NA_TRACE_EV(2, tr, 21);
#pragma unroll
        for (int i = 0; i < 4; ++i) mw[i] = mwn[i];
      }
      // ---- epilogue: O / l, LSE (overlaps the next tile's S MMAs) ----
      // All MMAs of the tile are complete once O is final, so the tile's Q
      // buffer is dead: stage the normalised O there (TMA box layout, same
      // swizzle) and write it with one TMA store, which also clips rows past
      // a ragged class end.  The buffer returns to the producer (B_QE) once
      // the store has read it.
      ptx::mbar_wait(bar + B_OF, ti & 1);
      ptx::tc_fence_after();
      if (tracer) NA_TRACE_EV(2, tr, 22);
      // bf16 (PRECISE): O = sum bf16(P) v / sum bf16(P), a convex
      // combination of the v's, so the 2^-9 rounding of P does not scale O
      // (exact when one key dominates); fp16 P is 8x finer and uses l.
      const float lo = kSumRounded ? lr : l;
      const float inv = lo > 0.f ? 1.f / lo : 0.f;
      const int qb = ti & 1;
      uint8_t* stage = smem + S::kQ + qb * S::kTile;
#pragma unroll
      constexpr int kEc = D < 32 ? 16 : 32;  // O columns per TMEM load
      for (int c0 = 0; c0 < D; c0 += kEc) {
        uint32_t ov[kEc];
        if constexpr (kEc == 32) NA_TMEM_LD32(trow + kColO + c0, ov);
        else NA_TMEM_LD16(trow + kColO + c0, ov);
        ptx::tmem_ld_wait();
#pragma unroll
        for (int c = 0; c < kEc; c += 8)
          *reinterpret_cast<uint4*>(stage + ((c0 + c) / 64) * S::kQHalf +
                                    ptx::swz_off(row, ((c0 + c) / 8) & 7, S::kRowBytes)) =
              make_uint4(pack2<BF16>(__uint_as_float(ov[c]) * inv, __uint_as_float(ov[c + 1]) * inv),
                         pack2<BF16>(__uint_as_float(ov[c + 2]) * inv, __uint_as_float(ov[c + 3]) * inv),
                         pack2<BF16>(__uint_as_float(ov[c + 4]) * inv, __uint_as_float(ov[c + 5]) * inv),
                         pack2<BF16>(__uint_as_float(ov[c + 6]) * inv, __uint_as_float(ov[c + 7]) * inv));
      }
      ptx::tc_fence_before();
      // O is free again once every thread's loads are done: the next tile's
      // PV_0 needs P_0, which these threads write after this point.
      if (tracer) NA_TRACE_EV(2, tr, 23);
      ptx::fence_proxy_async();           // staged O visible to the TMA engine
      ptx::named_bar_sync(1, kSoftmax);
      if (threadIdx.x == 0) {
        for (int h = 0; h < S::kHalves; ++h)
          for (int i = 0; i < pl.q_issues; ++i)
            t.template store_box<RANK>(&map_o, stage + h * S::kQHalf + i * pl.q_box_x * S::kRowBytes, i * pl.q_box_x,
                                       g, 64 * h);
        ptx::bulk_commit();
        ptx::bulk_wait_read<0>();
        ptx::mbar_arrive(bar + B_QE + qb);  // Q buffer reusable
      }
      if (lse && r.valid) lse[r.token_index(g, t)] = (m_ref + __log2f(l)) * 0.69314718055994531f;
      ++ti;
    }
    if (threadIdx.x == 0) ptx::bulk_wait<0>();  // all O stores complete before exit
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<C::kTmemCols>(tmem);
  }
}

template <int RANK, int D, bool BF16, bool PRECISE, bool SMALL>
cudaError_t launch_v(const Geom& g, const TcPlan& pl, const FwdMaps& maps, float* lse, cudaStream_t st) {
  auto kern = fna_fwd_tc<RANK, D, BF16, PRECISE, SMALL>;
  const int smem = FwdSmem<D>::kBytes + 1024;
  if constexpr (D > 64) {
    if (pl.n_kv > FwdSmem<D>::kKvRows) return cudaErrorInvalidConfiguration;  // planner bound
  }
  cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kern), smem);
  if (e != cudaSuccess) return e;
  const long long tiles = (long long)g.BH * pl.nres * pl.tiles;
  if (tiles > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
  const long long per = FwdCfg<SMALL>::kCtas;  // CTAs per SM (TMEM columns each: kTmemCols)
  const unsigned grid = (unsigned)(tiles < per * num_sms() ? tiles : per * num_sms());
  prof_begin(KID_FWD_TC, st);
  kern<<<grid, kThreads, smem, st>>>(maps, g, pl, lse, (unsigned)tiles);
  prof_end(st);
  return cudaGetLastError();
}

// The small-tile variant needs S 64 + P 32 + O <= 32 TMEM columns.
template <int RANK, int D, bool BF16, bool PRECISE = false>
cudaError_t launch(const Geom& g, const TcPlan& pl, const FwdMaps& maps, float* lse, cudaStream_t st) {
  if constexpr (D <= 32) {
    if (pl.n_kv <= 64) return launch_v<RANK, D, BF16, PRECISE, true>(g, pl, maps, lse, st);
  }
  return launch_v<RANK, D, BF16, PRECISE, false>(g, pl, maps, lse, st);
}

template <int RANK>
cudaError_t by_type(int dtype, const Geom& g, const TcPlan& pl, const FwdMaps& maps, float* lse,
                    cudaStream_t st) {
  if (dtype == 2) {
    const bool pr = bf16_precise(g);
    if (g.D == 128) return pr ? launch<RANK, 128, true, true>(g, pl, maps, lse, st)
                              : launch<RANK, 128, true>(g, pl, maps, lse, st);
    if (g.D == 64) return pr ? launch<RANK, 64, true, true>(g, pl, maps, lse, st)
                             : launch<RANK, 64, true>(g, pl, maps, lse, st);
    if (g.D == 16) return pr ? launch<RANK, 16, true, true>(g, pl, maps, lse, st)
                             : launch<RANK, 16, true>(g, pl, maps, lse, st);
    return pr ? launch<RANK, 32, true, true>(g, pl, maps, lse, st) : launch<RANK, 32, true>(g, pl, maps, lse, st);
  }
  if (g.D == 128) return launch<RANK, 128, false>(g, pl, maps, lse, st);
  if (g.D == 64) return launch<RANK, 64, false>(g, pl, maps, lse, st);
  if (g.D == 16) return launch<RANK, 16, false>(g, pl, maps, lse, st);
  return launch<RANK, 32, false>(g, pl, maps, lse, st);
}

}  // namespace

cudaError_t tc_fwd(int dtype, const Geom& g, const Layout& ly, const void* q, const void* k, const void* v, void* o,
                   float* lse, cudaStream_t st, int* launches) {
  const char* why;
  if (!tc_supported(dtype, g, &why)) return cudaErrorNotSupported;
  TcPlan pl = make_plan(g, /*q_tile_rows=*/128, plan_choice(g, dtype).fwd);
  FwdMaps maps;
  cudaError_t e;
  if ((e = make_map(&maps.q, dtype, g, ly, q, pl.tq, pl.q_box_x)) != cudaSuccess) return e;
  if ((e = make_map(&maps.k, dtype, g, ly, k, pl.ckv, pl.kv_box_x)) != cudaSuccess) return e;
  if ((e = make_map(&maps.v, dtype, g, ly, v, pl.ckv, pl.kv_box_x)) != cudaSuccess) return e;
  if ((e = make_map(&maps.o, dtype, g, ly, o, pl.tq, pl.q_box_x)) != cudaSuccess) return e;
  *launches = 1;
  switch (g.rank) {
    case 1: return by_type<1>(dtype, g, pl, maps, lse, st);
    case 2: return by_type<2>(dtype, g, pl, maps, lse, st);
    default: return by_type<3>(dtype, g, pl, maps, lse, st);
  }
}

#ifdef NA_TRACE
// Trace build only (libna_trace.so): point the forward kernel's event buffer.
extern "C" int na_debug_set_trace_fwd(void* p) {
  return cudaMemcpyToSymbol(na::g_trace, &p, sizeof(p)) == cudaSuccess ? 0 : 1;
}
#endif

}  // namespace na
