// tc_bwd.cu — fused neighborhood attention backward on sm_100a tensor cores.
//
// The backward is the paper's operator composition (§3.1) fused
// FlashAttention-style, recomputing the attention weights from the saved LSE
// instead of storing them:
//   dP = PN(dO, V)          dS = P o (dP - D),  D_x = <dO_x, O_x>
//   dQ = scale NN(dS, K)    dK = scale IN(dS, Q)    dV = IN(P, dO)
// Two kernels, each output element has exactly one writer (no atomics):
//   fna_dkdv_tc  key-stationary: a tile = 128 keys of one residue class; it
//                streams the query chunks of the tile's INVERSE halo
//                [inv_start(y_lo), inv_end(y_hi)] (the IN gather pattern,
//                P:253-258).  Per 64-query sub-chunk: S^T = K Q^T and
//                dP^T = V dO^T (SS MMAs), P^T = exp(scale S^T - LSE_q) and
//                dS^T = P^T (dP^T - D_q) by the compute warps (written back to
//                TMEM as 16-bit), then dV += P^T dO and dK += dS^T Q (TS MMAs).
//   fna_dq_tc    query-stationary over the forward halo: S = Q K^T, dP = dO V^T,
//                dS = P (dP - D), dQ += dS K.  For 1-D it also forms the
//                row vectors (-LSE log2 e, D) itself from an O tile loaded
//                with the stationary Q/dO tiles, and writes them for
//                fna_dkdv_tc, which runs after it (the fused preprocess);
//                2-D/3-D read them from the preprocess kernel.
// Persistent, 1 CTA per SM walking tiles blockIdx.x, +gridDim.x, ...
// Warp roles (352 threads): warps 0..7 two compute warpgroups (thread = TMEM
// lane = stationary row); warp 8 TMA producer (stationary tiles double-
// buffered, 4-stage ring of streamed chunks + their row vectors); warp 9
// TMEM owner + OUT-MMA issuer; warp 10 S/dP-MMA issuer (one elected lane
// each).  Sub-chunk gu (64 partner columns) is processed by warpgroup gu%2:
//   S/dP(gu) -> TMEM buffer gu%3; the warpgroup loads it, computes P and dS,
//   writes them packed over the columns it has read (B_P), and the OUT warp
//   issues the accumulating MMAs in order; their completion (B_PE) frees the
//   buffer for S/dP(gu+3).  No warpgroup ever waits for an OUT MMA.
// dK|dV share one 128-column accumulator drained at each tile start by the
// warpgroup not owning the tile's first sub-chunk; dQ's is double-buffered,
// each warpgroup drains half after its first sub-chunk of the next tile, and
// the one finishing second issues the store (ranks 1, 2).
// Outputs are staged in the tile's dead stationary smem and TMA-stored.
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

#ifdef NA_TRACE
static __constant__ int g_trace_sel;  // trace build: 1 = dK/dV kernel, 0 = dQ kernel
#define NA_BWD_TRACE_ON (g_trace_sel == (KV_STATIONARY ? 1 : 0))
#else
#define NA_BWD_TRACE_ON false
#endif

constexpr int kStages = 4;
constexpr int kThreads = 352;
constexpr int kCompute = 256;  // compute threads (warps 0..7)
// The warp scheduler favours the highest warp id among eligible warps, so the
// latency-critical single-lane roles take the highest ids.
constexpr int kProducerWarp = 8;
constexpr int kMmaWarp = 9;    // TMEM owner; OUT MMAs (dV, dK | dQ), in sub-chunk order
constexpr int kSWarp = 10;     // S / dP MMAs, as far ahead as the TMEM buffers allow
constexpr float kLog2e = 1.4426950408889634f;

// Both kernels stream 4 stages; a fused dQ (FUSE: rank 1) holds the O tiles
// it reads to form the row vectors itself (see the dQ compute warps) where
// dK/dV keeps the gathered row vectors of its streamed chunks.
// head_dim 128 ("wide"): every tile is stored as two 64-column SW128 halves
// [half][rows][128 B] (as in the forward); streamed chunks hold <= 64
// partner rows (planner), two stages, so the stationary double buffer
// (128 KB) and the ring (64 KB) fit.
template <int D, bool KV, bool FUSE, bool EXACT = false>
struct BwdSmem {
  static constexpr bool kWide = D > 64;
  static constexpr int kHalves = kWide ? 2 : 1;
  static constexpr int kSt = kWide ? 2 : 4;           // streamed stages
  static constexpr int kRowBytes = (kWide ? 64 : D) * 2;  // one swizzled row (of one half)
  static constexpr int kBRows = kWide ? 64 : 128;     // streamed rows per tile
  static constexpr int kAHalf = 128 * kRowBytes;
  static constexpr int kTile = kHalves * kAHalf;      // stationary tile
  static constexpr int kBHalf = kBRows * kRowBytes;
  static constexpr int kBTile = kHalves * kBHalf;     // streamed tile
  // Stationary buffers: head_dim <= 32 tiles are small (8 KB) and short
  // (C configs: one or two sub-chunks), so four buffers let the producer
  // load a tile's stationary pair three tiles ahead instead of waiting for
  // the store of the tile two back (whose latency was exposed per tile).
  static constexpr int kAB = D <= 32 ? 4 : 2;
  static constexpr int kA = 0;                        // stationary [kAB bufs][2 tiles] (K,V | Q,dO)
  static constexpr int kO = kA + 2 * kAB * kTile;     // fused dQ: stationary O tile [kAB bufs]
  static constexpr int kB0 = kO + (FUSE ? kAB * kTile : 0);  // streamed [kSt] (Q | K)
  static constexpr int kB1 = kB0 + kSt * kBTile;      // streamed [kSt] (dO | V)
  static constexpr int kVec = kB1 + kSt * kBTile;     // [kSt][-LSE2 x128 | D x128] fp32 (dK/dV)
  static constexpr int kBar = kVec + (KV ? kSt * 256 * 4 : 0);
  static constexpr int kDx = kBar + 512;              // (barriers + TMEM slot words) exact-D dQ: [2 groups][128] fp32 partials
  static constexpr int kBytes = kDx + (EXACT ? 2 * 128 * 4 : 0);
};

// TMEM columns (512): three sub-chunk buffers b = gu % 3 at [128b, 128b + 128):
// S at +0 and dP at +64 (64 partner columns each, fp32); the compute warps
// write P^T (dQ: nothing) over S's first 32 columns and dS^T (dQ: dS) over
// dP's, as packed 16-bit pairs, the A operands of the OUT MMAs.  A buffer is
// reused for sub-chunk gu + 3 once gu's OUT MMAs are done (B_PE), so the S/dP
// MMAs run up to three sub-chunks ahead.  [384,512) output accumulators:
// dK | dV (2D columns, single-buffered when 2D = 128) or dQ (D columns,
// double-buffered).
constexpr uint32_t kColOut = 384;
// head_dim 128: two sub-chunk buffers [0, 256), outputs [256, 512) (dK | dV
// = 2 x 128 columns; dQ 128 + the exact-D PK accumulator 128).
template <int D>
struct BwdTmem {
  static constexpr uint32_t kNB = D > 64 ? 2 : 3;  // rotating S/dP sub-chunk buffers
  static constexpr uint32_t kOut = kNB * 128;
};

enum : int {
  B_AF = 0,                 // stationary tiles full [kAB <= 4]
  B_AE = B_AF + 4,          // stationary tiles empty [kAB] (the TMA-store issuer, after the read)
  B_B = B_AE + 4,           // streamed stage full [kStages]
  B_E = B_B + kStages,      // streamed stage empty [kStages]
  B_S = B_E + kStages,      // S and dP of a sub-chunk ready [3] (TMEM buffer gu % 3)
  B_P = B_S + 3,            // P / dS written in place over that buffer [3] (128 arrivals)
  B_PE = B_P + 3,           // OUT MMAs of the buffer's sub-chunk done: buffer free [3]
  B_OF = B_PE + 3,          // outputs of a tile final [2]
  B_OE = B_OF + 2,          // outputs drained [2]
  B_DX = B_OE + 2,          // exact-D dQ: both groups' partial sums of the tile written (256 arrivals)
  B_DXE = B_DX + 1,         // exact-D dQ: partials read by both groups' epilogues (256 arrivals)
  B_COUNT = B_DXE + 1
};

// Tensor maps of one backward kernel: stationary tiles a0, a1; streamed
// chunks b0, b1; output tiles out0 (, out1) stored with TMA (stationary box).
struct BwdMaps {
  CUtensorMap a0, a1, b0, b1, out0, out1;
  CUtensorMap o;  // dQ: the stationary tile's O rows (fused preprocess)
};

template <int RANK, int D, bool BF16, bool KV_STATIONARY, bool PRECISE>
__device__ __forceinline__ void bwd_body(const BwdMaps& maps, const Geom& g, const TcPlan& pl,
                                         float* __restrict__ rv, const float* __restrict__ lse,
                                         unsigned num_tiles) {
  const CUtensorMap& map_a0 = maps.a0;
  const CUtensorMap& map_a1 = maps.a1;
  const CUtensorMap& map_b0 = maps.b0;
  const CUtensorMap& map_b1 = maps.b1;
  const CUtensorMap& map_out0 = maps.out0;
  const CUtensorMap& map_out1 = maps.out1;
  // dQ forms the row vectors itself (fused preprocess) for rank 1; for
  // multi-dimensional tiles the extra per-tile work measured slower than the
  // separate preprocess pass, so there dQ reads them.
  constexpr bool kFuse = !KV_STATIONARY && RANK == 1 && D <= 64;
  // bf16 dQ (R12): D_x is corrected in-kernel to sum_y P_xy dP_xy.
  // The row value read at the tile start, Dt_x = <dO_x, O_x> from the
  // stored (bf16-rounded) O, is only an estimate; the compute warps also
  // sum c_x = sum_y dS_xy = sum_y P_xy (dP_xy - Dt_x) = D_x - Dt_x in fp32
  // (the P_xy of a row sum to 1), and a second OUT MMA accumulates
  // PK_x = sum_y P_xy k_y next to dQ, so the epilogue forms
  //   dQ_x = scale (sum_y P_xy (dP_xy - Dt_x) k_y - c_x PK_x)
  // = scale sum_y P_xy (dP_xy - D_x) k_y, and writes D_x = Dt_x + c_x to the
  // row vectors the dK/dV kernel (run next) reads.  Dt_x keeps the large
  // first term free of cancellation; c_x is small.  fp16's stored O is 8x
  // finer and keeps Dt_x.
  // Only in the PRECISE variant (bf16_precise(): some window is small).
  constexpr bool kExactD = !KV_STATIONARY && BF16 && PRECISE;
  // bf16 (R13): the 16-bit A operands of the OUT MMAs (P, dS) are
  // split hi + lo, x = bf16(x) + bf16(x - bf16(x)), and both halves are
  // multiplied (a second MMA into the same accumulator), so the products
  // carry ~2^-17 instead of 2^-9 relative error; fp16's 2^-12 needs no split.
  constexpr bool kSplit = BF16 && PRECISE;
  using S = BwdSmem<D, KV_STATIONARY, kFuse, kExactD>;
  constexpr uint32_t kNB = BwdTmem<D>::kNB, kColOut = BwdTmem<D>::kOut;
  constexpr int kStages = S::kSt;
  // Output accumulator columns per tile; double-buffered when two fit.
  constexpr int kOutCols = (KV_STATIONARY || kExactD) ? 2 * D : D;
  constexpr bool kOutDouble = 2 * kOutCols <= 128;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte aligned by pointer arithmetic on the __shared__ array, so the
  // compiler keeps the shared address space (LDS/STS, not generic LD/ST).
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + S::kBar);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + B_COUNT);
  float* vec = reinterpret_cast<float*>(smem + S::kVec);
  const int ns = pl.n_kv > 64 ? 2 : 1;
  const uint32_t warp = ptx::warp_id(), lane = ptx::lane_id();

  if (threadIdx.x == 0) {
    for (int b = 0; b < S::kAB; ++b) {
      ptx::mbar_init(bar + B_AF + b, 1);
      ptx::mbar_init(bar + B_AE + b, 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(bar + B_OF + b, 1);
      ptx::mbar_init(bar + B_OE + b, KV_STATIONARY ? 128 : kCompute);
    }
    ptx::mbar_init(bar + B_DX, kCompute);
    ptx::mbar_init(bar + B_DXE, kCompute);
    for (int b = 0; b < 3; ++b) {
      ptx::mbar_init(bar + B_S + b, 1);
      ptx::mbar_init(bar + B_P + b, 128);
      ptx::mbar_init(bar + B_PE + b, 1);
    }
    for (int s = 0; s < kStages; ++s) {
      // dK/dV: + one cp.async arrival per producer lane (row-vector gather)
      ptx::mbar_init(bar + B_B + s, KV_STATIONARY ? 33 : 1);
      ptx::mbar_init(bar + B_E + s, 1);
    }
    ptx::fence_barrier_init();
    tmem_slot[1] = tmem_slot[2] = 0u;  // dQ drain counters
  }
  if constexpr (KV_STATIONARY) {  // (dQ has no row-vector stages)
    for (int i = threadIdx.x; i < kStages * 256; i += kThreads) vec[i] = 0.f;  // unloaded columns read 0
  }
  ptx::fence_proxy_async();  // before TMA writes the same smem
  if (pl.rows_kv < S::kBRows) {  // rows no TMA box writes must be finite (zero)
    const int nz = (S::kBRows - pl.rows_kv) * S::kRowBytes / 16;
    for (int i = threadIdx.x; i < 2 * kStages * S::kHalves * nz; i += kThreads) {
      const int buf = i / nz, off = i % nz;  // (tensor, stage) x half
      uint4* base = reinterpret_cast<uint4*>(smem + S::kB0 + buf * S::kBHalf + pl.rows_kv * S::kRowBytes);
      base[off] = make_uint4(0, 0, 0, 0);
    }
    ptx::fence_proxy_async();
  }
  if (warp == kMmaWarp) ptx::tmem_alloc<512>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == kProducerWarp) {
    // ===================== TMA producer (whole warp, one lane issues) =====================
    ptx::tma_prefetch(&map_a0);
    ptx::tma_prefetch(&map_a1);
    ptx::tma_prefetch(&map_b0);
    ptx::tma_prefetch(&map_b1);
    const uint32_t bytes = 2 * pl.rows_kv * S::kRowBytes * S::kHalves;
    // dK/dV: the streamed chunk's row vectors (-LSE*log2(e), D) are gathered
    // with 4-byte cp.async by the 32 producer lanes (columns lane, lane+32,
    // ...): chunk origins need no 16-byte alignment, unlike a TMA box.
    const FastDiv f_cx = pl.f_ckv[RANK - 1], f_cy = pl.f_ckv[RANK >= 2 ? RANK - 2 : 0];
    uint32_t kv_it = 0, ti = 0;
    int tr = 0;
    (void)tr;
    for (unsigned tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      TileCtx<RANK> t;
      if (!t.init(g, pl, tile, /*inverse=*/KV_STATIONARY)) continue;
      constexpr int kAB = S::kAB;
      const int ab = ti % kAB;
      if (ti >= kAB) ptx::mbar_wait(bar + B_AE + ab, ((ti / kAB) - 1) & 1);
      if (NA_BWD_TRACE_ON) NA_TRACE_EV(0, tr, 1);
      uint8_t* a0 = smem + S::kA + (2 * ab) * S::kTile;
      uint8_t* a1 = a0 + S::kTile;
      ptx::mbar_expect_tx_w(bar + B_AF + ab, (kFuse ? 3 : 2) * S::kTile);
      for (int h = 0; h < S::kHalves; ++h)
        for (int i = 0; i < pl.q_issues; ++i) {
          t.template load_box<RANK>(&map_a0, a0 + h * S::kAHalf + i * pl.q_box_x * S::kRowBytes, bar + B_AF + ab,
                                    t.q_origin, i * pl.q_box_x, g, 64 * h);
          t.template load_box<RANK>(&map_a1, a1 + h * S::kAHalf + i * pl.q_box_x * S::kRowBytes, bar + B_AF + ab,
                                    t.q_origin, i * pl.q_box_x, g, 64 * h);
        }
      for (int i = 0; i < pl.q_issues; ++i) {
        if constexpr (kFuse)
          t.template load_box<RANK>(&maps.o, smem + S::kO + ab * S::kTile + i * pl.q_box_x * S::kRowBytes,
                                    bar + B_AF + ab, t.q_origin, i * pl.q_box_x, g);
      }
      for (int j = 0; j < t.nchunks; ++j, ++kv_it) {
        const int s = kv_it % kStages;
        if (kv_it >= kStages) ptx::mbar_wait(bar + B_E + s, ((kv_it / kStages) - 1) & 1);
        if (NA_BWD_TRACE_ON) NA_TRACE_EV(0, tr, 2);
        int org[3];
        t.chunk_origin(pl, j, org);
        ptx::mbar_expect_tx_w(bar + B_B + s, bytes);
        for (int h = 0; h < S::kHalves; ++h)
          for (int i = 0; i < pl.kv_issues; ++i) {
            t.template load_box<RANK>(&map_b0,
                                      smem + S::kB0 + s * S::kBTile + h * S::kBHalf + i * pl.kv_box_x * S::kRowBytes,
                                      bar + B_B + s, org, i * pl.kv_box_x, g, 64 * h);
            t.template load_box<RANK>(&map_b1,
                                      smem + S::kB1 + s * S::kBTile + h * S::kBHalf + i * pl.kv_box_x * S::kRowBytes,
                                      bar + B_B + s, org, i * pl.kv_box_x, g, 64 * h);
          }
        if constexpr (KV_STATIONARY) {
          const float* src = rv + rv_base(g, t.bh, t.res);
          float* dst = vec + s * 256;
          for (int c = lane; c < pl.rows_kv; c += 32) {
            int l[3] = {0, 0, 0};
            if constexpr (RANK == 1) {
              l[0] = c;
            } else {
              const uint32_t rest = fdiv((uint32_t)c, f_cx);
              l[RANK - 1] = c - (int)(rest * f_cx.d);
              if constexpr (RANK == 2) {
                l[0] = (int)rest;
              } else {
                const uint32_t r2 = fdiv(rest, f_cy);
                l[1] = (int)(rest - r2 * f_cy.d);
                l[0] = (int)r2;
              }
            }
            bool in = true;
            long long off = 0;
#pragma unroll
            for (int a = 0; a < RANK; ++a) {
              const int x = org[a] + l[a];
              in = in && x < g.rv_lc[a];
              off += (long long)x * g.rv_cs[a];
            }
            // columns outside the padded class extents keep finite stale
            // values; they are masked (P = 0) by every row
            if (in) {
              ptx::cp_async4(dst + c, src + off);
              ptx::cp_async4(dst + 128 + c, src + g.rv_plane + off);
            }
          }
          ptx::cp_async_mbar_arrive_noinc(bar + B_B + s);
        }
      }
      ++ti;
    }
  } else if (warp == kMmaWarp || warp == kSWarp) {
    // ============ MMA issuers (whole warps, one elected lane issues) ============
    // Two independent in-order streams, so neither blocks the other: warp
    // kSWarp issues S/dP of sub-chunk c once its TMEM buffer is free (B_PE of
    // c-3) and its operands are resident; warp kMmaWarp issues OUT(k) once
    // sub-chunk k's packed operands are written.  A commit tracks the MMAs of
    // its own issuing thread: B_S (S warp); B_PE, B_E, B_OF (OUT warp) -- the
    // S/dP MMAs of a chunk are complete before its last OUT is issued (the
    // warpgroup read their results first), so B_E covers both.
    constexpr uint32_t kSw = ptx::sw_layout(D);
    constexpr uint32_t kSbo = 8 * S::kRowBytes;
    int tr = 0;
    (void)tr;
    if (warp == kSWarp) {
      const int n1 = pl.n_kv - 64;
      const uint32_t idesc_s0 = ptx::make_idesc(128, ns == 2 ? 64 : pl.n_kv, BF16, false);
      const uint32_t idesc_s1 = ptx::make_idesc(128, ns == 2 ? n1 : 16, BF16, false);
      uint32_t c_ti = 0, c_kv = 0, c_ub = 0;
      TileCtx<RANK> ct;
      for (unsigned tile = seek_tile<RANK, KV_STATIONARY>(g, pl, blockIdx.x, num_tiles, ct); tile < num_tiles;
           tile = seek_tile<RANK, KV_STATIONARY>(g, pl, tile + gridDim.x, num_tiles, ct)) {
        const int ab = c_ti % S::kAB;
        const uint32_t a0 = ptx::smem_u32(smem + S::kA + (2 * ab) * S::kTile);
        const uint32_t a1 = a0 + S::kTile;
        const int nsub = ct.nchunks * ns;
        for (int c_u = 0; c_u < nsub; ++c_u) {
          const uint32_t kv = c_kv + c_u / ns, gu = c_ub + c_u;
          const int h = c_u % ns, s = kv % kStages;
          const uint32_t b3 = gu % kNB, r3 = gu / kNB;
          if (gu >= kNB) ptx::mbar_wait(bar + B_PE + b3, (r3 - 1) & 1);  // buffer's previous OUT done
          if (c_u == 0) ptx::mbar_wait(bar + B_AF + ab, (c_ti / S::kAB) & 1);
          if (h == 0) ptx::mbar_wait(bar + B_B + s, (kv / kStages) & 1);
          ptx::tc_fence_after();
          const uint32_t off = h * 64 * S::kRowBytes;
          const uint32_t b0 = ptx::smem_u32(smem + S::kB0 + s * S::kBTile) + off;
          const uint32_t b1 = ptx::smem_u32(smem + S::kB1 + s * S::kBTile) + off;
          const uint32_t id = h ? idesc_s1 : idesc_s0;
          const uint32_t buf = b3 * 128;
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            // KV-stationary: S^T = K Q^T, dP^T = V dO^T.  Q-stationary: S = Q K^T, dP = dO V^T.
            // (head_dim 128: K-steps 4..7 read the second 64-column halves)
            const uint32_t ha = (kk >> 2) * S::kAHalf, hb = (kk >> 2) * S::kBHalf, ko = (kk & 3) * 32;
            ptx::mma_ss_w(tmem + buf, ptx::make_sdesc(a0 + ha + ko, 16, kSbo, kSw),
                          ptx::make_sdesc(b0 + hb + ko, 16, kSbo, kSw), id, kk > 0);
            ptx::mma_ss_w(tmem + buf + 64, ptx::make_sdesc(a1 + ha + ko, 16, kSbo, kSw),
                          ptx::make_sdesc(b1 + hb + ko, 16, kSbo, kSw), id, kk > 0);
          }
          ptx::mma_commit_w(bar + B_S + b3);
        }
        c_kv += ct.nchunks;
        c_ub += nsub;
        ++c_ti;
      }
    } else {
      const int n1 = pl.n_kv - 64;
      constexpr uint32_t idesc_o = ptx::make_idesc(128, D, BF16, true);
      uint32_t kv_base = 0, ub = 0, ti = 0;
      TileCtx<RANK> t;
      for (unsigned tile = seek_tile<RANK, KV_STATIONARY>(g, pl, blockIdx.x, num_tiles, t); tile < num_tiles;
           tile = seek_tile<RANK, KV_STATIONARY>(g, pl, tile + gridDim.x, num_tiles, t)) {
        const int nsub = t.nchunks * ns;
        const int ob = kOutDouble ? (ti & 1) : 0;
        const uint32_t out = kColOut + ob * kOutCols;
        for (int u = 0; u < nsub; ++u) {
          const uint32_t kv = kv_base + u / ns, gu = ub + u;
          const int h = u % ns, s = kv % kStages;
          const int width = h ? n1 : (ns == 2 ? 64 : pl.n_kv);
          const uint32_t off = h * 64 * S::kRowBytes;
          const uint32_t b0 = ptx::smem_u32(smem + S::kB0 + s * S::kBTile) + off;
          const uint32_t b1 = ptx::smem_u32(smem + S::kB1 + s * S::kBTile) + off;
          const uint32_t b3 = gu % kNB;
          const uint32_t pk = tmem + b3 * 128;  // P^T over S, dS^T over dP (in place)
          ptx::mbar_wait(bar + B_P + b3, (gu / kNB) & 1);
          if (NA_BWD_TRACE_ON) NA_TRACE_EV(1, tr, 11);
          if (u == 0) {  // the tile's first OUT MMA overwrites the output buffer: drained?
            if (kOutDouble) {
              if (ti >= 2) ptx::mbar_wait(bar + B_OE + ob, ((ti >> 1) - 1) & 1);
            } else {
              if (ti >= 1) ptx::mbar_wait(bar + B_OE, (ti - 1) & 1);
            }
          }
          ptx::tc_fence_after();
          for (int kk = 0; kk < width / 16; ++kk) {
            const uint32_t boff = kk * 16 * S::kRowBytes;
            const uint32_t acc = (u > 0 || kk > 0) ? 1u : 0u;
            // packed A operand columns of K-step kk (16 partner columns):
            // contiguous for fp16; bf16 keeps hi at +0 and lo at +16 of each
            // 32-column half (see the compute warps)
            const uint32_t ca = kSplit ? 32 * (kk >> 1) + 8 * (kk & 1) : 8 * kk;
            if constexpr (KV_STATIONARY) {
              // dV += P^T dO ; dK += dS^T Q   (B operands MN-major; bf16: hi + lo)
              // (LBO: the second 64-column atom of a head_dim 128 row, one half on)
              const uint64_t dod = ptx::make_sdesc(b1 + boff, S::kBHalf, kSbo, kSw);
              const uint64_t qd = ptx::make_sdesc(b0 + boff, S::kBHalf, kSbo, kSw);
              ptx::mma_ts_w(tmem + out + D, pk + ca, dod, idesc_o, acc);
              if constexpr (kSplit) ptx::mma_ts_w(tmem + out + D, pk + ca + 16, dod, idesc_o, 1u);
              ptx::mma_ts_w(tmem + out, pk + 64 + ca, qd, idesc_o, acc);
              if constexpr (kSplit) ptx::mma_ts_w(tmem + out, pk + 64 + ca + 16, qd, idesc_o, 1u);
            } else {
              // dQ += dS K (bf16: hi + lo), exact-D: PK += P K (same B operand)
              const uint64_t kd = ptx::make_sdesc(b0 + boff, S::kBHalf, kSbo, kSw);
              ptx::mma_ts_w(tmem + out, pk + 64 + ca, kd, idesc_o, acc);
              if constexpr (kSplit) ptx::mma_ts_w(tmem + out, pk + 64 + ca + 16, kd, idesc_o, 1u);
              if constexpr (kExactD) ptx::mma_ts_w(tmem + out + D, pk + ca, kd, idesc_o, acc);
            }
          }
          ptx::mma_commit_w(bar + B_PE + b3);
          if (h == ns - 1) ptx::mma_commit_w(bar + B_E + s);
          if (u == nsub - 1) ptx::mma_commit_w(bar + B_OF + ob);
          if (NA_BWD_TRACE_ON) NA_TRACE_EV(1, tr, 12);
        }
        kv_base += t.nchunks;
        ub += nsub;
        ++ti;
      }
    }
  } else {
    // ===================== compute warpgroups (2 x 128 threads) =====================
    const int grp = warp >> 2;           // processes sub-chunks with gu % 2 == grp
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const int gtid = (warp & 3) * 32 + lane;  // 0..127 within the group
    const uint32_t trow = tmem + ((uint32_t)(quarter * 32) << 16);
    const float sl2 = g.scale_log2;
    // TMA-store issuer: dK/dV, thread 0 of the draining group; dQ, thread 0
    // of whichever group finishes its half of the drain second (rank 1, 2;
    // for rank 3 that measured slower -- E dQ 1.51 -> 1.59 ms -- and there
    // both groups meet at a barrier and thread 0 stores).
    constexpr bool kLateStore = !KV_STATIONARY && RANK < 3;
    const bool issuer = (KV_STATIONARY || kLateStore) ? (gtid == 0) : (threadIdx.x == 0);
    uint32_t* drain_cnt = tmem_slot + 1;  // dQ: halves drained per output buffer [2] (monotone)
    uint32_t ub = 0, ti = 0;
    int tr = 0;
    (void)tr;
    const bool tracer = NA_BWD_TRACE_ON && lane == 0 && (warp == 0 || warp == 4);
    // A Q-stationary tile's row values (-LSE*log2(e), D = <dO, O>).
    // Fused preprocess (kFuse): -LSE*log2(e) from the LSE (prefetched from
    // global) and D from the stationary dO tile and the O tile loaded with
    // it, kept in registers for this kernel and written to the row-vector
    // layout (warpgroup 0) for the dK/dV kernel, which runs next; replaces
    // the separate preprocess pass over O and dO.  Otherwise: read from the
    // row-vector layout the preprocess kernel wrote.
    auto row_lse = [&](const TileCtx<RANK>& t, const RowCtx<RANK>& r) {
      return r.valid ? lse[r.token_index(g, t)] : 0.f;
    };
    auto row_read = [&](const TileCtx<RANK>& t, const RowCtx<RANK>& r, float& nl2, float& d) {
      nl2 = 0.f;
      d = 0.f;
      if (r.valid) {
        long long i = rv_base(g, t.bh, t.res);
#pragma unroll
        for (int a = 0; a < RANK; ++a) i += (long long)r.c[a] * g.rv_cs[a];
        nl2 = rv[i];
        d = rv[i + g.rv_plane];
      }
    };
    auto row_vals = [&](const TileCtx<RANK>& t, const RowCtx<RANK>& r, uint32_t tix, float lse_v,
                        float& nl2, float& d) {
      const int ab = tix % S::kAB;
      ptx::mbar_wait(bar + B_AF + ab, (tix / S::kAB) & 1);
      const uint8_t* ot = smem + S::kO + ab * S::kTile;
      const uint8_t* dt = smem + S::kA + (2 * ab + 1) * S::kTile;
      float2 acc[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};  // two packed-FMA chains
#pragma unroll
      for (int c = 0; c < D / 8; ++c) {
        const uint4 a = *reinterpret_cast<const uint4*>(ot + ptx::swz_off(row, c, S::kRowBytes));
        const uint4 b = *reinterpret_cast<const uint4*>(dt + ptx::swz_off(row, c, S::kRowBytes));
        const uint32_t aw[4] = {a.x, a.y, a.z, a.w}, bw[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
        for (int e = 0; e < 4; ++e)
          acc[e & 1] = __ffma2_rn(unpack2<BF16>(aw[e]), unpack2<BF16>(bw[e]), acc[e & 1]);
      }
      nl2 = r.valid ? -lse_v * kLog2e : 0.f;
      d = r.valid ? (acc[0].x + acc[1].x) + (acc[0].y + acc[1].y) : 0.f;
      if (grp == 0 && r.valid) {
        long long i = rv_base(g, t.bh, t.res);
#pragma unroll
        for (int a = 0; a < RANK; ++a) i += (long long)r.c[a] * g.rv_cs[a];
        rv[i] = nl2;
        rv[i + g.rv_plane] = d;
      }
    };
    // ---- epilogue of a finished tile ----
    // Every MMA of the tile is complete once its outputs are final (B_OF), so
    // the tile's stationary smem tiles are dead: the outputs are staged there
    // in the TMA box layout (same swizzle) and written with TMA stores (rows
    // past a ragged class end are clipped by the hardware).  The buffers
    // return to the producer (B_AE) once the stores have read them
    // (release_store, deferred to the issuer's next sub-chunk or tile end).
    // dK/dV (single output buffer): at the start of the next tile, ONE group
    // (the one not owning its first sub-chunk) drains dK (x scale) into the K
    // tile and dV into the V tile, while the other computes.  dQ (double
    // buffer): after each group's first sub-chunk of the next tile, the
    // groups drain one half of dQ's columns each.
    int store_ab = -1;  // issuer: stationary buffer whose store still reads smem
    auto release_store = [&]() {
      if (store_ab >= 0) {
        ptx::bulk_wait_read<0>();
        ptx::mbar_arrive(bar + B_AE + store_ab);  // stationary tiles reusable
        store_ab = -1;
      }
    };
    // Byte offset of 8-column chunk `ch` of this row in a staged stationary
    // tile (head_dim 128: chunks 8..15 in the second half).
    auto sto = [&](int ch) -> uint32_t {
      return (uint32_t)(ch >> 3) * S::kAHalf + ptx::swz_off(row, ch & 7, S::kRowBytes);
    };
    auto drain = [&](uint32_t src, uint8_t* stage, int col0, int ncols, float mul) {
      // 32 columns per TMEM round trip (two loads, one wait): the drain is
      // latency-bound on tcgen05.ld -> wait.
      int c0 = 0;
      for (; c0 + 32 <= ncols; c0 += 32) {
        uint32_t ov[32];
        NA_TMEM_LD32(trow + src + c0, ov);
        ptx::tmem_ld_wait();
        uint32_t pk[16];
#pragma unroll
        for (int c = 0; c < 32; c += 2)
          pk[c >> 1] = pack2<BF16>(__uint_as_float(ov[c]) * mul, __uint_as_float(ov[c + 1]) * mul);
        const int chunk = (col0 + c0) / 8;
#pragma unroll
        for (int q = 0; q < 4; ++q)
          *reinterpret_cast<uint4*>(stage + sto(chunk + q)) =
              make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
      }
      if (c0 + 8 == ncols) {  // an 8-column remainder (dQ halves at D = 16)
        uint32_t ov[8];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(ov[0]), "=r"(ov[1]), "=r"(ov[2]), "=r"(ov[3]), "=r"(ov[4]), "=r"(ov[5]),
                       "=r"(ov[6]), "=r"(ov[7])
                     : "r"(trow + src + c0));
        ptx::tmem_ld_wait();
        uint32_t pk[4];
#pragma unroll
        for (int c = 0; c < 8; c += 2)
          pk[c >> 1] = pack2<BF16>(__uint_as_float(ov[c]) * mul, __uint_as_float(ov[c + 1]) * mul);
        *reinterpret_cast<uint4*>(stage + sto((col0 + c0) / 8)) =
            make_uint4(pk[0], pk[1], pk[2], pk[3]);
      } else if (c0 < ncols) {  // a 16-column remainder (dQ halves at D = 32)
        uint32_t ov[16];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(ov[0]), "=r"(ov[1]), "=r"(ov[2]), "=r"(ov[3]), "=r"(ov[4]), "=r"(ov[5]), "=r"(ov[6]),
              "=r"(ov[7]), "=r"(ov[8]), "=r"(ov[9]), "=r"(ov[10]), "=r"(ov[11]), "=r"(ov[12]),
              "=r"(ov[13]), "=r"(ov[14]), "=r"(ov[15])
            : "r"(trow + src + c0));
        ptx::tmem_ld_wait();
        uint32_t pk[8];
#pragma unroll
        for (int c = 0; c < 16; c += 2)
          pk[c >> 1] = pack2<BF16>(__uint_as_float(ov[c]) * mul, __uint_as_float(ov[c + 1]) * mul);
        const int chunk = (col0 + c0) / 8;
        *reinterpret_cast<uint4*>(stage + sto(chunk)) =
            make_uint4(pk[0], pk[1], pk[2], pk[3]);
        *reinterpret_cast<uint4*>(stage + sto(chunk + 1)) =
            make_uint4(pk[4], pk[5], pk[6], pk[7]);
      }
    };
    // Exact-D dQ drain: (dQacc - c_x PK_x) * scale, 16 columns per round trip.
    auto drain_exact = [&](uint32_t src, uint32_t src_pk, uint8_t* stage, int col0, int ncols, float mul,
                           float corr) {
      if (ncols == 8) {  // D = 16: each group drains 8 columns
        uint32_t ov[8], kv_[8];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(ov[0]), "=r"(ov[1]), "=r"(ov[2]), "=r"(ov[3]), "=r"(ov[4]), "=r"(ov[5]),
                       "=r"(ov[6]), "=r"(ov[7])
                     : "r"(trow + src));
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(kv_[0]), "=r"(kv_[1]), "=r"(kv_[2]), "=r"(kv_[3]), "=r"(kv_[4]), "=r"(kv_[5]),
                       "=r"(kv_[6]), "=r"(kv_[7])
                     : "r"(trow + src_pk));
        ptx::tmem_ld_wait();
        uint32_t pk[4];
#pragma unroll
        for (int c = 0; c < 8; c += 2)
          pk[c >> 1] = pack2<BF16>((__uint_as_float(ov[c]) - corr * __uint_as_float(kv_[c])) * mul,
                                   (__uint_as_float(ov[c + 1]) - corr * __uint_as_float(kv_[c + 1])) * mul);
        *reinterpret_cast<uint4*>(stage + sto(col0 / 8)) =
            make_uint4(pk[0], pk[1], pk[2], pk[3]);
        return;
      }
      for (int c0 = 0; c0 < ncols; c0 += 16) {
        uint32_t ov[16], kv_[16];
        NA_TMEM_LD16(trow + src + c0, ov);
        NA_TMEM_LD16(trow + src_pk + c0, kv_);
        ptx::tmem_ld_wait();
        uint32_t pk[8];
#pragma unroll
        for (int c = 0; c < 16; c += 2)
          pk[c >> 1] = pack2<BF16>((__uint_as_float(ov[c]) - corr * __uint_as_float(kv_[c])) * mul,
                                   (__uint_as_float(ov[c + 1]) - corr * __uint_as_float(kv_[c + 1])) * mul);
        const int chunk = (col0 + c0) / 8;
        *reinterpret_cast<uint4*>(stage + sto(chunk)) =
            make_uint4(pk[0], pk[1], pk[2], pk[3]);
        *reinterpret_cast<uint4*>(stage + sto(chunk + 1)) =
            make_uint4(pk[4], pk[5], pk[6], pk[7]);
      }
    };
    float* dx_part = reinterpret_cast<float*>(smem + S::kDx);  // exact-D: [2 groups][128 rows]
    long long prow_rv = -1;  // exact-D: row-vector index of this row in the pending tile (-1: invalid row)
    float prow_d = 0.f;      // exact-D: its Dt_x
    auto rv_index = [&](const TileCtx<RANK>& t, const RowCtx<RANK>& r) -> long long {
      if (!r.valid) return -1;
      long long i = rv_base(g, t.bh, t.res);
#pragma unroll
      for (int a = 0; a < RANK; ++a) i += (long long)r.c[a] * g.rv_cs[a];
      return i;
    };
    auto epilogue = [&](const TileCtx<RANK>& t, uint32_t tix) {
      const int ob = kOutDouble ? (tix & 1) : 0, ab = tix % S::kAB;
      ptx::mbar_wait(bar + B_OF + ob, kOutDouble ? ((tix >> 1) & 1) : (tix & 1));
      if (tracer) NA_TRACE_EV(2 + grp, tr, 24);
      ptx::tc_fence_after();
      uint8_t* stage0 = smem + S::kA + (2 * ab) * S::kTile;
      const uint32_t src = kColOut + ob * kOutCols;  // (kColOut: this D's layout, BwdTmem)
      if constexpr (KV_STATIONARY) {
        drain(src, stage0, 0, D, g.scale);                 // dK -> K tile
        drain(src + D, stage0 + S::kTile, 0, D, 1.f);      // dV -> V tile
      } else if constexpr (kExactD) {
        ptx::mbar_wait(bar + B_DX, tix & 1);  // both groups' c_x partials of the tile
        const float corr = dx_part[row] + dx_part[128 + row];
        ptx::mbar_arrive(bar + B_DXE);
        drain_exact(src + grp * (D / 2), src + D + grp * (D / 2), stage0, grp * (D / 2), D / 2, g.scale, corr);
        if (grp == 0 && prow_rv >= 0) rv[prow_rv + g.rv_plane] = prow_d + corr;  // D_x for dK/dV
      } else {
        drain(src + grp * (D / 2), stage0, grp * (D / 2), D / 2, g.scale);  // half of dQ -> Q tile
      }
      ptx::tc_fence_before();
      ptx::mbar_arrive(bar + B_OE + ob);
      ptx::fence_proxy_async();  // staged tile visible to the TMA engine
      if (tracer) NA_TRACE_EV(2 + grp, tr, 25);
      if constexpr (KV_STATIONARY || kLateStore) ptx::named_bar_sync(3 + grp, 128);
      else ptx::named_bar_sync(3, kCompute);
      bool store_now = issuer;
      if constexpr (kLateStore) {
        // The two groups drain at different times (a sub-chunk apart):
        // the later one stores, so neither waits for the other.
        if (issuer) {
          uint32_t old;
          asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;"
                       : "=r"(old) : "r"(ptx::smem_u32(drain_cnt + ob)) : "memory");
          store_now = (old & 1u) == 1u;
        }
      }
      if (store_now) {
        for (int h = 0; h < S::kHalves; ++h)
          for (int i = 0; i < pl.q_issues; ++i) {
            t.template store_box<RANK>(&map_out0, stage0 + h * S::kAHalf + i * pl.q_box_x * S::kRowBytes,
                                       i * pl.q_box_x, g, 64 * h);
            if constexpr (KV_STATIONARY)
              t.template store_box<RANK>(&map_out1, stage0 + S::kTile + h * S::kAHalf + i * pl.q_box_x * S::kRowBytes,
                                         i * pl.q_box_x, g, 64 * h);
          }
        ptx::bulk_commit();
        store_ab = ab;
      }
    };

    TileCtx<RANK> t, tp;  // current tile; tile whose epilogue is pending
    RowCtx<RANK> r;
    bool pend = false;
    unsigned tile = seek_tile<RANK, KV_STATIONARY>(g, pl, blockIdx.x, num_tiles, t);
    if (tile < num_tiles) r.init(g, pl, t, row, /*inverse=*/KV_STATIONARY);
    float row_nl2 = 0.f, row_d = 0.f;
    if constexpr (kFuse) {
      if (tile < num_tiles) row_vals(t, r, 0, row_lse(t, r), row_nl2, row_d);
    } else if constexpr (!KV_STATIONARY) {
      if (tile < num_tiles) row_read(t, r, row_nl2, row_d);
    }
    uint32_t kv_base = 0;
    while (tile < num_tiles) {
      const int nsub = t.nchunks * ns;
      const int u_first = (int)((grp - ub) & 1u);
      if constexpr (KV_STATIONARY) {
        // The group not owning the tile's first sub-chunk drains the previous tile.
        if (pend && u_first == 1) epilogue(tp, ti - 1);
        pend = false;
      }
      // Next tile: found during this group's last sub-chunk of the tile (so a
      // Q-stationary tile's row values load while that sub-chunk computes).
      TileCtx<RANK> tn;
      RowCtx<RANK> rn;
      unsigned tile_n = num_tiles;
      bool tn_known = false;
      float nrow_nl2 = 0.f, nrow_d = 0.f;  // (kFuse: nrow_nl2 holds the prefetched LSE)
      // This group's sub-chunks u_first, u_first + 2, ...: chunk origins by
      // odometer (one chunk per step when a chunk has two sub-chunks, two
      // otherwise); each mask is computed in the previous sub-chunk's load shadow.
      int org[3] = {t.lo[0], t.lo[1], t.lo[2]};
      if (u_first / ns) t.next_origin(pl, org);
      uint32_t w[2];
      r.sub_mask(pl, org, u_first % ns, w);
      float2 dxacc = make_float2(0.f, 0.f);  // exact-D: this group's part of c_x = sum_y dS_xy
      for (int u = u_first; u < nsub; u += 2) {
        if (issuer && u != u_first) release_store();  // the store has had a sub-chunk to read
        const uint32_t gu = ub + u;
        const int j = u / ns, h = u % ns;
        // Partner (query) values of the chunk, TMA-loaded with it:
        // [-LSE*log2(e) x 128 | D x 128] (cp.async-gathered); this sub-chunk's 64 columns.
        const uint32_t kv = kv_base + j;
        const float* cl = vec + (kv % kStages) * 256 + h * 64;
        const float* cd = cl + 128;
        if (u + 2 >= nsub) {
          tile_n = seek_tile<RANK, KV_STATIONARY>(g, pl, tile + gridDim.x, num_tiles, tn);
          tn_known = true;
          if (tile_n < num_tiles) {
            rn.init(g, pl, tn, row, /*inverse=*/KV_STATIONARY);
            if constexpr (kFuse) nrow_nl2 = row_lse(tn, rn);  // LSE prefetch
            else if constexpr (!KV_STATIONARY) row_read(tn, rn, nrow_nl2, nrow_d);
          }
        }
        const uint32_t b3 = gu % kNB;
        const uint32_t buf = b3 * 128;  // S at +0, dP at +64; P / dS written back in place
        if (tracer) NA_TRACE_EV(2 + grp, tr, 19);
        ptx::mbar_wait(bar + B_S + b3, (gu / kNB) & 1);
        if constexpr (KV_STATIONARY) {
          // The chunk's stage is still held (its B_E needs this P), so its
          // phase is current: the row-vector bytes are visible after this.
          ptx::mbar_wait(bar + B_B + (kv % kStages), (kv / kStages) & 1);
        }
        if (tracer) NA_TRACE_EV(2 + grp, tr, 20);
        ptx::tc_fence_after();
        // Per 32-column half: load S and dP, compute P and dS, and store them
        // packed over the columns already read (the buffer stays this
        // sub-chunk's until its OUT MMAs are done; three buffers rotate).
        const uint32_t pk = trow + buf;
        uint32_t pk_p[2][16], pk_s[2][16];
        uint32_t wn[2] = {0u, 0u};
#pragma unroll
        for (int gq = 0; gq < 2; ++gq) {
          const bool any = __any_sync(0xffffffffu, w[gq] != 0u);
          uint32_t sv[32], pv[32];  // loaded unconditionally (a conditional load costs register zero-fills)
          NA_TMEM_LD32(trow + buf + 32 * gq, sv);
          NA_TMEM_LD32(trow + buf + 64 + 32 * gq, pv);
          if (gq == 0 && u + 2 < nsub) {  // next sub-chunk's mask, in the load shadow
            t.next_origin(pl, org);
            if (ns == 1) t.next_origin(pl, org);
            r.sub_mask(pl, org, h, wn);
          }
          ptx::tmem_ld_wait();
          if (tracer) NA_TRACE_EV(2 + grp, tr, 26 + 2 * gq);
          // P and dS of 4 partner columns c..c+3 (fp32 pairs)
          auto calc4 = [&](int c, bool full, float2& p0, float2& p1, float2& ds0, float2& ds1) {
            float4 nl4, dd4;
            if constexpr (KV_STATIONARY) {
              nl4 = *reinterpret_cast<const float4*>(cl + 32 * gq + c);
              dd4 = *reinterpret_cast<const float4*>(cd + 32 * gq + c);
            } else {
              nl4 = make_float4(row_nl2, row_nl2, row_nl2, row_nl2);
              dd4 = make_float4(row_d, row_d, row_d, row_d);
            }
            float2 x0 = __ffma2_rn(make_float2(__uint_as_float(sv[c]), __uint_as_float(sv[c + 1])),
                                   make_float2(sl2, sl2), make_float2(nl4.x, nl4.y));
            float2 x1 = __ffma2_rn(make_float2(__uint_as_float(sv[c + 2]), __uint_as_float(sv[c + 3])),
                                   make_float2(sl2, sl2), make_float2(nl4.z, nl4.w));
            if (!full) {
              const uint32_t ww = w[gq];
              x0.x = (ww >> c) & 1u ? x0.x : -INFINITY;
              x0.y = (ww >> (c + 1)) & 1u ? x0.y : -INFINITY;
              x1.x = (ww >> (c + 2)) & 1u ? x1.x : -INFINITY;
              x1.y = (ww >> (c + 3)) & 1u ? x1.y : -INFINITY;
            }
            p0 = make_float2(ptx::ex2(x0.x), ptx::ex2(x0.y));  // MUFU
            p1 = use_poly<KV_STATIONARY ? (RANK == 3 ? 1 : 0) : (D <= 32 ? 3 : 1)>(c) ? exp2_poly2(x1)                   // FMA pipe
                             : make_float2(ptx::ex2(x1.x), ptx::ex2(x1.y));
            ds0 = __fmul2_rn(p0, __fadd2_rn(make_float2(__uint_as_float(pv[c]), __uint_as_float(pv[c + 1])),
                                            make_float2(-dd4.x, -dd4.y)));
            ds1 = __fmul2_rn(p1, __fadd2_rn(make_float2(__uint_as_float(pv[c + 2]), __uint_as_float(pv[c + 3])),
                                            make_float2(-dd4.z, -dd4.w)));
            if constexpr (kExactD) dxacc = __fadd2_rn(dxacc, __fadd2_rn(ds0, ds1));
          };
          if constexpr (kSplit) {
            // bf16: per 16 partner columns j, hi words at +8j and lo words at
            // +16+8j of this half's 32 columns, over S (P) and dP (dS), which
            // this half has already loaded.
            const bool full = __all_sync(0xffffffffu, w[gq] == 0xffffffffu);
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              uint32_t ph[8], pl[8], sh[8], sl[8];
              if (!any) {
#pragma unroll
                for (int i = 0; i < 8; ++i) ph[i] = pl[i] = sh[i] = sl[i] = 0u;
              } else {
#pragma unroll
                for (int c = 16 * j; c < 16 * j + 16; c += 4) {
                  float2 p0, p1, ds0, ds1;
                  calc4(c, full, p0, p1, ds0, ds1);
                  const int i = (c - 16 * j) >> 1;
                  ph[i] = pack2<BF16>(p0.x, p0.y);
                  ph[i + 1] = pack2<BF16>(p1.x, p1.y);
                  sh[i] = pack2<BF16>(ds0.x, ds0.y);
                  sh[i + 1] = pack2<BF16>(ds1.x, ds1.y);
                  const float2 r0 = __ffma2_rn(unpack2<BF16>(ph[i]), make_float2(-1.f, -1.f), p0);
                  const float2 r1 = __ffma2_rn(unpack2<BF16>(ph[i + 1]), make_float2(-1.f, -1.f), p1);
                  const float2 t0 = __ffma2_rn(unpack2<BF16>(sh[i]), make_float2(-1.f, -1.f), ds0);
                  const float2 t1 = __ffma2_rn(unpack2<BF16>(sh[i + 1]), make_float2(-1.f, -1.f), ds1);
                  pl[i] = pack2<BF16>(r0.x, r0.y);
                  pl[i + 1] = pack2<BF16>(r1.x, r1.y);
                  sl[i] = pack2<BF16>(t0.x, t0.y);
                  sl[i + 1] = pack2<BF16>(t1.x, t1.y);
                }
              }
              const uint32_t a = pk + 32 * gq + 8 * j;
              NA_TMEM_ST8(a + 64, sh);       // dS (dS^T) hi
              NA_TMEM_ST8(a + 64 + 16, sl);  // dS lo
              NA_TMEM_ST8(a, ph);            // P (P^T) hi
              if constexpr (KV_STATIONARY) NA_TMEM_ST8(a + 16, pl);  // P^T lo (dV); dQ's PK needs no lo
            }
          } else {
            if (!any) {
#pragma unroll
              for (int c = 0; c < 16; ++c) pk_p[gq][c] = pk_s[gq][c] = 0u;
            } else {
              const bool full = __all_sync(0xffffffffu, w[gq] == 0xffffffffu);
#pragma unroll
              for (int c = 0; c < 32; c += 4) {
                float2 p0, p1, ds0, ds1;
                calc4(c, full, p0, p1, ds0, ds1);
                pk_p[gq][c >> 1] = pack2<BF16>(p0.x, p0.y);
                pk_p[gq][(c >> 1) + 1] = pack2<BF16>(p1.x, p1.y);
                pk_s[gq][c >> 1] = pack2<BF16>(ds0.x, ds0.y);
                pk_s[gq][(c >> 1) + 1] = pack2<BF16>(ds1.x, ds1.y);
              }
            }
            if constexpr (KV_STATIONARY) {
              NA_TMEM_ST16(pk + 16 * gq, pk_p[gq]);       // P^T  -> A of dV += P^T dO
              NA_TMEM_ST16(pk + 64 + 16 * gq, pk_s[gq]);  // dS^T -> A of dK += dS^T Q
            } else {
              NA_TMEM_ST16(pk + 64 + 16 * gq, pk_s[gq]);  // dS -> A of dQ += dS K
            }
          }
          if (tracer) NA_TRACE_EV(2 + grp, tr, 27 + 2 * gq);
        }
        ptx::tmem_st_wait();
        ptx::tc_fence_before();
        ptx::mbar_arrive(bar + B_P + b3);
        if (tracer) NA_TRACE_EV(2 + grp, tr, 21);
        w[0] = wn[0];
        w[1] = wn[1];
        if constexpr (!KV_STATIONARY) {
          if (pend) {  // previous tile's dQ, now that the tensor core has this sub-chunk
            epilogue(tp, ti - 1);
            pend = false;
          }
        }
      }
      if (tracer) NA_TRACE_EV(2 + grp, tr, 22);
      if constexpr (!KV_STATIONARY) {
        if (pend) {  // this group had no sub-chunk in the tile
          epilogue(tp, ti - 1);
          pend = false;
        }
      }
      if constexpr (kExactD) {
        // publish this group's c_x partial once both epilogues have read the
        // previous tile's (single slot)
        if (ti > 0) ptx::mbar_wait(bar + B_DXE, (ti - 1) & 1);
        dx_part[grp * 128 + row] = dxacc.x + dxacc.y;
        ptx::mbar_arrive(bar + B_DX);
        prow_rv = rv_index(t, r);
        prow_d = row_d;
      }
      if (issuer) release_store();
      tp = t;
      pend = true;
      ub += nsub;
      kv_base += t.nchunks;
      ++ti;
      if (!tn_known) {
        tile_n = seek_tile<RANK, KV_STATIONARY>(g, pl, tile + gridDim.x, num_tiles, tn);
        if (tile_n < num_tiles) {
          rn.init(g, pl, tn, row, /*inverse=*/KV_STATIONARY);
          if constexpr (kFuse) nrow_nl2 = row_lse(tn, rn);
          else if constexpr (!KV_STATIONARY) row_read(tn, rn, nrow_nl2, nrow_d);
        }
      }
      tile = tile_n;
      t = tn;
      r = rn;
      if constexpr (kFuse) {
        if (tile < num_tiles) row_vals(t, r, ti, nrow_nl2, row_nl2, row_d);
      } else {
        row_nl2 = nrow_nl2;
        row_d = nrow_d;
      }
      if (tracer) NA_TRACE_EV(2 + grp, tr, 23);
    }
    if (pend) {
      if constexpr (KV_STATIONARY) {
        if ((int)((grp - ub) & 1u) == 1) epilogue(tp, ti - 1);
      } else {
        epilogue(tp, ti - 1);
      }
    }
    if (issuer) {
      release_store();
      ptx::bulk_wait<0>();  // stores done before exit
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem);
  }
}

// dK, dV: key-stationary over the inverse halo.
template <int RANK, int D, bool BF16, bool PRECISE>
__global__ void __launch_bounds__(kThreads, 1)
    fna_dkdv_tc(const __grid_constant__ BwdMaps maps, Geom g, TcPlan pl, float* __restrict__ rv,
                unsigned num_tiles) {
  bwd_body<RANK, D, BF16, true, PRECISE>(maps, g, pl, rv, nullptr, num_tiles);
}

// dQ: query-stationary over the forward halo.
template <int RANK, int D, bool BF16, bool PRECISE>
__global__ void __launch_bounds__(kThreads, 1)
    fna_dq_tc(const __grid_constant__ BwdMaps maps, Geom g, TcPlan pl, float* __restrict__ rv,
              const float* __restrict__ lse, unsigned num_tiles) {
  bwd_body<RANK, D, BF16, false, PRECISE>(maps, g, pl, rv, lse, num_tiles);
}

// Everything that can fail on the host (function attributes; the tensor maps
// are encoded by the caller) happens before the first launch, so an error
// leaves the stream and the workspace untouched (include/na.h).
template <int RANK, int D, bool BF16, bool PRECISE = false>
cudaError_t launch_all(int dtype, const Geom& g, const Layout& ly, const TcPlan* pls, const BwdMaps& mkv, const BwdMaps& mq,
                       const void* o, const void* d_o, float* rv, const float* lse, cudaStream_t st) {
  constexpr bool kFuse = RANK == 1 && D <= 64;  // dQ forms the row vectors (see bwd_body)
  const int smem_kv = BwdSmem<D, true, false>::kBytes + 1024;
  const int smem_q = BwdSmem<D, false, kFuse, BF16 && PRECISE>::kBytes + 1024;
  auto kdkdv = fna_dkdv_tc<RANK, D, BF16, PRECISE>;
  auto kdq = fna_dq_tc<RANK, D, BF16, PRECISE>;
  cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kdkdv), smem_kv);
  if (e != cudaSuccess) return e;
  if ((e = ensure_smem_attr(reinterpret_cast<const void*>(kdq), smem_q)) != cudaSuccess) return e;
  const long long tiles_kv = (long long)g.BH * pls[0].nres * pls[0].tiles;
  const long long tiles_q = (long long)g.BH * pls[1].nres * pls[1].tiles;
  if (tiles_kv > 0x7fffffffLL || tiles_q > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
  const unsigned grid_kv = (unsigned)(tiles_kv < num_sms() ? tiles_kv : num_sms());
  const unsigned grid_q = (unsigned)(tiles_q < num_sms() ? tiles_q : num_sms());
  // Row-vector layout: rank 1, written by the dQ kernel (fused preprocess;
  // slots no token maps to, ragged residue classes, must read as 0);
  // otherwise by the preprocess kernel.
  e = kFuse ? rv_clear_padding(g, rv, st) : bwd_preprocess(dtype, g, ly, o, d_o, lse, rv, st);
  if (e != cudaSuccess) return e;
  // dQ first: when fused it also writes the row vectors (-LSE*log2(e), D)
  // the dK/dV kernel streams.
  prof_begin(KID_DQ_TC, st);
  kdq<<<grid_q, kThreads, smem_q, st>>>(mq, g, pls[1], rv, lse, (unsigned)tiles_q);
  prof_end(st);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  prof_begin(KID_DKDV_TC, st);
  kdkdv<<<grid_kv, kThreads, smem_kv, st>>>(mkv, g, pls[0], rv, (unsigned)tiles_kv);
  prof_end(st);
  return cudaGetLastError();
}

template <int RANK>
cudaError_t by_type(int dtype, const Geom& g, const Layout& ly, const TcPlan* pl, const BwdMaps& mkv, const BwdMaps& mq,
                    const void* o, const void* d_o, float* rv, const float* lse, cudaStream_t st) {
  if (dtype == 2) {
    const bool pr = bf16_precise(g);
    if (g.D == 128)
      return pr ? launch_all<RANK, 128, true, true>(dtype, g, ly, pl, mkv, mq, o, d_o, rv, lse, st)
                : launch_all<RANK, 128, true>(dtype, g, ly, pl, mkv, mq, o, d_o, rv, lse, st);
    if (g.D == 64)
      return pr ? launch_all<RANK, 64, true, true>(dtype, g, ly, pl, mkv, mq, o, d_o, rv, lse, st)
                : launch_all<RANK, 64, true>(dtype, g, ly, pl, mkv, mq, o, d_o, rv, lse, st);
    if (g.D == 16)
      return pr ? launch_all<RANK, 16, true, true>(dtype, g, ly, pl, mkv, mq, o, d_o, rv, lse, st)
                : launch_all<RANK, 16, true>(dtype, g, ly, pl, mkv, mq, o, d_o, rv, lse, st);
    return pr ? launch_all<RANK, 32, true, true>(dtype, g, ly, pl, mkv, mq, o, d_o, rv, lse, st)
              : launch_all<RANK, 32, true>(dtype, g, ly, pl, mkv, mq, o, d_o, rv, lse, st);
  }
  if (g.D == 128) return launch_all<RANK, 128, false>(dtype, g, ly, pl, mkv, mq, o, d_o, rv, lse, st);
  if (g.D == 64) return launch_all<RANK, 64, false>(dtype, g, ly, pl, mkv, mq, o, d_o, rv, lse, st);
  if (g.D == 16) return launch_all<RANK, 16, false>(dtype, g, ly, pl, mkv, mq, o, d_o, rv, lse, st);
  return launch_all<RANK, 32, false>(dtype, g, ly, pl, mkv, mq, o, d_o, rv, lse, st);
}

}  // namespace

cudaError_t tc_bwd(int dtype, const Geom& g, const Layout& ly, const void* q, const void* k, const void* v,
                   const void* o, const void* d_o, const float* lse, void* dq, void* dk, void* dv,
                   float* Dvec, cudaStream_t st, int* launches) {
  const char* why;
  if (!tc_supported(dtype, g, &why)) return cudaErrorNotSupported;
  // Each kernel has its own plan (na_tune may measure different winners).
  const PlanChoice pc = plan_choice(g, dtype);
  const TcPlan pls[2] = {make_plan(g, 128, pc.dkdv), make_plan(g, 128, pc.dq)};
  // dK/dV kernel: stationary K, V tiles; streamed Q, dO chunks; outputs dK, dV.
  // dQ kernel: stationary Q, dO tiles; streamed K, V chunks; output dQ.
  BwdMaps mkv, mq;
  const void* tile_src[2][2] = {{k, v}, {q, d_o}};
  const void* chunk_src[2][2] = {{q, d_o}, {k, v}};
  BwdMaps* mm[2] = {&mkv, &mq};
  cudaError_t e;
  for (int w = 0; w < 2; ++w) {
    const TcPlan& pl = pls[w];
    if ((e = make_map(&mm[w]->a0, dtype, g, ly, tile_src[w][0], pl.tq, pl.q_box_x)) != cudaSuccess) return e;
    if ((e = make_map(&mm[w]->a1, dtype, g, ly, tile_src[w][1], pl.tq, pl.q_box_x)) != cudaSuccess) return e;
    if ((e = make_map(&mm[w]->b0, dtype, g, ly, chunk_src[w][0], pl.ckv, pl.kv_box_x)) != cudaSuccess) return e;
    if ((e = make_map(&mm[w]->b1, dtype, g, ly, chunk_src[w][1], pl.ckv, pl.kv_box_x)) != cudaSuccess) return e;
  }
  if ((e = make_map(&mkv.out0, dtype, g, ly, dk, pls[0].tq, pls[0].q_box_x)) != cudaSuccess) return e;
  if ((e = make_map(&mkv.out1, dtype, g, ly, dv, pls[0].tq, pls[0].q_box_x)) != cudaSuccess) return e;
  if ((e = make_map(&mq.out0, dtype, g, ly, dq, pls[1].tq, pls[1].q_box_x)) != cudaSuccess) return e;
  mq.out1 = mq.out0;
  if ((e = make_map(&mq.o, dtype, g, ly, o, pls[1].tq, pls[1].q_box_x)) != cudaSuccess) return e;
  mkv.o = mq.o;
  *launches = (g.rank == 1 && g.D <= 64) ? 2 : 3;  // rank 1: preprocess fused into dQ (head_dim <= 64)
  switch (g.rank) {
    case 1: return by_type<1>(dtype, g, ly, pls, mkv, mq, o, d_o, Dvec, lse, st);
    case 2: return by_type<2>(dtype, g, ly, pls, mkv, mq, o, d_o, Dvec, lse, st);
    default: return by_type<3>(dtype, g, ly, pls, mkv, mq, o, d_o, Dvec, lse, st);
  }
}

#ifdef NA_TRACE
// Trace build only (libna_trace.so): point the backward kernels' event buffer.
extern "C" int na_debug_set_trace_bwd(void* p, int which) {
  if (cudaMemcpyToSymbol(na::g_trace_sel, &which, sizeof(which)) != cudaSuccess) return 1;
  return cudaMemcpyToSymbol(na::g_trace, &p, sizeof(p)) == cudaSuccess ? 0 : 1;
}
#endif

}  // namespace na
