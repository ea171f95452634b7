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
//                dS = P (dP - D), dQ += dS K.
// Persistent, 1 CTA per SM walking tiles blockIdx.x, +gridDim.x, ...
// Warp roles (320 threads): warp 0 TMA producer, warp 1 TMEM owner + MMA
// issuer (whole warps, one elected lane issues), warps 2..9 two compute
// warpgroups (thread = TMEM lane = stationary row).  Sub-chunk with global
// index gu lives in TMEM buffer gu%2 and is processed by warpgroup gu%2, so
// the tensor core computes the next sub-chunk while a warpgroup works:
//   MMA order per tile: ST_0, ST_1, [P_0] OUT_0, ST_2, [P_1] OUT_1, ST_3, ...
// Stationary tiles are double-buffered in smem and the output accumulators
// in TMEM, so tile i+1's loads and MMAs overlap tile i's epilogue.
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
static __device__ int g_trace_sel;  // trace build: 1 = dK/dV kernel, 0 = dQ kernel
#define NA_BWD_TRACE_ON (g_trace_sel == (KV_STATIONARY ? 1 : 0))
#else
#define NA_BWD_TRACE_ON false
#endif

constexpr int kStages = 2;
constexpr int kThreads = 320;
constexpr int kCompute = 256;  // compute threads (warps 0..7)
// The warp scheduler favours the highest warp id among eligible warps, so the
// latency-critical single-lane roles take the highest ids.
constexpr int kProducerWarp = 8;
constexpr int kMmaWarp = 9;
constexpr float kLog2e = 1.4426950408889634f;

template <int D>
struct BwdSmem {
  static constexpr int kRowBytes = D * 2;
  static constexpr int kTile = 128 * kRowBytes;
  static constexpr int kA = 0;                        // stationary [2 bufs][2 tiles] (K,V | Q,dO)
  static constexpr int kB0 = kA + 4 * kTile;          // streamed [kStages] (Q | K)
  static constexpr int kB1 = kB0 + kStages * kTile;   // streamed [kStages] (dO | V)
  static constexpr int kVec = kB1 + kStages * kTile;  // [kStages][-LSE2 x128 | D x128] fp32 (dK/dV)
  static constexpr int kBar = kVec + kStages * 256 * 4;
  static constexpr int kBytes = kBar + 256;
};

// TMEM columns: [0,128) two 64-column S-like buffers, [128,256) two dP-like
// buffers, [256 + 128*ob, ...) output accumulators of tile parity ob
// (first output at +0, second at +D).
constexpr uint32_t kColS = 0, kColP = 128, kColOut = 256;

enum : int {
  B_AF = 0,                 // stationary tiles full [2]
  B_AE = B_AF + 2,          // stationary tiles empty [2]
  B_B = B_AE + 2,           // streamed stage full [kStages]
  B_E = B_B + kStages,      // streamed stage empty [kStages]
  B_S = B_E + kStages,      // S and dP of a sub-chunk ready [2]
  B_P = B_S + 2,            // packed operands of a sub-chunk written [2] (128 arrivals)
  B_OF = B_P + 2,           // outputs of a tile final [2]
  B_OE = B_OF + 2,          // outputs drained by the epilogue [2] (256 arrivals)
  B_COUNT = B_OE + 2
};

// Tensor maps of one backward kernel: stationary tiles a0, a1; streamed
// chunks b0, b1; output tiles out0 (, out1) stored with TMA (stationary box).
struct BwdMaps {
  CUtensorMap a0, a1, b0, b1, out0, out1;
  CUtensorMap rv;  // dK/dV: the streamed chunk's row vector (-LSE*log2(e), D)
};

template <int RANK, int D, bool BF16, bool KV_STATIONARY>
__device__ __forceinline__ void bwd_body(const BwdMaps& maps, const Geom& g, const TcPlan& pl,
                                         const float* __restrict__ rv, unsigned num_tiles) {
  const CUtensorMap& map_a0 = maps.a0;
  const CUtensorMap& map_a1 = maps.a1;
  const CUtensorMap& map_b0 = maps.b0;
  const CUtensorMap& map_b1 = maps.b1;
  const CUtensorMap& map_out0 = maps.out0;
  const CUtensorMap& map_out1 = maps.out1;
  using S = BwdSmem<D>;
  using T = typename std::conditional<BF16, __nv_bfloat16, __half>::type;
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
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(bar + B_AF + b, 1);
      ptx::mbar_init(bar + B_AE + b, KV_STATIONARY ? 2 : 1);  // released by the store issuers
      ptx::mbar_init(bar + B_S + b, 1);
      ptx::mbar_init(bar + B_P + b, 128);
      ptx::mbar_init(bar + B_OF + b, 1);
      ptx::mbar_init(bar + B_OE + b, kCompute);
    }
    for (int s = 0; s < kStages; ++s) {
      ptx::mbar_init(bar + B_B + s, 1);
      ptx::mbar_init(bar + B_E + s, 1);
    }
    ptx::fence_barrier_init();
  }
  for (int i = threadIdx.x; i < kStages * 256; i += kThreads) vec[i] = 0.f;  // unloaded columns read 0
  ptx::fence_proxy_async();  // before TMA writes the same smem
  if (pl.rows_kv < 128) {  // rows no TMA box writes must be finite (zero)
    const int nz = (128 - pl.rows_kv) * S::kRowBytes / 16;
    for (int i = threadIdx.x; i < 2 * kStages * nz; i += kThreads) {
      const int buf = i / nz, off = i % nz;
      uint4* base = reinterpret_cast<uint4*>(smem + S::kB0 + buf * S::kTile + pl.rows_kv * S::kRowBytes);
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
    const uint32_t bytes = 2 * pl.rows_kv * S::kRowBytes + (KV_STATIONARY ? 2 * pl.rows_kv * 4 : 0);
    uint32_t kv_it = 0, ti = 0;
    int tr = 0;
    (void)tr;
    for (unsigned tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      TileCtx<RANK> t;
      if (!t.init(g, pl, tile, /*inverse=*/KV_STATIONARY)) continue;
      const int ab = ti & 1;
      if (ti >= 2) ptx::mbar_wait(bar + B_AE + ab, ((ti >> 1) - 1) & 1);
      if (NA_BWD_TRACE_ON) NA_TRACE_EV(0, tr, 1);
      uint8_t* a0 = smem + S::kA + (2 * ab) * S::kTile;
      uint8_t* a1 = a0 + S::kTile;
      ptx::mbar_expect_tx_w(bar + B_AF + ab, 2 * 128 * S::kRowBytes);
      for (int i = 0; i < pl.q_issues; ++i) {
        t.template load_box<RANK>(&map_a0, a0 + i * pl.q_box_x * S::kRowBytes, bar + B_AF + ab,
                                  t.q_origin, i * pl.q_box_x, g);
        t.template load_box<RANK>(&map_a1, a1 + i * pl.q_box_x * S::kRowBytes, bar + B_AF + ab,
                                  t.q_origin, i * pl.q_box_x, g);
      }
      for (int j = 0; j < t.nchunks; ++j, ++kv_it) {
        const int s = kv_it % kStages;
        if (kv_it >= kStages) ptx::mbar_wait(bar + B_E + s, ((kv_it / kStages) - 1) & 1);
        if (NA_BWD_TRACE_ON) NA_TRACE_EV(0, tr, 2);
        int org[3];
        t.chunk_origin(pl, j, org);
        ptx::mbar_expect_tx_w(bar + B_B + s, bytes);
        for (int i = 0; i < pl.kv_issues; ++i) {
          t.template load_box<RANK>(&map_b0, smem + S::kB0 + s * S::kTile + i * pl.kv_box_x * S::kRowBytes,
                                    bar + B_B + s, org, i * pl.kv_box_x, g);
          t.template load_box<RANK>(&map_b1, smem + S::kB1 + s * S::kTile + i * pl.kv_box_x * S::kRowBytes,
                                    bar + B_B + s, org, i * pl.kv_box_x, g);
        }
        if constexpr (KV_STATIONARY) t.template load_rv<RANK>(&maps.rv, vec + s * 256, bar + B_B + s, org, g);
      }
      ++ti;
    }
  } else if (warp == kMmaWarp) {
    // ===================== MMA issuer (whole warp, one lane issues) =====================
    constexpr uint32_t kSw = D == 64 ? 2u : 4u;
    constexpr uint32_t kSbo = 8 * S::kRowBytes;
    const int n1 = pl.n_kv - 64;
    const uint32_t idesc_s0 = ptx::make_idesc(128, ns == 2 ? 64 : pl.n_kv, BF16, false);
    const uint32_t idesc_s1 = ptx::make_idesc(128, ns == 2 ? n1 : 16, BF16, false);
    constexpr uint32_t idesc_o = ptx::make_idesc(128, D, BF16, true);
    int tr = 0;
    (void)tr;
    // Issue cursor: the S/dP MMAs of sub-chunk (tile, u) run two sub-chunks
    // ahead of the OUT MMAs, ACROSS tile boundaries, so the next tile's first
    // sub-chunks are computed while this tile's last ones are consumed.
    TileCtx<RANK> ct;
    unsigned ctile = seek_tile<RANK, KV_STATIONARY>(g, pl, blockIdx.x, num_tiles, ct);
    uint32_t c_ti = 0, c_kv = 0, c_ub = 0;
    int c_u = 0;
    auto issue_next = [&]() {
      if (ctile >= num_tiles) return;
      const int ab = c_ti & 1;
      if (c_u == 0) {
        ptx::mbar_wait(bar + B_AF + ab, (c_ti >> 1) & 1);
        if (NA_BWD_TRACE_ON) NA_TRACE_EV(1, tr, 14);
        ptx::tc_fence_after();
      }
      const uint32_t a0 = ptx::smem_u32(smem + S::kA + (2 * ab) * S::kTile);
      const uint32_t a1 = a0 + S::kTile;
      const uint32_t kv = c_kv + c_u / ns, gu = c_ub + c_u;
      const int h = c_u % ns, s = kv % kStages;
      if (h == 0) {
        ptx::mbar_wait(bar + B_B + s, (kv / kStages) & 1);
        ptx::tc_fence_after();
      }
      const uint32_t off = h * 64 * S::kRowBytes;
      const uint32_t b0 = ptx::smem_u32(smem + S::kB0 + s * S::kTile) + off;
      const uint32_t b1 = ptx::smem_u32(smem + S::kB1 + s * S::kTile) + off;
      const uint32_t id = h ? idesc_s1 : idesc_s0;
      const uint32_t buf = (gu & 1) * 64;
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
        // KV-stationary: S^T = K Q^T, dP^T = V dO^T.  Q-stationary: S = Q K^T, dP = dO V^T.
        ptx::mma_ss_w(tmem + kColS + buf, ptx::make_sdesc(a0 + kk * 32, 16, kSbo, kSw),
                      ptx::make_sdesc(b0 + kk * 32, 16, kSbo, kSw), id, kk > 0);
        ptx::mma_ss_w(tmem + kColP + buf, ptx::make_sdesc(a1 + kk * 32, 16, kSbo, kSw),
                      ptx::make_sdesc(b1 + kk * 32, 16, kSbo, kSw), id, kk > 0);
      }
      ptx::mma_commit_w(bar + B_S + (gu & 1));
      if (++c_u == ct.nchunks * ns) {
        c_kv += ct.nchunks;
        c_ub += ct.nchunks * ns;
        ++c_ti;
        c_u = 0;
        ctile = seek_tile<RANK, KV_STATIONARY>(g, pl, ctile + gridDim.x, num_tiles, ct);
      }
    };
    issue_next();
    issue_next();
    uint32_t kv_base = 0, ub = 0, ti = 0;
    TileCtx<RANK> t;
    for (unsigned tile = seek_tile<RANK, KV_STATIONARY>(g, pl, blockIdx.x, num_tiles, t); tile < num_tiles;
         tile = seek_tile<RANK, KV_STATIONARY>(g, pl, tile + gridDim.x, num_tiles, t)) {
      const int nsub = t.nchunks * ns;
      const int ob = ti & 1;
      const uint32_t out = kColOut + ob * 128;
      if (ti >= 2) ptx::mbar_wait(bar + B_OE + ob, ((ti >> 1) - 1) & 1);  // outputs drained
      if (NA_BWD_TRACE_ON) NA_TRACE_EV(1, tr, 15);
      for (int u = 0; u < nsub; ++u) {
        const uint32_t kv = kv_base + u / ns, gu = ub + u;
        const int h = u % ns, s = kv % kStages;
        const int width = h ? n1 : (ns == 2 ? 64 : pl.n_kv);
        const uint32_t off = h * 64 * S::kRowBytes;
        const uint32_t b0 = ptx::smem_u32(smem + S::kB0 + s * S::kTile) + off;
        const uint32_t b1 = ptx::smem_u32(smem + S::kB1 + s * S::kTile) + off;
        const uint32_t buf = (gu & 1) * 64;
        ptx::mbar_wait(bar + B_P + (gu & 1), (gu >> 1) & 1);
        if (NA_BWD_TRACE_ON) NA_TRACE_EV(1, tr, 11);
        ptx::tc_fence_after();
        for (int kk = 0; kk < width / 16; ++kk) {
          const uint32_t boff = kk * 16 * S::kRowBytes;
          const uint32_t acc = (u > 0 || kk > 0) ? 1u : 0u;
          if constexpr (KV_STATIONARY) {
            // dV += P^T dO ; dK += dS^T Q   (B operands MN-major)
            ptx::mma_ts_w(tmem + out + D, tmem + kColS + buf + kk * 8,
                          ptx::make_sdesc(b1 + boff, 128 * S::kRowBytes, kSbo, kSw), idesc_o, acc);
            ptx::mma_ts_w(tmem + out, tmem + kColP + buf + kk * 8,
                          ptx::make_sdesc(b0 + boff, 128 * S::kRowBytes, kSbo, kSw), idesc_o, acc);
          } else {
            // dQ += dS K
            ptx::mma_ts_w(tmem + out, tmem + kColS + buf + kk * 8,
                          ptx::make_sdesc(b0 + boff, 128 * S::kRowBytes, kSbo, kSw), idesc_o, acc);
          }
        }
        if (h == ns - 1) ptx::mma_commit_w(bar + B_E + s);
        // The tile's outputs are committed BEFORE the cursor may block on the
        // stationary tiles of tile ti+2, which need this tile's epilogue.
        if (u == nsub - 1) ptx::mma_commit_w(bar + B_OF + ob);
        if (NA_BWD_TRACE_ON) NA_TRACE_EV(1, tr, 12);
        issue_next();
      }
      kv_base += t.nchunks;
      ub += nsub;
      ++ti;
    }
  } else {
    // ===================== compute warpgroups (2 x 128 threads) =====================
    const int grp = warp >> 2;           // processes sub-chunks with gu % 2 == grp
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const int gtid = (warp & 3) * 32 + lane;  // 0..127 within the group
    const uint32_t trow = tmem + ((uint32_t)(quarter * 32) << 16);
    const float sl2 = g.scale_log2;
    const bool issuer = KV_STATIONARY ? (gtid == 0) : (threadIdx.x == 0);  // TMA store issuer
    uint32_t ub = 0, ti = 0, it = 0;
    int tr = 0;
    (void)tr;
    const bool tracer = NA_BWD_TRACE_ON && lane == 0 && (warp == 0 || warp == 4);
    // Row (query) values (-LSE * log2(e), D) of a Q-stationary tile, from the
    // row-vector layout written by the preprocess kernel.
    auto row_vals = [&](const TileCtx<RANK>& t, const RowCtx<RANK>& r, float& nl2, float& d) {
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
    // ---- epilogue of a finished tile ----
    // Runs after this group's FIRST sub-chunk of the next tile (its P is
    // already with the tensor core), so the MMAs never wait for it.  Every MMA
    // of the tile is complete once its outputs are final (B_OF), so the tile's
    // stationary smem tiles are dead: stage the outputs there in the TMA box
    // layout (same swizzle) and write them with TMA stores (rows past a ragged
    // class end are clipped by the hardware).  The buffers return to the
    // producer (B_AE) once the stores have read them (release_store).
    // KV-stationary: group 0 stages dK (x scale) in the K tile, group 1 dV in
    // the V tile.  Q-stationary: the groups split dQ's columns in the Q tile.
    int store_ab = -1;  // issuer: stationary buffer whose store still reads smem
    auto release_store = [&]() {
      if (store_ab >= 0) {
        ptx::bulk_wait_read<0>();
        ptx::mbar_arrive(bar + B_AE + store_ab);  // stationary tiles reusable
        store_ab = -1;
      }
    };
    auto epilogue = [&](const TileCtx<RANK>& t, uint32_t tix) {
      const int ob = tix & 1, ab = tix & 1;
      ptx::mbar_wait(bar + B_OF + ob, (tix >> 1) & 1);
      if (tracer) NA_TRACE_EV(2 + grp, tr, 24);
      ptx::tc_fence_after();
      uint8_t* stage = smem + S::kA + (2 * ab + (KV_STATIONARY ? grp : 0)) * S::kTile;
      constexpr int kCols = KV_STATIONARY ? D : D / 2;
      const int col0 = KV_STATIONARY ? 0 : grp * (D / 2);  // first column this group writes
      const uint32_t src = kColOut + ob * 128 + (KV_STATIONARY ? grp * D : grp * (D / 2));
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
        uint32_t pk[8];
#pragma unroll
        for (int c = 0; c < 16; c += 2)
          pk[c >> 1] = pack2<BF16>(__uint_as_float(ov[c]) * mul, __uint_as_float(ov[c + 1]) * mul);
        const int chunk = (col0 + c0) / 8;
        *reinterpret_cast<uint4*>(stage + ptx::swz_off(row, chunk, S::kRowBytes)) =
            make_uint4(pk[0], pk[1], pk[2], pk[3]);
        *reinterpret_cast<uint4*>(stage + ptx::swz_off(row, chunk + 1, S::kRowBytes)) =
            make_uint4(pk[4], pk[5], pk[6], pk[7]);
      }
      ptx::tc_fence_before();
      ptx::mbar_arrive(bar + B_OE + ob);
      ptx::fence_proxy_async();  // staged tile visible to the TMA engine
      if (tracer) NA_TRACE_EV(2 + grp, tr, 25);
      if constexpr (KV_STATIONARY) ptx::named_bar_sync(3 + grp, 128);
      else ptx::named_bar_sync(3, kCompute);
      if (tracer) NA_TRACE_EV(2 + grp, tr, 26);
      if (issuer) {
        const CUtensorMap* om = (KV_STATIONARY && grp) ? &map_out1 : &map_out0;
        for (int i = 0; i < pl.q_issues; ++i)
          t.template store_box<RANK>(om, stage + i * pl.q_box_x * S::kRowBytes, i * pl.q_box_x, g);
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
    if constexpr (!KV_STATIONARY) {
      if (tile < num_tiles) row_vals(t, r, row_nl2, row_d);
    }
    uint32_t kv_base = 0;
    while (tile < num_tiles) {
      const int nsub = t.nchunks * ns;
      const int u_first = (int)((grp - ub) & 1u);
      // Next tile: found during this group's last sub-chunk of the tile (so a
      // Q-stationary tile's row values load while that sub-chunk computes).
      TileCtx<RANK> tn;
      RowCtx<RANK> rn;
      unsigned tile_n = num_tiles;
      bool tn_known = false;
      float nrow_nl2 = 0.f, nrow_d = 0.f;
      uint32_t mw[4] = {0u, 0u, 0u, 0u};
      for (int u = u_first; u < nsub; u += 2, ++it) {
        if (issuer && u != u_first) release_store();  // previous tile's store has had a sub-chunk to read
        const uint32_t gu = ub + u;
        const int j = u / ns, h = u % ns;
        int org[3];
        t.chunk_origin(pl, j, org);
        r.chunk_mask(pl, org, mw);
        const uint32_t w0 = h ? mw[2] : mw[0], w1 = h ? mw[3] : mw[1];
        // Partner (query) values of the chunk, TMA-loaded with it:
        // [-LSE*log2(e) x rows_kv | D x rows_kv]; this sub-chunk's 64 columns.
        const uint32_t kv = kv_base + j;
        const float* cl = vec + (kv % kStages) * 256 + h * 64;
        const float* cd = cl + pl.rows_kv;
        if (u + 2 >= nsub) {
          tile_n = seek_tile<RANK, KV_STATIONARY>(g, pl, tile + gridDim.x, num_tiles, tn);
          tn_known = true;
          if (tile_n < num_tiles) {
            rn.init(g, pl, tn, row, /*inverse=*/KV_STATIONARY);
            if constexpr (!KV_STATIONARY) row_vals(tn, rn, nrow_nl2, nrow_d);
          }
        }
        const uint32_t buf = (gu & 1) * 64;
        if (tracer) NA_TRACE_EV(2 + grp, tr, 19);
        ptx::mbar_wait(bar + B_S + (gu & 1), (gu >> 1) & 1);
        if constexpr (KV_STATIONARY) {
          // The chunk's stage is still held (its B_E needs this P), so its
          // phase is current: the row-vector bytes are visible after this.
          ptx::mbar_wait(bar + B_B + (kv % kStages), (kv / kStages) & 1);
        }
        if (tracer) NA_TRACE_EV(2 + grp, tr, 20);
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
          for (int c = 0; c < 32; c += 4) {
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
              x0.x = (w >> c) & 1u ? x0.x : -INFINITY;
              x0.y = (w >> (c + 1)) & 1u ? x0.y : -INFINITY;
              x1.x = (w >> (c + 2)) & 1u ? x1.x : -INFINITY;
              x1.y = (w >> (c + 3)) & 1u ? x1.y : -INFINITY;
            }
            const float2 p0 = make_float2(ptx::ex2(x0.x), ptx::ex2(x0.y));  // MUFU
            const float2 p1 = use_poly(c) ? exp2_poly2(x1)                   // FMA pipe
                                          : make_float2(ptx::ex2(x1.x), ptx::ex2(x1.y));
            const float2 ds0 = __fmul2_rn(p0, __fadd2_rn(make_float2(__uint_as_float(pv[c]),
                                                                     __uint_as_float(pv[c + 1])),
                                                         make_float2(-dd4.x, -dd4.y)));
            const float2 ds1 = __fmul2_rn(p1, __fadd2_rn(make_float2(__uint_as_float(pv[c + 2]),
                                                                     __uint_as_float(pv[c + 3])),
                                                         make_float2(-dd4.z, -dd4.w)));
            pk_p[16 * gq + (c >> 1)] = pack2<BF16>(p0.x, p0.y);
            pk_p[16 * gq + (c >> 1) + 1] = pack2<BF16>(p1.x, p1.y);
            pk_s[16 * gq + (c >> 1)] = pack2<BF16>(ds0.x, ds0.y);
            pk_s[16 * gq + (c >> 1) + 1] = pack2<BF16>(ds1.x, ds1.y);
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
        ptx::mbar_arrive(bar + B_P + (gu & 1));
        if (tracer) NA_TRACE_EV(2 + grp, tr, 21);
        if (pend) {  // previous tile's outputs, now that the tensor core has this sub-chunk
          epilogue(tp, ti - 1);
          pend = false;
        }
      }
      if (tracer) NA_TRACE_EV(2 + grp, tr, 22);
      if (pend) {  // this group had no sub-chunk in the tile
        epilogue(tp, ti - 1);
        pend = false;
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
          if constexpr (!KV_STATIONARY) row_vals(tn, rn, nrow_nl2, nrow_d);
        }
      }
      tile = tile_n;
      t = tn;
      r = rn;
      row_nl2 = nrow_nl2;
      row_d = nrow_d;
      if (tracer) NA_TRACE_EV(2 + grp, tr, 23);
    }
    if (pend) epilogue(tp, ti - 1);
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
template <int RANK, int D, bool BF16>
__global__ void __launch_bounds__(kThreads, 1)
    fna_dkdv_tc(const __grid_constant__ BwdMaps maps, Geom g, TcPlan pl, const float* __restrict__ rv,
                unsigned num_tiles) {
  bwd_body<RANK, D, BF16, true>(maps, g, pl, rv, num_tiles);
}

// dQ: query-stationary over the forward halo.
template <int RANK, int D, bool BF16>
__global__ void __launch_bounds__(kThreads, 1)
    fna_dq_tc(const __grid_constant__ BwdMaps maps, Geom g, TcPlan pl, const float* __restrict__ rv,
              unsigned num_tiles) {
  bwd_body<RANK, D, BF16, false>(maps, g, pl, rv, num_tiles);
}

template <int RANK, int D, bool BF16>
cudaError_t launch_both(const Geom& g, const TcPlan& pl, const BwdMaps& mkv, const BwdMaps& mq,
                        const float* rv, cudaStream_t st) {
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
  const long long tiles = (long long)g.BH * pl.nres * pl.tiles;
  if (tiles > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
  const unsigned grid = (unsigned)(tiles < num_sms() ? tiles : num_sms());
  prof_begin(KID_DKDV_TC, st);
  kdkdv<<<grid, kThreads, smem, st>>>(mkv, g, pl, rv, (unsigned)tiles);
  prof_end(st);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  prof_begin(KID_DQ_TC, st);
  kdq<<<grid, kThreads, smem, st>>>(mq, g, pl, rv, (unsigned)tiles);
  prof_end(st);
  return cudaGetLastError();
}

template <int RANK>
cudaError_t by_type(int dtype, const Geom& g, const TcPlan& pl, const BwdMaps& mkv, const BwdMaps& mq,
                    const float* rv, cudaStream_t st) {
  const bool bf = dtype == 2;
  if (g.D == 64)
    return bf ? launch_both<RANK, 64, true>(g, pl, mkv, mq, rv, st)
              : launch_both<RANK, 64, false>(g, pl, mkv, mq, rv, st);
  return bf ? launch_both<RANK, 32, true>(g, pl, mkv, mq, rv, st)
            : launch_both<RANK, 32, false>(g, pl, mkv, mq, rv, st);
}

}  // namespace

cudaError_t tc_bwd(int dtype, const Geom& g, const void* q, const void* k, const void* v,
                   const void* o, const void* d_o, const float* lse, void* dq, void* dk, void* dv,
                   float* Dvec, cudaStream_t st, int* launches) {
  const char* why;
  if (!tc_supported(dtype, g, &why)) return cudaErrorNotSupported;
  cudaError_t e = bwd_preprocess(dtype, g, o, d_o, lse, Dvec, st);  // row-vector layout
  if (e != cudaSuccess) return e;
  TcPlan pl = make_plan(g, 128);
  // dK/dV kernel: stationary K, V tiles; streamed Q, dO chunks; outputs dK, dV.
  // dQ kernel: stationary Q, dO tiles; streamed K, V chunks; output dQ.
  BwdMaps mkv, mq;
  const void* tile_src[2][2] = {{k, v}, {q, d_o}};
  const void* chunk_src[2][2] = {{q, d_o}, {k, v}};
  BwdMaps* mm[2] = {&mkv, &mq};
  for (int w = 0; w < 2; ++w) {
    if ((e = make_map(&mm[w]->a0, dtype, g, tile_src[w][0], pl.tq, pl.q_box_x)) != cudaSuccess) return e;
    if ((e = make_map(&mm[w]->a1, dtype, g, tile_src[w][1], pl.tq, pl.q_box_x)) != cudaSuccess) return e;
    if ((e = make_map(&mm[w]->b0, dtype, g, chunk_src[w][0], pl.ckv, pl.kv_box_x)) != cudaSuccess) return e;
    if ((e = make_map(&mm[w]->b1, dtype, g, chunk_src[w][1], pl.ckv, pl.kv_box_x)) != cudaSuccess) return e;
  }
  if ((e = make_map(&mkv.out0, dtype, g, dk, pl.tq, pl.q_box_x)) != cudaSuccess) return e;
  if ((e = make_map(&mkv.out1, dtype, g, dv, pl.tq, pl.q_box_x)) != cudaSuccess) return e;
  if ((e = make_map(&mq.out0, dtype, g, dq, pl.tq, pl.q_box_x)) != cudaSuccess) return e;
  mq.out1 = mq.out0;
  if ((e = make_map_rv(&mkv.rv, g, Dvec, pl.ckv)) != cudaSuccess) return e;
  mq.rv = mkv.rv;
  *launches = 3;
  switch (g.rank) {
    case 1: return by_type<1>(dtype, g, pl, mkv, mq, Dvec, st);
    case 2: return by_type<2>(dtype, g, pl, mkv, mq, Dvec, st);
    default: return by_type<3>(dtype, g, pl, mkv, mq, Dvec, st);
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
