// tc_plan.h — tile plan shared by the host launcher and the tcgen05 kernels.
//
// Space-aware tiling (Fig. 3 / Fig. 4): a CTA owns a
// multi-dimensional box of 128 query tokens of ONE residue class (dilation
// = more CTAs) and streams the haloed key/value region of that
// box as multi-dimensional TMA boxes ("KV chunks", <= 128 keys each).
// All extents are in compacted (per-residue-class) coordinates; axis 0 is
// the outermost spatial axis, axis rank-1 the innermost (contiguous) one.
#pragma once
#include <stdint.h>

namespace na {

// Division of n < 2^31 by a runtime constant d >= 1 as a multiply-high and
// shift (round-up method): q = (umulhi(n, mul) + n) >> shift.
struct FastDiv {
  uint32_t d, mul, shift;
};

inline FastDiv make_fastdiv(uint32_t d) {
  uint32_t l = 0;
  while ((1ull << l) < d) ++l;
  const uint64_t mul = (((1ull << l) - d) << 32) / d + 1;
  return FastDiv{d, (uint32_t)mul, l};
}

#ifdef __CUDACC__
__device__ __forceinline__ uint32_t fdiv(uint32_t n, const FastDiv& f) {
  return (__umulhi(n, f.mul) + n) >> f.shift;
}
__device__ __forceinline__ uint32_t fmod_(uint32_t n, uint32_t q, const FastDiv& f) {
  return n - q * f.d;
}
#endif

constexpr int kTopPlans = 4;  // planner candidates kept for measurement (na_tune)
constexpr int kMaxPlans = kTopPlans + 1;  // + the best small-chunk plan (head_dim <= 32)

// Which candidate plan each tensor-core kernel uses.
struct PlanChoice {
  int fwd, dkdv, dq;
};

struct TcPlan {
  int tq[3];       // query tile extent per axis (power of two, product 128; 1 beyond rank)
  int tq_shift[3]; // log2(tq)
  int ckv[3];      // KV chunk box extent per axis (product <= 128)
  int ntile[3];    // tiles per axis over the largest residue class
  int tiles;       // prod(ntile)
  int nres;        // prod(dilation): residue classes per (b, h)
  int rows_kv;     // prod(ckv): keys one chunk loads
  int n_kv;        // rows_kv rounded up to 16 (MMA N of S = Q K^T)
  int q_issues;    // TMA issues per Q tile (rank 1 with large dilation splits x)
  int kv_issues;   // TMA issues per K or V chunk
  int q_box_x;     // compacted x extent per Q issue
  int kv_box_x;    // compacted x extent per KV issue
  FastDiv f_tiles, f_nres, f_dil[3], f_ntile[3], f_ckv[3];
  // Multi-dimensional chunk masks (RowCtx::chunk_mask): a chunk column is
  // (row, lx) with row = the chunk's outer coordinates flattened and lx the
  // innermost one, at bit row * cx + lx.  rep = sum over rows of 2^(row*cx)
  // as two 64-bit halves; rep_sh = 64 - row* * cx for the row straddling
  // bit 64 (0: none).  x-window bits times rep = the window replicated on
  // every row (the copies never overlap, so the product has no carries).
  unsigned long long rep_lo, rep_hi;
  int rep_sh;
  // Rank 3 with several outermost slices per chunk (ckv[0] > 1, so one slice
  // of S = ckv[1] * ckv[2] bits fits 64): rep1 = sum over y of 2^(y*cx)
  // builds one slice's pattern; rep2 = sum over t of 2^(t*S) (two halves and
  // the straddle shift, as above) replicates it over the slices.
  unsigned long long rep1, rep2_lo, rep2_hi;
  int rep2_sh;
};

}  // namespace na
