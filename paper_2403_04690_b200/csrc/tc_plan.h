// tc_plan.h — tile plan shared by the host launcher and the tcgen05 kernels.
//
// Space-aware tiling (Fig. 3 / Fig. 4): a CTA owns a
// multi-dimensional box of 128 query tokens of ONE residue class (dilation
// = more CTAs) and streams the haloed key/value region of that
// box as multi-dimensional TMA boxes ("KV chunks", <= 128 keys each).
// All extents are in compacted (per-residue-class) coordinates; axis 0 is
// the outermost spatial axis, axis rank-1 the innermost (contiguous) one.
#pragma once

namespace na {

struct TcPlan {
  int tq[3];       // query tile extent per axis (product 128; 1 beyond rank)
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
};

}  // namespace na
