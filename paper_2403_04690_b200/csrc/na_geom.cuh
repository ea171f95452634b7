// na_geom.cuh — neighborhood geometry of the product path (host + device).
//
// Per axis a with extent L, kernel k, dilation dil and causal flag c, a token
// coordinate x splits into its residue class r = x % dil and its compacted
// coordinate x' = x / dil inside that class (§3.4: a dilated
// problem is a set of non-dilated problems).  The class has
// Lr = ceil((L - r) / dil) members.  All window arithmetic below is in
// compacted coordinates of one class.
//
//   forward window of query x' (Fig. 2):
//     non-causal: start = clamp(x' - k/2, 0, Lr - k), [start, start + k - 1]
//     causal    : [max(0, x' - k + 1), x']
//   inverse window of key y' = { x' : y' in window(x') } (the IN operator's
//   gather pattern), an interval:
//     non-causal: lo = (y' <= k-1) ? 0 : y' - k/2 ;
//                 hi = (y' >= Lr-k) ? Lr-1 : y' + k/2
//     causal    : [y', min(Lr - 1, y' + k - 1)]
//   Both bounds are monotone non-decreasing in the coordinate, so the halo of
//   a contiguous tile [x0, x1] is [start(x0), end(x1)] and the inverse halo
//   of a key tile [y0, y1] is [lo(y0), hi(y1)] — exact, not a superset.
//
// Independent of oracle/ (which enumerates windows directly); the two are
// compared in tests.
#pragma once
#include <stdint.h>

#ifndef NA_HD
#define NA_HD __host__ __device__ __forceinline__
#endif

namespace na {

NA_HD int class_size(int L, int dil, int r) { return (L - r + dil - 1) / dil; }

NA_HD int win_start(int xc, int Lr, int k, int causal) {
  if (causal) return xc - k + 1 > 0 ? xc - k + 1 : 0;
  int s = xc - k / 2;
  s = s < Lr - k ? s : Lr - k;
  return s > 0 ? s : 0;
}

NA_HD int win_end(int xc, int Lr, int k, int causal) {
  if (causal) return xc;
  return win_start(xc, Lr, k, 0) + k - 1;
}

NA_HD int inv_start(int yc, int Lr, int k, int causal) {
  if (causal) return yc;
  return yc <= k - 1 ? 0 : yc - k / 2;
}

NA_HD int inv_end(int yc, int Lr, int k, int causal) {
  if (causal) return yc + k - 1 < Lr - 1 ? yc + k - 1 : Lr - 1;
  return yc >= Lr - k ? Lr - 1 : yc + k / 2;
}

// Problem geometry handed to every kernel by value.
struct Geom {
  int rank;        // 1..3
  int BH;          // batch * heads
  int N;           // tokens per (b, h)
  int D;           // head dim
  int L[3], k[3], dil[3], causal[3];  // padded with (1, 1, 1, 0) beyond rank
  int tstride[3];  // token stride of each axis in the flat spatial index
  float scale;     // softmax scale
  float scale_log2;  // scale * log2(e)
  // Backward row-vector layout (tensor-core path): per (b,h) and residue
  // class, two planes [-LSE_x * log2(e) | D_x] indexed by compacted
  // coordinates, rv_lc[a] = ceil(L/dil) per axis (innermost padded to a
  // multiple of 4 so every TMA stride is a multiple of 16 bytes).
  int nres;          // residue classes per (b,h) = prod dil
  int rv_lc[3];      // compacted extent per axis (innermost padded)
  int rv_cs[3];      // element stride per compacted axis
  long long rv_plane;  // elements per plane = rv_cs[0] * rv_lc[0]
};

// Element strides of the Q/K/V/O-type tensors (head_dim stride 1): from one
// (b, h) slice to the next, and per spatial axis (0 beyond rank).
// Contiguous [B,H,X...,D]: sBH = N*D, sX[a] = tstride[a]*D.  LSE, the row
// vectors and the workspace are always contiguous.  Kept out of Geom: the
// tensor-core kernels never read strides (their TMA tensor maps carry them),
// and growing their by-value Geom parameter measurably changed their
// register allocation (dK/dV spills, +9-15 %).
struct Layout {
  long long sBH, sX[3];
  int contig;  // 1: the contiguous layout
};

// Element offset of flat token `tok` of slice `bh` in a Q/K/V/O-type tensor
// (the token's coordinate on axis a is (tok / tstride[a]) % L[a]).
NA_HD long long elem_of_token(const Geom& g, const Layout& ly, int bh, int tok) {
  long long off = (long long)bh * ly.sBH;
  for (int a = 0; a < g.rank; ++a) off += (long long)((tok / g.tstride[a]) % g.L[a]) * ly.sX[a];
  return off;
}

// Offset of plane 0 of class `res` of head `bh` in the row-vector layout.
NA_HD long long rv_base(const Geom& g, int bh, int res) {
  return ((long long)bh * g.nres + res) * 2 * g.rv_plane;
}

}  // namespace na
