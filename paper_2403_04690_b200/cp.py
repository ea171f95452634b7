"""Context (spatial) parallelism for fused neighborhood attention -- SURVEY.md
8(f) rank 3, the paper's stated future work.

The token space is split along the outermost spatial axis (axis 0) into G
contiguous slabs, one per rank: rank g OWNS rows [a_g, b_g) = [g*L/G,
(g+1)*L/G).  Neighborhood attention is local, so a rank needs only a halo of
neighbouring rows, exchanged point-to-point (NCCL send/recv over NVLink; gloo
in the CPU tests):

  * slab_g = [max(0, a_g - h), min(L, b_g + h)) with h = k_0 * dilation_0.
    Every query whose window reaches an owned key lies within (k_0/2)*dil
    (causal: (k_0-1)*dil) of it, and that query's own window lies within the
    same distance again, so with h = k_0*dil:
      - an owned query's window is inside the slab, and the slab problem's
        clamping (window shifted inward at the borders) only
        triggers where the slab reaches the global border -- the windows are
        the global ones, in every residue class (a slab is a translation of
        the token grid, so each class of the slab is a translated global
        class);
      - a query of the inverse halo of an owned key also has its true window
        (its LSE, O and D_x are exact on the slab), and a query near the
        slab edge, whose window the slab clamps inward, reaches at most
        (k_0-1)*dil < h into the slab: it never touches an owned key.
  * forward: exchange the Q, K, V halo rows, run the fused kernel on the slab,
    keep the owned rows of O and LSE (and the slab O/LSE for the backward).
  * backward: exchange the dO halo rows, run the fused backward on the slab
    (with the slab's own forward O/LSE), keep the owned rows of dQ, dK, dV.
The halo rows are recomputed on each side (compute overhead 2h / (b-a));
nothing is reduced across ranks.  No NA arithmetic lives here: the
per-slab compute is a pluggable pair of functions (libna's na_fwd / na_bwd
in the product; the tests may plug in anything with the same signature).
"""
from __future__ import annotations

from dataclasses import dataclass

import torch


@dataclass(frozen=True)
class Split:
    """Owned range and slab (halo'd range) of every rank along axis 0."""
    L: int
    world: int
    halo: int

    def own(self, g: int) -> tuple:
        return (g * self.L // self.world, (g + 1) * self.L // self.world)

    def slab(self, g: int) -> tuple:
        a, b = self.own(g)
        return (max(0, a - self.halo), min(self.L, b + self.halo))


def make_split(extent, kernel_size, dilation, world: int) -> Split:
    """Split axis 0 of `extent` over `world` ranks with halo k_0 * dilation_0."""
    k0 = kernel_size[0] if isinstance(kernel_size, (list, tuple)) else kernel_size
    d0 = (dilation[0] if isinstance(dilation, (list, tuple)) else dilation) or 1
    L = int(extent[0])
    if L < world:
        raise ValueError(f"axis 0 has {L} rows for {world} ranks")
    return Split(L, world, int(k0) * int(d0))


def slab_of(full: torch.Tensor, split: Split, g: int) -> torch.Tensor:
    """Rows slab(g) of a full [B, H, L0, ...] tensor (single-process emulation
    of what exchange_halo assembles on rank g; tests and drivers)."""
    s, e = split.slab(g)
    return full[:, :, s:e].contiguous()


def exchange_halo(t_own: torch.Tensor, split: Split, rank: int, group=None) -> torch.Tensor:
    """Slab of a tensor sharded by rows of spatial axis 0.

    t_own: [B, H, b-a, ...] (this rank's owned rows).  Returns [B, H, e-s, ...]
    for slab (s, e): owned rows copied, every other row received from its
    owner (batched point-to-point send/recv; one message per (src, dst) pair
    whose ranges overlap)."""
    import torch.distributed as dist
    a, b = split.own(rank)
    s, e = split.slab(rank)
    out = torch.empty((*t_own.shape[:2], e - s, *t_own.shape[3:]), dtype=t_own.dtype, device=t_own.device)
    out[:, :, a - s:b - s].copy_(t_own)
    ops, recvs = [], []
    for g in range(split.world):
        if g == rank:
            continue
        # rows rank needs from g
        ga, gb = split.own(g)
        lo, hi = max(ga, s), min(gb, e)
        if lo < hi:
            buf = torch.empty((*t_own.shape[:2], hi - lo, *t_own.shape[3:]), dtype=t_own.dtype,
                              device=t_own.device)
            ops.append(dist.P2POp(dist.irecv, buf, g, group))
            recvs.append((lo - s, buf))
        # rows g needs from rank
        gs, ge = split.slab(g)
        lo, hi = max(a, gs), min(b, ge)
        if lo < hi:
            ops.append(dist.P2POp(dist.isend, t_own[:, :, lo - a:hi - a].contiguous(), g, group))
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    for off, buf in recvs:
        out[:, :, off:off + buf.shape[2]].copy_(buf)
    return out


class ContextParallel:
    """Forward + backward of fused NA with the token space split along axis 0.

    fwd_fn(q, k, v, **kw) -> (o, lse) and bwd_fn(q, k, v, o, do, lse, **kw) ->
    (dq, dk, dv) compute one slab problem (default: libna's na_fwd / na_bwd).
    kw: kernel_size, dilation, is_causal (global problem parameters; the slab
    is the same problem on a sub-range of axis 0)."""

    def __init__(self, extent, kernel_size, dilation=None, is_causal=None, group=None,
                 fwd_fn=None, bwd_fn=None):
        import torch.distributed as dist
        r = len(extent)
        self.kw = dict(kernel_size=list(kernel_size) if isinstance(kernel_size, (list, tuple))
                       else [kernel_size] * r,
                       dilation=list(dilation) if dilation else [1] * r,
                       is_causal=[bool(c) for c in is_causal] if is_causal else [False] * r)
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.split = make_split(extent, self.kw["kernel_size"], self.kw["dilation"], self.world)
        if fwd_fn is None or bwd_fn is None:
            from . import na as _na
            fwd_fn = fwd_fn or _na.na_fwd
            bwd_fn = bwd_fn or _na.na_bwd
        self.fwd_fn, self.bwd_fn = fwd_fn, bwd_fn

    def own_rows(self, full: torch.Tensor) -> torch.Tensor:
        """This rank's owned rows of a full [B, H, L0, ...] tensor (for drivers and tests)."""
        a, b = self.split.own(self.rank)
        return full[:, :, a:b]

    def _own_of_slab(self, t: torch.Tensor) -> torch.Tensor:
        a, b = self.split.own(self.rank)
        s, _ = self.split.slab(self.rank)
        return t[:, :, a - s:b - s]

    def forward(self, q, k, v):
        """q, k, v: owned rows [B, H, b-a, ..., D].  Returns (o, lse) owned
        rows and a context for backward()."""
        ex = lambda t: exchange_halo(t, self.split, self.rank, self.group)
        qs, ks, vs = ex(q), ex(k), ex(v)
        o, lse = self.fwd_fn(qs, ks, vs, **self.kw)
        ctx = (qs, ks, vs, o, lse)
        return self._own_of_slab(o), self._own_of_slab(lse), ctx

    def backward(self, ctx, do):
        """do: owned rows of dL/dO.  Returns owned rows of (dq, dk, dv)."""
        qs, ks, vs, o, lse = ctx
        dos = exchange_halo(do, self.split, self.rank, self.group)
        dq, dk, dv = self.bwd_fn(qs, ks, vs, o, dos, lse, **self.kw)
        return tuple(self._own_of_slab(t) for t in (dq, dk, dv))
