"""Seeded synthetic inputs shared by the tests, the bench and smoke().

This module holds NO neighborhood-attention arithmetic: it only draws
unit-normal tensors (the north_star's "unit-normal inputs") and the problem
shapes of BASELINE.json's configs.  Both the CUDA path and the oracle consume
what it produces; neither imports the other.

Seeding: every (b, h) slice of tensor t has its own
generator seeded with ``1000 * TENSOR_ID[t] + (b * H + h) + salt``, so a
rank that owns a contiguous range of flattened B*H slices generates exactly
the values a single GPU would, whatever the GPU count.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import torch

TENSOR_ID = {"q": 0, "k": 1, "v": 2, "do": 3}


@dataclass(frozen=True)
class Config:
    name: str
    batch: int
    heads: int
    extent: tuple
    head_dim: int
    kernel_size: tuple
    dilation: tuple
    is_causal: tuple
    dtype: torch.dtype
    note: str = field(default="", compare=False)

    @property
    def rank(self) -> int:
        return len(self.extent)

    @property
    def tokens(self) -> int:
        n = 1
        for e in self.extent:
            n *= e
        return n

    @property
    def window(self) -> int:
        l = 1
        for k in self.kernel_size:
            l *= k
        return l

    def shape(self, bh: int | None = None):
        if bh is None:
            return (self.batch, self.heads, *self.extent, self.head_dim)
        return (bh, *self.extent, self.head_dim)


def _cfg(name, b, h, ext, d, k, dil, causal, dt, note=""):
    return Config(name, b, h, tuple(ext), d, tuple(k), tuple(dil), tuple(causal), dt, note)


# BASELINE.json "configs" (index in brackets), one entry per (dilation, causal) variant.
CONFIGS = {
    # [0] 1-D fp32, the oracle finishes it in seconds
    "A": _cfg("A", 1, 1, [64], 16, [7], [1], [0], torch.float32),
    # [1] 1-D fp16 B=8 H=16 L=16384 D=64 k=255, dilation {1,4} x {causal, non-causal}
    "B_d1": _cfg("B_d1", 8, 16, [16384], 64, [255], [1], [0], torch.float16),
    "B_d1_causal": _cfg("B_d1_causal", 8, 16, [16384], 64, [255], [1], [1], torch.float16),
    "B_d4": _cfg("B_d4", 8, 16, [16384], 64, [255], [4], [0], torch.float16),
    "B_d4_causal": _cfg("B_d4_causal", 8, 16, [16384], 64, [255], [4], [1], torch.float16),
    # [2] 2-D fp16 NAT/DiNAT B=32 H=8 56x56 D=32 k=7x7 dilation {1,8}
    "C_d1": _cfg("C_d1", 32, 8, [56, 56], 32, [7, 7], [1, 1], [0, 0], torch.float16),
    "C_d8": _cfg("C_d8", 32, 8, [56, 56], 32, [7, 7], [8, 8], [0, 0], torch.float16),
    # [3] 2-D bf16 B=4 H=16 128x128 D=64 k=13x13 dilation 2
    "D_d2": _cfg("D_d2", 4, 16, [128, 128], 64, [13, 13], [2, 2], [0, 0], torch.bfloat16),
    # [4] 3-D fp16 B=2 H=16 16x64x64 D=64 k=7x7x7 causal on T
    "E": _cfg("E", 2, 16, [16, 64, 64], 64, [7, 7, 7], [1, 1, 1], [1, 0, 0], torch.float16),
}


def slice_tensor(cfg: Config, name: str, bh0: int, bh1: int, device="cpu", salt: int = 0,
                 dtype: torch.dtype | None = None) -> torch.Tensor:
    """Tensor `name` for flattened slices [bh0, bh1): shape [bh1-bh0, X..., D]."""
    dtype = dtype or cfg.dtype
    per = cfg.tokens * cfg.head_dim
    out = torch.empty((bh1 - bh0, *cfg.extent, cfg.head_dim), dtype=dtype, device=device)
    gen = torch.Generator(device=device)
    for i, bh in enumerate(range(bh0, bh1)):
        gen.manual_seed(1000 * TENSOR_ID[name] + bh + salt)
        x = torch.randn((per,), generator=gen, device=device, dtype=torch.float32)
        out[i].copy_(x.view(*cfg.extent, cfg.head_dim).to(dtype))
    return out


def make_inputs(cfg: Config, device="cpu", bh_range=None, salt: int = 0, with_do: bool = True,
                dtype: torch.dtype | None = None):
    """Q, K, V (and dO) shaped [B, H, X..., D] (or [bh1-bh0, X..., D] when a
    range of flattened slices is requested)."""
    bh0, bh1 = bh_range or (0, cfg.batch * cfg.heads)
    names = ["q", "k", "v"] + (["do"] if with_do else [])
    ts = [slice_tensor(cfg, n, bh0, bh1, device, salt, dtype) for n in names]
    if bh_range is None:
        ts = [t.view(cfg.shape()) for t in ts]
    return ts


def small_config(extent, kernel_size, dilation=None, is_causal=None, head_dim=16, batch=1,
                 heads=2, dtype=torch.float32, name="small") -> Config:
    r = len(extent)
    return _cfg(name, batch, heads, extent, head_dim, kernel_size, dilation or [1] * r,
                is_causal or [0] * r, dtype)
