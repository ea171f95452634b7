"""Timing of head_dim 128 against head_dim 64 at equal work (heads halved),
outside the BASELINE configs (kernel study; GPU box).

    python tools/time_shapes.py

Each pair has the same FLOPs (4 N l D per head) and HBM bytes; fwd / bwd ms
are CUDA-event averages over 10 calls after 3 warm-ups, L2 flushed before
each, plus per-kernel times from the library's profiling hook.
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import na_synth  # noqa: E402
import paper_2403_04690_b200.na as nab  # noqa: E402

_c = na_synth._cfg
PAIRS = [
    (_c("1d_D64", 8, 16, [16384], 64, [255], [1], [0], torch.float16),
     _c("1d_D128", 8, 8, [16384], 128, [255], [1], [0], torch.float16)),
    (_c("2d_D64", 4, 16, [128, 128], 64, [13, 13], [2, 2], [0, 0], torch.float16),
     _c("2d_D128", 4, 8, [128, 128], 128, [13, 13], [2, 2], [0, 0], torch.float16)),
    (_c("3d_D64", 2, 16, [16, 64, 64], 64, [7, 7, 7], [1, 1, 1], [1, 0, 0], torch.float16),
     _c("3d_D128", 2, 8, [16, 64, 64], 128, [7, 7, 7], [1, 1, 1], [1, 0, 0], torch.float16)),
]


def time_cfg(cfg, flush):
    q, k, v, do = na_synth.make_inputs(cfg, device="cuda")
    kw = dict(kernel_size=list(cfg.kernel_size), dilation=list(cfg.dilation),
              is_causal=[bool(c) for c in cfg.is_causal])
    o, lse = nab.na_fwd(q, k, v, **kw)
    g = [torch.empty_like(q) for _ in range(3)]
    for _ in range(3):
        nab.na_bwd(q, k, v, o, do, lse, dq=g[0], dk=g[1], dv=g[2], **kw)
    tf = tb = 0.0
    nab.profile_enable(True)
    for _ in range(10):
        flush.zero_()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record()
        nab.na_fwd(q, k, v, out=o, lse=lse, **kw)
        e[1].record()
        nab.na_bwd(q, k, v, o, do, lse, dq=g[0], dk=g[1], dv=g[2], **kw)
        e[2].record()
        torch.cuda.synchronize()
        tf += e[0].elapsed_time(e[1]) / 10
        tb += e[1].elapsed_time(e[2]) / 10
    per = {}
    for kname, ms in nab.profile_collect():
        per.setdefault(kname, []).append(ms)
    nab.profile_enable(False)
    fl = 4.0 * cfg.batch * cfg.heads * cfg.tokens * cfg.head_dim
    for kk in cfg.kernel_size:
        fl *= kk
    ks = "  ".join(f"{n}={sum(v) / len(v):.3f}" for n, v in sorted(per.items()))
    print(f"{cfg.name:8s} fwd {tf:.3f} ms ({fl / tf / 1e9:.0f} TFLOP/s)  fwd+bwd {tf + tb:.3f} ms "
          f"({3.5 * fl / (tf + tb) / 1e9:.0f} TFLOP/s) | {ks}")


if __name__ == "__main__":
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    for a, b in PAIRS:
        time_cfg(a, flush)
        time_cfg(b, flush)
