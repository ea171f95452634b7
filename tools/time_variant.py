"""A/B timing of one library build (kernel experiments; GPU box).

    python tools/time_variant.py [path/to/libna_variant.so] [config ...]

Loads the given libna build (default: the in-tree libna.so), then for each
config (default: the four bench variants) times forward and backward with
CUDA events over 10 launches after 3 warm-ups, flushing L2 before each, and
prints the per-kernel averages from the library's profiling hook.
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import na_synth  # noqa: E402
import paper_2403_04690_b200.na as nab  # noqa: E402

args = sys.argv[1:]
if args and args[0].endswith(".so"):
    nab.LIB_PATH = os.path.abspath(args.pop(0))
names = args or ["B_d1", "B_d4", "B_d1_causal", "B_d4_causal"]
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
print(f"lib {nab.LIB_PATH}")
for name in names:
    cfg = na_synth.CONFIGS[name]
    q, k, v, do = na_synth.make_inputs(cfg, device="cuda")
    kw = dict(kernel_size=list(cfg.kernel_size), dilation=list(cfg.dilation),
              is_causal=[bool(c) for c in cfg.is_causal])
    o, lse = nab.na_fwd(q, k, v, **kw)
    grads = [torch.empty_like(q) for _ in range(3)]
    for _ in range(3):
        nab.na_bwd(q, k, v, o, do, lse, dq=grads[0], dk=grads[1], dv=grads[2], **kw)
    tf = tb = 0.0
    nab.profile_enable(True)
    for _ in range(10):
        flush.zero_()
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record()
        nab.na_fwd(q, k, v, out=o, lse=lse, **kw)
        e1.record()
        nab.na_bwd(q, k, v, o, do, lse, dq=grads[0], dk=grads[1], dv=grads[2], **kw)
        e2.record()
        torch.cuda.synchronize()
        tf += e0.elapsed_time(e1) / 10
        tb += e1.elapsed_time(e2) / 10
    per = {}
    for kname, ms in nab.profile_collect():
        per.setdefault(kname, []).append(ms)
    nab.profile_enable(False)
    ks = "  ".join(f"{n}={sum(v) / len(v):.3f}" for n, v in sorted(per.items()))
    print(f"{name:12s} fwd {tf:.3f} ms  bwd {tb:.3f} ms  | {ks}")
