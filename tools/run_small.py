"""Tiny fwd+bwd launches of every kernel family (for compute-sanitizer runs)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import na_synth  # noqa: E402
import paper_2403_04690_b200 as na  # noqa: E402

cases = [
    ([300], [33], [2], [1], 64, torch.float16),
    ([20, 27], [7, 5], [2, 1], [0, 0], 32, torch.bfloat16),
    ([6, 10, 12], [3, 5, 5], [1, 1, 2], [1, 0, 0], 64, torch.float16),
    ([300], [33], [2], [1], 64, torch.bfloat16),
    ([20, 27], [7, 5], [2, 1], [0, 0], 64, torch.float16),
    ([6, 10, 12], [3, 5, 5], [1, 1, 2], [1, 0, 0], 32, torch.bfloat16),
    ([50], [7], [1], [0], 16, torch.float32),
]
for ext, ker, dil, cau, d, dt in cases:
    cfg = na_synth.small_config(ext, ker, dil, cau, head_dim=d, dtype=dt)
    q, k, v, do = na_synth.make_inputs(cfg, device="cuda", salt=2)
    kw = dict(kernel_size=ker, dilation=dil, is_causal=[bool(c) for c in cau])
    for impl in (["tc", "simt"] if dt != torch.float32 else ["simt"]):
        o, lse = na.na_fwd(q, k, v, impl=impl, **kw)
        na.na_bwd(q, k, v, o, do, lse, impl=impl, **kw)
torch.cuda.synchronize()
print("ok")
