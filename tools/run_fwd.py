"""Run one config's forward (after warmup) for ncu captures: python tools/run_fwd.py B_d1 [bwd]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import na_synth  # noqa: E402
import paper_2403_04690_b200 as na  # noqa: E402

cfg = na_synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "B_d1"]
q, k, v, do = na_synth.make_inputs(cfg, device="cuda")
kw = dict(kernel_size=list(cfg.kernel_size), dilation=list(cfg.dilation),
          is_causal=[bool(c) for c in cfg.is_causal])
for _ in range(2):
    o, lse = na.na_fwd(q, k, v, **kw)
    if "bwd" in sys.argv:
        na.na_bwd(q, k, v, o, do, lse, **kw)
torch.cuda.synchronize()
print("done")
