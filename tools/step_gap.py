"""Why a forward inside the bench step is slower than the isolated per-config
forward (VERDICT r1 "what's weak" 4): time the four config-B forwards
(kernel-only, the library's event hook) in four settings on the same inputs:

  step      : as in bench.py's step (each forward right after the previous
              variant's backward, the first after the 256 MB write flush)
  dirty     : each forward right after a 256 MB zero-fill (L2 full of dirty
              lines to write back), the per_config protocol
  clean     : each forward right after a 256 MB READ pass (L2 holds clean,
              unrelated lines; nothing to write back)
  after_bwd : each forward right after a backward of the same variant

    python tools/step_gap.py      # GPU box
"""
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import na_synth  # noqa: E402
import paper_2403_04690_b200 as na  # noqa: E402

names = ["B_d1", "B_d1_causal", "B_d4", "B_d4_causal"]
cfgs = [na_synth.CONFIGS[n] for n in names]
c = cfgs[0]
q, k, v, do = na_synth.make_inputs(c, device="cuda")
outs = []
for cfg in cfgs:
    o = torch.empty_like(q)
    lse = torch.empty(q.shape[:-1], dtype=torch.float32, device="cuda")
    outs.append((o, lse, [torch.empty_like(q) for _ in range(3)]))
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
sink = torch.empty(1, device="cuda")


def kw(cfg):
    return dict(kernel_size=list(cfg.kernel_size), dilation=list(cfg.dilation),
                is_causal=[bool(x) for x in cfg.is_causal])


def fwd(i):
    o, lse, _ = outs[i]
    na.na_fwd(q, k, v, out=o, lse=lse, **kw(cfgs[i]))


def bwd(i):
    o, lse, g = outs[i]
    na.na_bwd(q, k, v, o, do, lse, dq=g[0], dk=g[1], dv=g[2], **kw(cfgs[i]))


def fwd_times(before, reps=5):
    ts = []
    for _ in range(reps):
        for i in range(4):
            before(i)
            na.profile_enable(True)
            fwd(i)
            rec = na.profile_collect()
            na.profile_enable(False)
            ts.append(sum(t for n, t in rec if n == "fna_fwd_tc"))
            bwd(i)
    return statistics.median(ts)


for i in range(4):
    fwd(i)
    bwd(i)
torch.cuda.synchronize()
res = {
    "step": fwd_times(lambda i: flush.zero_() if i == 0 else None),
    "dirty": fwd_times(lambda i: flush.zero_()),
    "clean": fwd_times(lambda i: sink.copy_(flush.sum().reshape(1))),
    "after_bwd": fwd_times(lambda i: bwd(i)),
}
for kk, vv in res.items():
    print(f"{kk:10s} forward kernel median {vv:.4f} ms")
