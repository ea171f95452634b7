"""Per-CTA timeline of the forward kernel from the trace build (libna_trace.so).

    python tools/trace_fwd.py [config]     # on a GPU box

Events (clock64 cycles, relative to the CTA's first event):
  role 0 producer: 1 = K/V stage free, loads issued
  role 1 MMA:      10 = K ready (S issue), 11 = P_u ready, 12 = PV_u issued
  role 2 softmax (warp 2 lane 0): 20 = S_u ready, 21 = P_u written,
                   22 = O ready (epilogue), 23 = O drained
"""
import ctypes
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import na_synth  # noqa: E402
import paper_2403_04690_b200.na as nab  # noqa: E402

nab.LIB_PATH = os.environ.get("NA_TRACE_LIB", os.path.join(ROOT, "paper_2403_04690_b200", "libna_trace.so"))
L = nab.lib()
L.na_debug_set_trace_fwd.argtypes = [ctypes.c_void_p]

name = sys.argv[1] if len(sys.argv) > 1 else "B_d1"
cfg = na_synth.CONFIGS[name]
q, k, v = na_synth.make_inputs(cfg, device="cuda", with_do=False)
kw = dict(kernel_size=list(cfg.kernel_size), dilation=list(cfg.dilation),
          is_causal=[bool(c) for c in cfg.is_causal])
for _ in range(3):
    nab.na_fwd(q, k, v, **kw)
buf = torch.zeros(64 * 4 * 256, dtype=torch.int64, device="cuda")
assert L.na_debug_set_trace_fwd(ctypes.c_void_p(buf.data_ptr())) == 0
torch.cuda.synchronize()
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ev0.record()
nab.na_fwd(q, k, v, **kw)
ev1.record()
torch.cuda.synchronize()
print(f"{name}: forward {ev0.elapsed_time(ev1):.3f} ms")
t = buf.view(64, 4, 256).cpu()
for cta in (0, 1, 37):
    evs = []
    for role in range(4):
        for x in t[cta, role].tolist():
            if x == 0:
                break
            evs.append(((x >> 8), role, x & 0xFF))
    if not evs:
        continue
    t0 = min(e[0] for e in evs)
    evs.sort()
    print(f"--- CTA {cta}: {len(evs)} events, span {evs[-1][0] - t0} cycles")
    line = []
    for c, role, tag in evs[:140]:
        line.append(f"{c - t0:>7}:{tag}")
        if len(line) == 10:
            print("  " + "  ".join(line))
            line = []
    if line:
        print("  " + "  ".join(line))
    # per-event-type mean gaps
    import collections
    by = collections.defaultdict(list)
    for c, role, tag in evs:
        by[tag].append(c)
    for tag, cs in sorted(by.items()):
        if len(cs) > 2:
            d = [b - a for a, b in zip(cs, cs[1:])]
            print(f"   tag {tag:2d}: n={len(cs):3d} mean gap {sum(d) / len(d):8.1f} cycles")
