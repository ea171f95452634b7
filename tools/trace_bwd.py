"""Per-CTA timeline of a backward kernel (dK/dV: arg2=1, dQ: arg2=0) from libna_trace.so.

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
L.na_debug_set_trace_bwd.argtypes = [ctypes.c_void_p, ctypes.c_int]
which = int(sys.argv[2]) if len(sys.argv) > 2 else 1

name = sys.argv[1] if len(sys.argv) > 1 else "B_d1"
cfg = na_synth.CONFIGS[name]
q, k, v, do = na_synth.make_inputs(cfg, device="cuda")
kw = dict(kernel_size=list(cfg.kernel_size), dilation=list(cfg.dilation),
          is_causal=[bool(c) for c in cfg.is_causal])
o, lse = nab.na_fwd(q, k, v, **kw)
for _ in range(3):
    nab.na_bwd(q, k, v, o, do, lse, **kw)
buf = torch.zeros(64 * 4 * 256, dtype=torch.int64, device="cuda")
assert L.na_debug_set_trace_bwd(ctypes.c_void_p(buf.data_ptr()), which) == 0
torch.cuda.synchronize()
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ev0.record()
nab.na_bwd(q, k, v, o, do, lse, **kw)
ev1.record()
torch.cuda.synchronize()
print(f"{name}: backward {ev0.elapsed_time(ev1):.3f} ms (kernel {which})")
t = buf.view(64, 4, 256).cpu()
import collections
for cta in (0, 37):
    print(f"--- CTA {cta}")
    allev = [[((x >> 8), x & 0xFF) for x in t[cta, role].tolist() if x != 0] for role in range(4)]
    t0 = min(e[0][0] for e in allev if e)  # one clock origin for every role of the CTA
    merged = sorted((c, role, tag) for role, e in enumerate(allev) for c, tag in e)
    tmax = merged[0][0] + 60000
    print("  merged (cycle:role.tag): " + "  ".join(f"{c - t0}:{r}.{tag}" for c, r, tag in merged if c < tmax))
    for role in range(4):
        evs = allev[role]
        if not evs:
            continue
        print(f"  role {role}: " + "  ".join(f"{c - t0}:{tag}" for c, tag in evs[:40]))
        by = collections.defaultdict(list)
        for i2 in range(1, len(evs)):
            by[(evs[i2 - 1][1], evs[i2][1])].append(evs[i2][0] - evs[i2 - 1][0])
        print("     mean gaps: " + ", ".join(f"{a}->{b}: {sum(v) / len(v):.0f} (n={len(v)})"
                                            for (a, b), v in sorted(by.items()) if len(v) > 3))
