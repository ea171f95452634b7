"""bf16 error/time study: the plain vs the error-compensated (PRECISE) kernel
variants (R13) on the same inputs.

For each case and output: max |gpu - exact|, the excess over the R14 bound,
max |exact|, and the error BEYOND the correct rounding of the exact value
(max of |gpu - exact| - |bf16(exact) - exact|), i.e. what the kernel's own
arithmetic adds.  Then fwd / fwd+bwd ms of config D_d2 in both variants.

    NA_BF16_PRECISE_STUDY is read by libna (study builds only).
    python tools/bf16_study.py      # on a GPU box
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import na_synth  # noqa: E402
import oracle  # noqa: E402
import paper_2403_04690_b200 as na  # noqa: E402
import paper_2403_04690_b200.na as nab  # noqa: E402

if "--lib" in sys.argv:  # a study build of libna (e.g. NA_DEFINES variants)
    nab.LIB_PATH = os.path.abspath(sys.argv[sys.argv.index("--lib") + 1])
from na_tol import excess  # noqa: E402

CASES = [
    ([10, 20, 24], [3, 5, 5], [1, 2, 1], [0, 0, 0], 16),
    ([10, 20, 24], [3, 5, 5], [1, 2, 1], [0, 0, 0], 64),
    ([37, 20], [7, 5], [1, 2], [0, 0], 64),
    ([30, 44], [9, 13], [3, 2], [0, 1], 32),
    ([300], [255], [1], [0], 64),
    ([300], [33], [3], [0], 64),
    ([40, 40], [9, 9], [1, 1], [0, 0], 64),
    ([48, 48], [13, 13], [2, 2], [0, 0], 64),
    ([12, 24, 24], [5, 5, 5], [1, 1, 1], [0, 0, 0], 64),
    ([16, 32, 32], [7, 7, 7], [1, 1, 1], [1, 0, 0], 64),
]


def rnd_err(ref):
    r = torch.from_numpy(np.asarray(ref, np.float64))
    return (r.to(torch.bfloat16).double() - r).abs().numpy()


def run(cfg, q, k, v, do):
    kw = dict(kernel_size=list(cfg.kernel_size), dilation=list(cfg.dilation),
              is_causal=[bool(c) for c in cfg.is_causal])
    qd, kd, vd, dod = (t.cuda() for t in (q, k, v, do))
    o, lse = na.na_fwd(qd, kd, vd, **kw)
    dq, dk, dv = na.na_bwd(qd, kd, vd, o, dod, lse, **kw)
    torch.cuda.synchronize()
    return [t.double().cpu().numpy() for t in (o, dq, dk, dv)]


def study_case(ext, ker, dil, cau, D):
    cfg = na_synth.small_config(ext, ker, dil, cau, head_dim=D, batch=1, heads=2, dtype=torch.bfloat16)
    q, k, v, do = na_synth.make_inputs(cfg, salt=7)
    op = oracle.make_problem(1, 2, list(ext), D, list(ker), list(dil), list(cau))
    ro, _ = oracle.fwd(op, q, k, v)
    rdq, rdk, rdv = oracle.bwd(op, q, k, v, do, stored_o=False)
    refs = [np.asarray(x, np.float64).reshape(1, 2, -1, D) for x in (ro, rdq, rdk, rdv)]
    print(f"case {ext} k{ker} d{dil} c{cau} D{D}")
    for mode in ("0", "1"):
        os.environ["NA_BF16_PRECISE_STUDY"] = mode
        got = run(cfg, q, k, v, do)
        row = []
        for name, g, r in zip(("O", "dQ", "dK", "dV"), got, refs):
            g = g.reshape(r.shape)
            e = np.abs(g - r)
            extra = float((e - rnd_err(r)).max())
            row.append(f"{name} err {e.max():.4f} exc {excess(g, r, torch.bfloat16):+.4f} "
                       f"|ref| {np.abs(r).max():.2f} beyond-rnd {extra:.4f}")
        print(f"  {'precise' if mode == '1' else 'plain  '}: " + " | ".join(row))


def time_config(name, reps=20):
    cfg = na_synth.CONFIGS[name]
    q, k, v, do = na_synth.make_inputs(cfg, device="cuda")
    kw = dict(kernel_size=list(cfg.kernel_size), dilation=list(cfg.dilation),
              is_causal=[bool(c) for c in cfg.is_causal])
    for mode in ("0", "1"):
        os.environ["NA_BF16_PRECISE_STUDY"] = mode
        for _ in range(3):
            o, lse = na.na_fwd(q, k, v, **kw)
            na.na_bwd(q, k, v, o, do, lse, **kw)
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        tf = tb = 0.0
        for _ in range(reps):
            e[0].record()
            o, lse = na.na_fwd(q, k, v, **kw)
            e[1].record()
            na.na_bwd(q, k, v, o, do, lse, **kw)
            e[2].record()
            torch.cuda.synchronize()
            tf += e[0].elapsed_time(e[1])
            tb += e[1].elapsed_time(e[2])
        print(f"{name} {'precise' if mode == '1' else 'plain  '}: fwd {tf / reps:.4f} ms  bwd {tb / reps:.4f} ms")


if __name__ == "__main__":
    for c in CASES:
        study_case(*c)
    time_config("D_d2")
