"""Ablation of the 16-bit gradient error (VERDICT r1 "what's weak" 1).

For each case: the GPU backward run (a) on the GPU forward's O and (b) on
the oracle's exact O rounded to the dtype; max-abs errors of dQ/dK/dV
against the EXACT oracle gradient and against the stored-O oracle.  If (b)
is much closer to exact than (a), the error comes from the forward's O
(16-bit P in the PV MMA) feeding D_x = <dO_x, O_x>; if not, from the
backward's own 16-bit P / dS operands.

    python tools/err_ablation.py [--dtype bf16|fp16]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import na_synth  # noqa: E402
import oracle  # noqa: E402
import paper_2403_04690_b200 as na  # noqa: E402

CASES = [
    ([6, 10, 13], [3, 5, 7], [1, 1, 1], [1, 0, 0]),
    ([8, 9, 12], [3, 3, 3], [2, 1, 2], [0, 1, 0]),
    ([16, 12, 12], [7, 7, 7], [1, 1, 1], [1, 0, 0]),
    ([12, 16, 16], [5, 3, 3], [1, 1, 1], [1, 0, 0]),
    ([10, 20, 24], [3, 5, 5], [1, 2, 1], [0, 0, 0]),
    ([37, 20], [7, 5], [1, 2], [0, 0]),
    ([23, 41], [3, 9], [2, 1], [1, 0]),
    ([30, 44], [9, 13], [3, 2], [0, 1]),
    ([300], [7], [1], [0]),
    ([300], [64], [2], [1]),
    ([257], [31], [4], [1]),
    ([300], [255], [1], [0]),
    ([128, 128], [13, 13], [2, 2], [0, 0]),
]


def mx(a, b):
    return float(np.abs(np.asarray(a, np.float64) - np.asarray(b, np.float64)).max())


BITS = {torch.bfloat16: 8, torch.float16: 11}


def spacing(r, dt):
    """ulp of the dtype at |r| (normal range)."""
    mag = np.maximum(np.abs(r), 2.0 ** -14)
    return 2.0 ** (np.floor(np.log2(mag)) - BITS[dt] + 1)


def crit(g, r, dt):
    """excess over max(1e-2, half-ulp), over max(1e-2, ulp); and the worst
    distance in ulps from the correctly rounded reference."""
    g = np.asarray(g, np.float64)
    r = np.asarray(r, np.float64)
    u = spacing(r, dt)
    e = np.abs(g - r)
    rr = torch.from_numpy(r).to(dt).double().numpy()
    return (float((e - np.maximum(1e-2, u / 2)).max()), float((e - np.maximum(1e-2, u)).max()),
            float((np.abs(g - rr) / u).max()), float(np.abs(rr - r).max()))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dtype", default="bf16")
    args = ap.parse_args()
    dt = {"bf16": torch.bfloat16, "fp16": torch.float16}[args.dtype]
    rows = []
    for D in (32, 64):
        for ext, ker, dil, cau in CASES:
            cfg = na_synth.small_config(ext, ker, dil, cau, head_dim=D, batch=1, heads=2, dtype=dt)
            q, k, v, do = na_synth.make_inputs(cfg, salt=7)
            op = oracle.make_problem(1, 2, list(ext), D, list(ker), list(dil), list(cau))
            ro, _ = oracle.fwd(op, q, k, v)
            ex = oracle.bwd(op, q, k, v, do, stored_o=False)
            st = oracle.bwd(op, q, k, v, do, stored_o=True)
            kw = dict(kernel_size=ker, dilation=dil, is_causal=[bool(c) for c in cau], impl="tc")
            qd, kd, vd, dod = (t.cuda() for t in (q, k, v, do))
            o, lse = na.na_fwd(qd, kd, vd, **kw)
            ga = na.na_bwd(qd, kd, vd, o, dod, lse, **kw)
            o_ref = torch.from_numpy(ro).to(dt).view_as(qd).cuda()
            gb = na.na_bwd(qd, kd, vd, o_ref, dod, lse, **kw)
            torch.cuda.synchronize()
            shp = ro.shape
            r = {"case": f"{ext} k{ker} d{dil} c{cau} D{D}",
                 "O_err": mx(o.float().cpu().reshape(shp), ro)}
            c = crit(o.float().cpu().reshape(shp), ro, dt)
            r.update({"O_xs_half": round(c[0], 5), "O_xs_ulp": round(c[1], 5), "O_ulps": round(c[2], 2),
                      "O_round_floor": round(c[3], 5)})
            for tag, g in (("gpuO", ga), ("refO", gb)):
                for nm, gg, e, s in zip(("dQ", "dK", "dV"), g, ex, st):
                    h = gg.float().cpu().reshape(shp)
                    r[f"{nm}_{tag}_exact"] = round(mx(h, e), 5)
                    r[f"{nm}_{tag}_stored"] = round(mx(h, s), 5)
                    if tag == "gpuO":
                        c = crit(h, e, dt)
                        r[f"{nm}_xs_half"] = round(c[0], 5)
                        r[f"{nm}_xs_ulp"] = round(c[1], 5)
                        r[f"{nm}_ulps"] = round(c[2], 2)
                        r[f"{nm}_round_floor"] = round(c[3], 5)
            r["stored_vs_exact_dQ"] = round(mx(st[0], ex[0]), 5)
            rows.append(r)
            print(json.dumps(r), flush=True)
    worst = {k: max(r[k] for r in rows) for k in rows[0] if k != "case"}
    print("WORST", json.dumps(worst), flush=True)


if __name__ == "__main__":
    main()
