import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), 'tests'))
import torch, numpy as np, na_synth, oracle
import paper_2403_04690_b200 as na
from na_tol import LSE_TOL, excess, max_abs
cases = [([15, 5, 12], [1, 1, 4], [3, 3, 3], [0, 0, 1], 64, torch.bfloat16),
 ([4, 12, 14], [1, 1, 2], [3, 3, 3], [0, 0, 1], 128, torch.bfloat16),
 ([14, 17, 6], [2, 2, 5], [2, 3, 1], [1, 1, 1], 64, torch.bfloat16),
 ([42, 7], [5, 1], [2, 3], [1, 1], 32, torch.bfloat16),
 ([14, 5, 10], [1, 1, 3], [3, 1, 2], [0, 1, 0], 32, torch.bfloat16),
 ([15, 12, 16], [3, 6, 1], [1, 1, 1], [0, 1, 0], 64, torch.bfloat16),
 ([13, 30], [2, 4], [1, 2], [1, 1], 64, torch.bfloat16),
 ([14, 6, 3], [1, 6, 3], [3, 1, 1], [0, 1, 1], 128, torch.bfloat16),
 ([11, 12, 11], [1, 5, 1], [1, 2, 1], [0, 1, 0], 128, torch.bfloat16)]
for ext, ker, dil, cau, D, dt in cases:
    cfg = na_synth.small_config(ext, ker, dil, cau, head_dim=D, batch=1, heads=2, dtype=dt)
    p = na.make_problem(1, 2, list(ext), D, ker, dil, [bool(c) for c in cau], dtype=dt, impl="tc")
    q, k, v, do = na_synth.make_inputs(cfg, salt=17)
    op = oracle.make_problem(1, 2, list(ext), D, ker, dil, [int(c) for c in cau], 0.0)
    ro, rlse = oracle.fwd(op, q, k, v)
    rdq, rdk, rdv = oracle.bwd(op, q, k, v, do, stored_o=False)
    shp = (1, 2, cfg.tokens, D)
    n = na.na_plan_candidates(p)
    kw = dict(kernel_size=ker, dilation=dil, is_causal=[bool(c) for c in cau], impl="tc")
    for pick in sorted({0, n - 1}):
        na.na_set_plan_choice(p, (pick, pick, pick))
        qd, kd, vd, dod = (t.cuda() for t in (q, k, v, do))
        o, lse = na.na_fwd(qd, kd, vd, **kw)
        dq, dk, dv = na.na_bwd(qd, kd, vd, o, dod, lse, **kw)
        torch.cuda.synchronize()
        res = [(nm, round(float(excess(a.float().cpu().reshape(shp), r, dt)), 5), round(float(max_abs(a.float().cpu().reshape(shp), r)), 5))
               for nm, a, r in (("O", o, ro), ("dQ", dq, rdq), ("dK", dk, rdk), ("dV", dv, rdv))]
        le = float(max_abs(lse.cpu().reshape(shp[:-1]), rlse))
        print(ext, ker, dil, cau, D, "pick", pick, "precise", na.na_bf16_precise(p) if hasattr(na, 'na_bf16_precise') else '?', "LSE", round(le, 5), res, flush=True)
    na.na_set_plan_choice(p, (0, 0, 0))
