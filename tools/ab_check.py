"""Bitwise A/B check of a kernel variant against a base build (GPU box).

    python tools/ab_check.py BASE.so VARIANT.so [VARIANT2.so ...]

A scheduling-only change (warp roles, load order, barrier placement) must
leave every output bit unchanged.  Each library runs in its own process
over the small instantiation sweep of tools/run_small.py plus the bench
configs; the processes print a SHA-1 per output tensor, and this script
reports the cases whose digests differ.
"""
import hashlib
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def digests(libpath):
    import torch
    sys.path.insert(0, ROOT)
    import na_synth
    import paper_2403_04690_b200.na as nab
    nab.LIB_PATH = os.path.abspath(libpath)
    small = [
        ([300], [33], [2], [1], 64, torch.float16),
        ([20, 27], [7, 5], [2, 1], [0, 0], 32, torch.bfloat16),
        ([6, 10, 12], [3, 5, 5], [1, 1, 2], [1, 0, 0], 64, torch.float16),
        ([300], [33], [2], [1], 64, torch.bfloat16),
        ([20, 27], [7, 5], [2, 1], [0, 0], 64, torch.float16),
        ([6, 10, 12], [3, 5, 5], [1, 1, 2], [1, 0, 0], 32, torch.bfloat16),
        ([300], [33], [2], [1], 128, torch.float16),
        ([9, 20], [5, 7], [1, 2], [0, 1], 128, torch.bfloat16),
        ([6, 10, 12], [3, 5, 5], [1, 1, 2], [1, 0, 0], 128, torch.float16),
        ([56, 56], [7, 7], [8, 8], [0, 0], 32, torch.float16),
        ([24, 20], [5, 5], [1, 1], [0, 0], 16, torch.float16),
        ([40, 40], [13, 11], [1, 1], [0, 0], 64, torch.bfloat16),
        ([1000], [127], [1], [0], 64, torch.float16),
        ([777], [63], [3], [1], 32, torch.float16),
    ]
    cases = [(f"small{i}", na_synth.small_config(e, k, d, c, head_dim=hd, dtype=dt, batch=2, heads=3))
             for i, (e, k, d, c, hd, dt) in enumerate(small)]
    cases += [(n, na_synth.CONFIGS[n]) for n in ("B_d1", "B_d4_causal", "C_d1", "C_d8", "D_d2", "E")]
    out = {}
    for name, cfg in cases:
        q, k, v, do = na_synth.make_inputs(cfg, device="cuda", salt=5)
        kw = dict(kernel_size=list(cfg.kernel_size), dilation=list(cfg.dilation),
                  is_causal=[bool(c) for c in cfg.is_causal])
        o, lse = nab.na_fwd(q, k, v, impl="tc", **kw)
        dq, dk, dv = nab.na_bwd(q, k, v, o, do, lse, impl="tc", **kw)
        torch.cuda.synchronize()
        out[name] = {t: hashlib.sha1(x.contiguous().view(torch.uint8).cpu().numpy().tobytes()).hexdigest()[:16]
                     for t, x in (("O", o), ("LSE", lse), ("dQ", dq), ("dK", dk), ("dV", dv))}
    return out


if __name__ == "__main__":
    if sys.argv[1] == "--worker":
        print("DIGESTS " + json.dumps(digests(sys.argv[2])))
        sys.exit(0)
    libs = sys.argv[1:]
    res = {}
    for lp in libs:
        r = subprocess.run([sys.executable, __file__, "--worker", lp], capture_output=True, text=True, timeout=900)
        line = [x for x in r.stdout.splitlines() if x.startswith("DIGESTS ")]
        if r.returncode != 0 or not line:
            print(f"{lp}: FAILED rc={r.returncode}\n{r.stderr[-3000:]}")
            continue
        res[lp] = json.loads(line[0][8:])
    base = res.get(libs[0])
    for lp in libs[1:]:
        if lp not in res or base is None:
            continue
        diff = [(c, t) for c in base for t in base[c] if res[lp].get(c, {}).get(t) != base[c][t]]
        print(f"{os.path.basename(lp)}: {'BITWISE EQUAL' if not diff else 'DIFFERS ' + str(diff)}")
