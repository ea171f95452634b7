"""Warp-stall breakdown of one kernel from an `ncu --set full --import-source on` report.

    python tools/ncu_stalls.py <report.ncu-rep> <kernel-regex> [top]

Prints the kernel's stall-reason totals (sampled), the top source lines
(cuda view) and the top SASS instructions by samples, each with its two
dominant stall reasons.  Reads the report with `ncu -i ... --page source`.
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def page(rep, kernel, view):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kernel}",
                          "--print-source", view], capture_output=True, text=True, check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def stall_cols(header):
    return [(i, h) for i, h in enumerate(header) if h.startswith("stall_") and "Not Issued" not in h]


def main():
    rep, kernel = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
    rows = page(rep, kernel, "sass")
    hdr = next(r for r in rows if r and r[0] == "Address")
    si = hdr.index("Warp Stall Sampling (All Samples)")
    ie = hdr.index("Instructions Executed")
    sc = stall_cols(hdr)
    tot = defaultdict(float)
    insts = []
    seen = set()
    for r in rows:
        if r and r[0] in seen:
            continue
        if r:
            seen.add(r[0])
        if len(r) != len(hdr) or r[0] in ("Address",):
            continue
        try:
            s = float(r[si])
        except ValueError:
            continue
        st = {h: float(r[i] or 0) for i, h in sc}
        for h, v in st.items():
            tot[h] += v
        insts.append((s, r[1].strip(), float(r[ie] or 0), st))
    alls = sum(tot.values())
    print(f"kernel /{kernel}/: {alls:.0f} stall samples, {sum(x[2] for x in insts):.0f} warp instructions")
    for h, v in sorted(tot.items(), key=lambda kv: -kv[1])[:10]:
        print(f"  {h:24s} {100 * v / max(alls, 1):5.1f}%")
    print(f"\ntop {top} SASS instructions by samples:")
    for s, src, n, st in sorted(insts, key=lambda x: -x[0])[:top]:
        dom = sorted(st.items(), key=lambda kv: -kv[1])[:2]
        print(f"  {s:7.0f} {100 * s / max(alls, 1):5.1f}%  n={n:9.0f}  {src[:60]:60s} "
              + " ".join(f"{h[6:]}={v:.0f}" for h, v in dom))
    rows = page(rep, kernel, "cuda,sass")
    agg = {}
    fname = ""
    h2 = None
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
        if r and r[0] == "Line No":
            h2 = r
            continue
        if h2 is None or len(r) != len(h2) or not r[0].isdigit() or r[2] != "-":
            continue
        try:
            s = float(r[4])
        except ValueError:
            continue
        st = {h: float(r[i] or 0) for i, h in stall_cols(h2)}
        agg[f"{fname}:{r[0]}"] = (s, r[1].strip()[:64], st)
    print(f"\ntop {top} source lines by samples:")
    for loc, (s, src, st) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        dom = sorted(st.items(), key=lambda kv: -kv[1])[:2]
        print(f"  {s:7.0f} {100 * s / max(alls, 1):5.1f}%  {loc:20s} {src:64s} "
              + " ".join(f"{h[6:]}={v:.0f}" for h, v in dom))


if __name__ == "__main__":
    main()
