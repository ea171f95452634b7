"""Summarise ncu output into small committed files under profiles/.

    python tools/ncu_summary.py launches <launches.csv> <out.md>   # gpu__time_duration list
    python tools/ncu_summary.py full <prof.ncu-rep> <out.md> [traffic.json]

`launches`: per-kernel launch count, total and mean device time and share of
the captured window (cold-cache, serialised: compare shares, not absolutes).
`full`: key metrics of each profiled kernel (time, DRAM bytes, pipe
utilisation, stall reasons) and, optionally, traffic.json = DRAM bytes per
launch keyed by kernel function name (read by bench.py's roofline.traffic).
"""
import collections
import csv
import io
import json
import re
import subprocess
import sys

OURS = re.compile(r"fna_\w+")


def short(name):
    m = OURS.search(name)
    base = m.group(0) if m else name.split("(")[0][-60:]
    t = re.match(r"<([^>]*)>", name[m.end():]) if m else None
    return base + (f"<{t.group(1)}>" if t else "")


def launches(path, out):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    i_name, i_metric, i_val = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    per = collections.OrderedDict()
    for r in rows[start + 1:]:
        if len(r) <= i_val or r[i_metric] != "gpu__time_duration.sum":
            continue
        v = float(r[i_val].replace(",", ""))
        unit = r[hdr.index("Metric Unit")]
        ms = v * {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(unit, 1e-6)
        k = short(r[i_name])
        d = per.setdefault(k, [0, 0.0])
        d[0] += 1
        d[1] += ms
    ours = {k: v for k, v in per.items() if k.startswith("fna_")}
    tot = sum(v[1] for v in ours.values())
    with open(out, "w") as f:
        f.write(f"# ncu launch list (gpu__time_duration.sum, --clock-control none) — {path}\n\n")
        f.write("Our kernels only (torch RNG/copy kernels of input generation omitted).\n\n")
        f.write("| kernel | launches | total ms | mean ms | share of our time |\n|---|---|---|---|---|\n")
        for k, (n, ms) in sorted(ours.items(), key=lambda x: -x[1][1]):
            f.write(f"| {k} | {n} | {ms:.3f} | {ms / n:.4f} | {ms / tot:.3f} |\n")
        f.write(f"\nAll launches captured: {sum(v[0] for v in per.values())}; ours: "
                f"{sum(v[0] for v in ours.values())}.\n")
    print(open(out).read())


METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed.avg.per_cycle_active", "IPC"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def full(rep, out, traffic_path=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    idx = {h: i for i, h in enumerate(hdr)}
    traffic = {}
    with open(out, "w") as f:
        f.write(f"# ncu --set full summary — {rep}\n\n")
        for r in data:
            name = short(r[idx["Kernel Name"]])
            f.write(f"## {name}\n\n| metric | value |\n|---|---|\n")
            for m, label in METRICS:
                if m in idx:
                    f.write(f"| {label} (`{m}`) | {r[idx[m]]} {units[idx[m]]} |\n")
            stalls = [(h.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(r[i]))
                      for h, i in idx.items()
                      if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")
                      and r[i].replace(".", "").isdigit()]
            tot = sum(v for _, v in stalls) or 1.0
            top = ", ".join(f"{k} {100 * v / tot:.0f}%" for k, v in sorted(stalls, key=lambda x: -x[1])[:6])
            f.write(f"\nTop stall reasons (pc sampling): {top}\n\n")
            def to_bytes(m):
                v = float(r[idx[m]].replace(",", ""))
                return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(units[idx[m]], 1)
            fn = name.split("<")[0]
            traffic.setdefault(fn, to_bytes("dram__bytes_read.sum") + to_bytes("dram__bytes_write.sum"))
    print(open(out).read())
    if traffic_path:
        json.dump(traffic, open(traffic_path, "w"), indent=1)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
