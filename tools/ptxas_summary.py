"""Per-kernel registers / spills from `nvcc -Xptxas -v` for one source file.

    python tools/ptxas_summary.py paper_2403_04690_b200/csrc/tc_bwd.cu
"""
import re
import subprocess
import sys

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__file__)))
from paper_2403_04690_b200 import build as b  # noqa: E402

src = sys.argv[1]
cmd = [b.NVCC, *b.ARCH, *b.FLAGS, "-Xptxas", "-v", "-c", src, "-o", "/tmp/ptxas_summary.o"]
err = subprocess.run(cmd, capture_output=True, text=True).stderr
cur = None
for line in err.splitlines():
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
        cur = re.sub(r"\(.*", "", cur.replace("void ", "").replace("na::(anonymous namespace)::", ""))
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        spill = f"spill {m.group(1)}/{m.group(2)}"
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        print(f"{cur:60s} regs {m.group(1):>4s}  {spill}")
        cur = None
