"""Incremental libna.so rebuild for kernel experiments: recompiles only the
named sources (default: every source newer than its object) and relinks.

    python tools/rebuild.py [tc_fwd.cu ...] [--out path.so]
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2403_04690_b200 import build as b  # noqa: E402

args = sys.argv[1:]
out = b.OUT
if "--out" in args:
    i = args.index("--out")
    out = os.path.abspath(args[i + 1])
    del args[i:i + 2]
srcs = b.sources()
deps = max(os.path.getmtime(d) for d in b._deps() if not d.endswith((".cu", ".cpp")))
# named sources compile into a directory of their own (parallel variant builds)
vdir = b.BUILD if out == b.OUT else os.path.join(b.BUILD, "v_" + os.path.basename(out))
os.makedirs(vdir, exist_ok=True)
objs = []
for s in srcs:
    obj = os.path.join(b.BUILD, os.path.basename(s) + ".o")
    # a named source, or any source whose in-tree object predates a header
    # (objects built against another struct layout must not be mixed)
    stale = not os.path.exists(obj) or os.path.getmtime(obj) < max(os.path.getmtime(s), deps)
    want = (os.path.basename(s) in args or os.path.getmtime(obj) < deps) if args else stale
    if want:
        print("compile", os.path.basename(s), flush=True)
        obj = b._compile(s, False, vdir)
    objs.append(obj)
cmd = [b.NVCC, *b.ARCH, "-shared", "-o", out, *objs, "-lcudart_static", "-ldl", "-lrt", "-lpthread"]
subprocess.run(cmd, check=True)
print(out)
