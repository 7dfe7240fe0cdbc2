"""Count SASS instructions (by unit) of tools/probe/sass_floor.cu's kernels,
minus the load/store skeleton (k_load_store)."""
import collections
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
cubin = "/tmp/sass_floor.cubin"
subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "--fmad=false", "-O3",
                "-cubin", "-I", str(ROOT / "include"), "-o", cubin,
                str(ROOT / "tools" / "probe" / "sass_floor.cu")], check=True)
sass = subprocess.run(["cuobjdump", "-sass", cubin], capture_output=True, text=True).stdout
funcs = {}
cur = None
for ln in sass.splitlines():
    m = re.search(r"Function : (\w+)", ln)
    if m:
        cur = funcs.setdefault(m.group(1), collections.Counter())
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9]*)", ln)
    if m and cur is not None:
        cur[m.group(1)] += 1
FP64 = {"DFMA", "DADD", "DMUL", "DSETP", "FRND", "DMNMX", "F2F", "I2F", "F2I", "MUFU"}
base = funcs.get("k_load_store", collections.Counter())
for name, c in sorted(funcs.items()):
    if name == "k_load_store":
        continue
    d = c - base
    fp64 = sum(v for k, v in d.items() if k in FP64)
    tot = sum(d.values())
    print(f"{name:16s} total {tot:3d}  fp64-pipe {fp64:3d}  " +
          " ".join(f"{k}:{v}" for k, v in sorted(d.items(), key=lambda kv: -kv[1])))
