"""Per-file / per-function-group instruction totals from an ncu source page
(needs -lineinfo).  Usage: python tools/ncu_cats.py rep.ncu-rep per_unit"""
import collections
import re
import subprocess
import sys

rep, unit = sys.argv[1], sys.argv[2]
out = subprocess.run([sys.executable, "tools/ncu_lines.py", rep, unit, "100000"],
                     capture_output=True, text=True).stdout
c = collections.Counter()
for l in out.splitlines():
    m = re.match(r"\s*([\d.]+) stall=\s*\d+ (\S+?):(\d+)", l)
    if not m:
        continue
    v, f, ln = float(m.group(1)), m.group(2), int(m.group(3))
    c[f] += v
    if f == "ti64_point.cuh":
        cat = ("tfuncs" if ln < 120 else "rates" if ln < 195 else "corr" if ln < 235 else
               "seed" if ln < 315 else "substep")
        c["  point:" + cat] += v
    if f == "ti64_fastmath.cuh":
        c["  fm:" + ("ln" if 60 <= ln < 70 or 110 <= ln < 135 else "exp")] += v
print(out.splitlines()[0])
for k, v in sorted(c.items(), key=lambda x: -x[1]):
    print(f"{v:8.1f} {k}")
