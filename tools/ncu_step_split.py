"""Instruction and stall split of one K2 capture by code region, per step.
Usage: python tools/ncu_step_split.py rep.ncu-rep steps [top]"""
import collections
import re
import subprocess
import sys

rep, steps = sys.argv[1], float(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run([sys.executable, "tools/ncu_lines.py", rep, "1", "100000"],
                     capture_output=True, text=True).stdout
rows = []
for l in out.splitlines()[1:]:
    m = re.match(r"\s*([\d.]+) stall=\s*(\d+) (\S+?):(\d+)\s+(.*)", l)
    if m:
        rows.append((int(m.group(2)), float(m.group(1)), m.group(3), int(m.group(4)), m.group(5)[:80]))
tot = sum(r[0] for r in rows) or 1
ti = sum(r[1] for r in rows)
print(f"stall samples {tot}, instructions per step {ti / steps:.1f}")
c, ci = collections.Counter(), collections.Counter()
src = open("paper_2402_17580_b200/csrc/ti64_point.cuh").read().splitlines()


def region(f, ln):
    if f == "ti64_fastmath.cuh":
        return "fm:" + ("ln" if 60 <= ln < 70 or 110 <= ln < 135 else "exp")
    if f == "ti64_point.cuh":
        return "point"
    if f == "ti64_sources.cuh":
        return "generator"
    if f == "ti64_kernels.cu":
        return "loop"
    return f


for st, ins, f, ln, s in rows:
    k = region(f, ln)
    c[k] += st
    ci[k] += ins
for k, v in c.most_common():
    print(f"{v / tot * 100:5.1f}% stall  {ci[k] / steps:7.1f} instr/step  {k}")
rows.sort(reverse=True)
for r in rows[:top]:
    print(f"{r[0] / tot * 100:5.1f}% {r[1] / steps:6.1f}/step {r[2]}:{r[3]} {r[4]}")
