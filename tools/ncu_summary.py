"""Summarise an ncu report: SOL numbers, pipe utilisation, occupancy and the
per-opcode SASS instruction mix (per point-update if --updates is given)."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
updates = float(sys.argv[2]) if len(sys.argv) > 2 else None


def page(name, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", name, "--csv", *extra],
                         capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


raw = page("raw")
hdr, units, vals = raw[0], raw[1], raw[2]
want = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "smsp__inst_executed.sum",
        "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum",
        "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
        "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum"]
for w in want:
    if w in hdr:
        i = hdr.index(w)
        print(f"{w:70s} {vals[i]:>20s} {units[i]}")

rows = page("source", ["--print-source", "sass"])
h = rows[1]
iS, iE = h.index("Source"), h.index("Instructions Executed")
iW = h.index("Warp Stall Sampling (All Samples)")
ops, st = collections.Counter(), collections.Counter()
tot = 0
for r in rows[2:]:
    if len(r) <= iE:
        continue
    try:
        e = int(r[iE] or 0)
    except ValueError:
        continue
    src = r[iS].strip().split()
    if not src:
        continue
    op = src[1] if src[0].startswith("@") else src[0]
    op = op.split(".")[0]
    ops[op] += e
    st[op] += int(r[iW] or 0)
    tot += e
scale = updates / 32.0 if updates else 1.0
print(f"\nwarp instructions: {tot}  per warp-update: {tot / scale:.1f}" if updates else f"\nwarp instructions: {tot}")
for k, v in ops.most_common(25):
    print(f"  {k:10s} {v / scale:10.2f}   stall samples {st[k]}")
