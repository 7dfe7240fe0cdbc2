"""Where the instruction-fetch stalls (stall_no_inst) of a kernel sit: per SASS
address the executed count and the no_inst samples, summed over windows of
the code so hot regions and their fetch stalls can be compared.
Usage: python tools/ncu_noinst.py rep.ncu-rep [window_instructions]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
win = int(sys.argv[2]) if len(sys.argv) > 2 else 64
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ia, isrc, iex = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed")
ini, iall = hdr.index("stall_no_inst"), hdr.index("# Samples")
data = []
for r in rows[2:]:
    if len(r) <= ini:
        continue
    try:
        data.append((int(r[ia], 16), r[isrc].strip(), int(r[iex] or 0), int(r[ini] or 0),
                     int(r[iall] or 0)))
    except ValueError:
        continue
base = data[0][0]
tot_ex = sum(d[2] for d in data)
tot_ni = sum(d[3] for d in data)
tot_s = sum(d[4] for d in data)
print(f"instructions {len(data)} ({len(data) * 16 / 1024:.1f} KiB), executed {tot_ex:.4g}, "
      f"samples {tot_s}, no_inst samples {tot_ni} ({100 * tot_ni / max(tot_s, 1):.1f} %)")
print("window(first idx)  exec%   samples%  no_inst%  first instruction")
for k in range(0, len(data), win):
    w = data[k:k + win]
    ex = sum(d[2] for d in w)
    ni = sum(d[3] for d in w)
    sm = sum(d[4] for d in w)
    if ex * 200 > tot_ex or ni * 200 > tot_ni:
        print(f"{k:6d} {100 * ex / tot_ex:7.2f} {100 * sm / tot_s:8.2f} {100 * ni / max(tot_ni, 1):8.2f}   "
              f"{w[0][1][:60]}")
