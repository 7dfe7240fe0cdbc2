"""Per-source-line instruction / stall totals from an ncu report
(needs -lineinfo).  Usage: python tools/ncu_lines.py rep.ncu-rep [per_unit] [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
unit = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, hdr, res = None, None, []
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0] not in ("", "Function Name") and len(r) > 8:
        try:
            e = int(r[7] or 0)
            st = int(r[4] or 0)
        except ValueError:
            continue
        if e:
            res.append((e, st, fname, r[0], r[1].strip()[:80]))
res.sort(reverse=True)
tot = sum(x[0] for x in res)
print(f"total warp instructions {tot} -> {tot / unit:.1f} per unit")
for e, st, f, ln, src in res[:top]:
    print(f"{e / unit:8.2f} stall={st:7d} {f}:{ln:5s} {src}")
