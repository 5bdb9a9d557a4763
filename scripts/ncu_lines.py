"""Top source lines of an ncu report by warp-stall samples and executed instructions.

    python scripts/ncu_lines.py <file.ncu-rep> [n]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
data, fname = [], ""
hdr = None
for r in rows:
    if len(r) == 2 and r[0] in ("File Name", "File Path"):
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = {h: j for j, h in enumerate(r)}
        if "Instructions Executed" not in hdr:
            hdr = None
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    if not r[0]:
        continue  # SASS rows (the source line above carries their sums)
    try:
        st = float(r[hdr["Warp Stall Sampling (All Samples)"]] or 0)
        ins = float(r[hdr["Instructions Executed"]] or 0)
    except ValueError:
        continue
    data.append((st, ins, f"{fname}:{r[0]}", r[1][:100]))
ts = sum(d[0] for d in data) or 1
ti = sum(d[1] for d in data) or 1
print(f"total stall samples {ts:.0f}, warp instructions {ti:.0f}")
for d in sorted(data, key=lambda x: -x[0])[:n]:
    print(f"{100 * d[0] / ts:5.1f}% stall {100 * d[1] / ti:5.1f}% inst  {d[2]:22s} {d[3]}")
