"""Per-source-line instruction and stall shares from an ncu report
(`ncu -i X --page source --csv --print-source cuda,sass`).

    python tools/ncu_lines.py report.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
res, cur, ix = [], None, None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        ix = {h: k for k, h in enumerate(r)}
        continue
    if ix is None or len(r) < 8 or not r[0].isdigit():
        continue
    try:
        e = float(r[7] or 0)
        s = float(r[4] or 0)
    except ValueError:
        continue
    res.append((cur, int(r[0]), r[1].strip()[:95], e, s))
tot = sum(x[3] for x in res) or 1
stot = sum(x[4] for x in res) or 1
print(f"total warp instructions {tot:.4g}, stall samples {stot:.0f}")
for f, ln, src, e, s in sorted(res, key=lambda x: -(x[3] / tot + x[4] / stot))[:top]:
    print(f"{f:22s}{ln:5d} inst {e / tot * 100:5.1f}%  stall {s / stot * 100:5.1f}%  {src}")
