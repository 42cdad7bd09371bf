"""Hot CUDA source lines of an ncu report (source page, cuda+sass): warp-stall
samples summed per source line.  usage: ncu_hot.py report.ncu-rep [n]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hdr]
samp = h.index("Warp Stall Sampling (All Samples)")
inst = h.index("Instructions Executed")
per_line = defaultdict(lambda: [0.0, 0.0, ""])
line, src, fname = None, "", ""
total = 0.0
for r in rows[hdr + 1:]:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) < len(h) or r[0] == "Line No":
        continue
    if r[0]:
        line, src = (fname, int(r[0])), r[1]
    try:
        s = float(r[samp] or 0)
        e = float(r[inst] or 0)
    except ValueError:
        continue
    if line is None:
        continue
    per_line[line][0] += s
    per_line[line][1] += e
    per_line[line][2] = src
    total += s
print(f"total stall samples {total:.0f}")
for ln, (s, e, src) in sorted(per_line.items(), key=lambda kv: -kv[1][0])[:n]:
    print(f"{ln[0][:14]:14s}:{ln[1]:5d} {100 * s / total:5.1f}% inst {e:10.0f}  {src.strip()[:80]}")
