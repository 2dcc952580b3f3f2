"""Summarise an ncu source page by CUDA source line: warp-stall samples per
line, top N.

  ncu -i X.ncu-rep --page source --csv --print-source=cuda,sass > f.csv
  python tools/ncu_hot.py f.csv [N]
"""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
rows = list(csv.reader(open(path)))
cur_file, hdr, agg, src = None, None, defaultdict(float), {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 5:
        continue
    try:
        line = int(r[0])
        samples = float(r[4] or 0)
    except ValueError:
        continue
    key = (cur_file, line)
    agg[key] += samples
    src[key] = r[1][:100]
tot = sum(agg.values()) or 1
for (f, l), v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
    print(f"{100 * v / tot:5.1f}% {f}:{l}  {src[(f, l)]}")
