"""Per-CUDA-line warp-stall samples of one kernel in an ncu report
(`ncu -i REP --page source --csv --print-source cuda,sass`): the top lines
by samples with their dominant stall reasons.
Usage: python tools/ncu_lines.py REPORT.ncu-rep [top=40] [kernel-regex]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
if len(sys.argv) > 3:
    cmd += ["-k", "regex:" + sys.argv[3]]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, header, acc, total = "?", None, defaultdict(lambda: [0, "", defaultdict(int)]), 0
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        header = r
        continue
    if header is None or r[0] in ("", "Function Name"):
        continue
    try:
        s = int(r[4])
    except (ValueError, IndexError):
        continue
    key = (fname, int(r[0]))
    acc[key][0] += s
    acc[key][1] = r[1][:90]
    total += s
    for i, h in enumerate(header):
        if h.startswith("stall_") and "Not Issued" not in h and i < len(r):
            try:
                acc[key][2][h[6:]] += int(r[i])
            except ValueError:
                pass
print(f"total samples {total}")
for (f, ln), (s, src, st) in sorted(acc.items(), key=lambda kv: -kv[1][0])[:top]:
    reasons = ", ".join(f"{k} {v}" for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:3] if v)
    print(f"{100.0 * s / max(total, 1):5.1f}% {f}:{ln:<5} {src:<90} [{reasons}]")
