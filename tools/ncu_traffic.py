"""Extracts per-launch DRAM traffic of the fused decode kernel from an
`ncu --set full` report and writes profiles/ncu_traffic.json (read by
bench.py for roofline.traffic).

  python tools/ncu_traffic.py gpurun_out/attend_fused.ncu-rep [out.json]
"""
import csv
import io
import json
import os
import subprocess
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0, "ms": 1e3}

rep = sys.argv[1]
out = sys.argv[2] if len(sys.argv) > 2 else os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                          "profiles", "ncu_traffic.json")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]


def val(r, name):
    i = hdr.index(name)
    return float(r[i].replace(",", "")) * UNIT.get(units[i], 1.0)


res = {"source": os.path.basename(rep), "launches": []}
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")]
    if "attend_kernel" not in name and "tuple_select_kernel" not in name:
        continue
    rd, wr = val(r, "dram__bytes_read.sum"), val(r, "dram__bytes_write.sum")
    res["launches"].append({"kernel": r[hdr.index("Kernel Name")], "dram_read_bytes": rd, "dram_write_bytes": wr,
                            "duration_us_under_ncu": val(r, "gpu__time_duration.sum")})
if res["launches"]:  # per decode step: every captured launch (pair select + attention on the split path)
    res["attend_kernel_fused"] = sum(x["dram_read_bytes"] + x["dram_write_bytes"] for x in res["launches"])
    res["note"] = "per decode step: the pair-select launch + the attention launch"

json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res))
