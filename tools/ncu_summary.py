"""Key metrics of every kernel launch in ncu reports (`--set full`) ->
JSON: duration, DRAM bytes and throughput, achieved occupancy, registers,
shared memory, IPC, issue slots, eligible warps, grid / cluster shape.
Usage: python tools/ncu_summary.py OUT.json NAME=REPORT.ncu-rep [...]"""
import csv
import io
import json
import subprocess
import sys

METRICS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "launch__registers_per_thread": "registers_per_thread",
    "launch__shared_mem_per_block_dynamic": "dynamic_smem_per_cta",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "smsp__warps_eligible.avg.per_cycle_active": "eligible_warps_per_cycle",
    "sm__inst_executed.avg.per_cycle_active": "ipc",
    "launch__grid_size": "grid_size",
    "launch__cluster_dim_x": "cluster_x",
    "launch__occupancy_limit_registers": "occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem": "occupancy_limit_smem",
    "lts__t_sector_hit_rate.pct": "l2_hit_rate_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
}

out = {}
for arg in sys.argv[2:]:
    name, rep = arg.split("=", 1)
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) < 3:
        continue
    hdr, units = rows[0], rows[1]
    launches = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for m, key in METRICS.items():
            if m in hdr:
                i = hdr.index(m)
                d[key] = [r[i], units[i]]
        launches.append(d)
    out[name] = launches
json.dump(out, open(sys.argv[1], "w"), indent=1)
for k, v in out.items():
    for d in v:
        print(k, d["kernel"][:60], {kk: vv[0] for kk, vv in d.items() if kk in ("duration", "dram_throughput_pct",
                                                                                  "achieved_occupancy_pct")})
