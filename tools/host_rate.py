"""Host enqueue cost of ctx.decode (wall time per call without synchronizing)
against the device time per call, for a bench config.
Usage: python tools/host_rate.py [config=cfg1] [kind=gaussian]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2407_12820_b200 as pq  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
kind = sys.argv[2] if len(sys.argv) > 2 else "gaussian"
c = bench.CONFIGS[name]
k = bench.cfg_k(c)
ctx = pq.Context(0)
layer, q = bench.make_layer(ctx, name, kind, seed=1)[:2]
out = torch.empty((c["units"], c["g"], 128), device="cuda")
for _ in range(20):
    ctx.decode(layer, q, k, out=out)
torch.cuda.synchronize()
n = 300
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
e0.record()
for _ in range(n):
    ctx.decode(layer, q, k, out=out)
e1.record()
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"{name}: host enqueue {1e6 * (t1 - t0) / n:.1f} us/call, device {1e3 * e0.elapsed_time(e1) / n:.1f} us/call")
