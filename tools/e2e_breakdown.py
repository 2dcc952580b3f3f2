"""Where the end-to-end (host buffers) decode time goes: wall time per call
of pqkv_decode_host vs the same decode on device buffers with a
synchronize per call vs the device-timed decode.
Usage: python tools/e2e_breakdown.py [config=northstar]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2407_12820_b200 as pq  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "northstar"
c = bench.CONFIGS[name]
k = bench.cfg_k(c)
ctx = pq.Context(0)
layers = [bench.make_layer(ctx, name, "gaussian", seed=s)[:2] for s in range(4)]
hq = [q.cpu().pin_memory() for _, q in layers]
ho = torch.empty_like(hq[0]).pin_memory()
N = 200
for i in range(10):
    ctx.decode_host(layers[i % 4][0], hq[i % 4], ho, k)
t0 = time.perf_counter()
for i in range(N):
    ctx.decode_host(layers[i % 4][0], hq[i % 4], ho, k)
host = (time.perf_counter() - t0) / N * 1e6
out = torch.empty_like(layers[0][1])
t0 = time.perf_counter()
for i in range(N):
    ctx.decode(layers[i % 4][0], layers[i % 4][1], k, out=out)
    torch.cuda.synchronize()
devsync = (time.perf_counter() - t0) / N * 1e6
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(N):
    ctx.decode(layers[i % 4][0], layers[i % 4][1], k, out=out)
e1.record()
torch.cuda.synchronize()
dev = e0.elapsed_time(e1) * 1e3 / N
t0 = time.perf_counter()
for i in range(N):
    layers[i % 4][0].ref()
refc = (time.perf_counter() - t0) / N * 1e6
print(f"{name}: decode_host wall {host:.1f} us/call | device decode + sync per call {devsync:.1f} us | "
      f"device back-to-back {dev:.1f} us | ctypes layer ref {refc:.2f} us")
