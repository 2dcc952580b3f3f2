"""Host-overhead probe for the end-to-end decode (pqkv_decode_host): per-step
wall time of (a) decode_host (pinned host q/out, H2D + launch + D2H + sync),
(b) device decode + synchronize per step, (c) back-to-back device decodes
(CUDA events), on one north-star layer."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2407_12820_b200 as pq  # noqa: E402

S, H, DH = 131072, 32, 128
ctx = pq.Context(0)
keys, vals, q = ctx.gen_workload(S, DH, h_kv=H, g=1, kind="gaussian", seed=3)
mids = keys[:, 4:4 + S - 68].contiguous()
cen, codes = ctx.pq_build(mids, 2, 6, 10, list(range(H)))
del mids
tabs = ctx.tuple_tables(codes, 6)
layer = pq.DecodeLayer(keys=keys, values=vals, centroids=cen, codes=codes, total=S, n_init=4, n_local=64, b=6,
                       tables=tabs)
K = round(S / 5)
hq = q.cpu().pin_memory()
ho = torch.empty_like(hq).pin_memory()
for _ in range(5):
    ctx.decode_host(layer, hq, ho, K)
N = 200
t0 = time.perf_counter()
for _ in range(N):
    ctx.decode_host(layer, hq, ho, K)
a = (time.perf_counter() - t0) / N * 1e6
t0 = time.perf_counter()
for _ in range(N):
    ctx.decode(layer, q, K)
    torch.cuda.synchronize()
b = (time.perf_counter() - t0) / N * 1e6
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(N):
    ctx.decode(layer, q, K)
e1.record()
torch.cuda.synchronize()
c = e0.elapsed_time(e1) / N * 1e3
t0 = time.perf_counter()
for _ in range(N):
    ctx.decode(layer, q, K)
host_only = (time.perf_counter() - t0) / N * 1e6
torch.cuda.synchronize()
print(f"decode_host {a:.1f} us/step | device decode + sync {b:.1f} | back-to-back (events) {c:.1f} | "
      f"host launch cost (no sync, queued) {host_only:.1f}")
