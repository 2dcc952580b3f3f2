"""Device-timed us/layer of bench configs (4 rotating layers, 300 decodes)
for quick A/B runs.  Usage: python tools/quick_times.py cfg3_layer:gaussian [...]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2407_12820_b200 as pq  # noqa: E402

ctx = pq.Context(0)
for spec in sys.argv[1:]:
    name, kind = spec.split(":")
    c = bench.CONFIGS[name]
    k = bench.cfg_k(c)
    ls = [bench.make_layer(ctx, name, kind, seed=s)[:2] for s in range(4)]
    for i in range(20):
        ctx.decode(ls[i % 4][0], ls[i % 4][1], k)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for i in range(300):
        ctx.decode(ls[i % 4][0], ls[i % 4][1], k)
    e1.record()
    torch.cuda.synchronize()
    print(f"{name:14s} {kind:9s} {e0.elapsed_time(e1) / 300 * 1e3:7.1f} us/layer")
    del ls
    torch.cuda.empty_cache()
