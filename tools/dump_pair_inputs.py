"""Dumps the pair-select inputs of head 0 of one bench layer (queries,
centroids, pair histogram, chunk histograms, k) as raw little-endian files
for tools/microbench/pair_select_probe.cu.
Usage: python tools/dump_pair_inputs.py [config=northstar] [kind=powerlaw] [outdir=gpurun_out/pairdump]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_2407_12820_b200 as pq  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "northstar"
kind = sys.argv[2] if len(sys.argv) > 2 else "powerlaw"
out = sys.argv[3] if len(sys.argv) > 3 else os.path.join(ROOT, "gpurun_out", "pairdump")
os.makedirs(out, exist_ok=True)
ctx = pq.Context(0)
layer, q, _ = bench.make_layer(ctx, name, kind, seed=1)
c = bench.CONFIGS[name]
th, ch = layer.tables
np.ascontiguousarray(q[0].cpu().numpy(), np.float32).tofile(os.path.join(out, "q.f32"))
np.ascontiguousarray(layer.centroids[0].cpu().numpy(), np.float32).tofile(os.path.join(out, "cen.f32"))
np.ascontiguousarray(th[0].cpu().numpy()).view(np.uint32).tofile(os.path.join(out, "thist.u32"))
np.ascontiguousarray(ch[0].cpu().numpy()).view(np.uint16).tofile(os.path.join(out, "chist.u16"))
with open(os.path.join(out, "meta.txt"), "w") as f:
    f.write(f"{c['g']} {ch.shape[1]} {bench.cfg_k(c)}\n")
print("dumped", out, "g", c["g"], "chunks", ch.shape[1], "k", bench.cfg_k(c), "nnz pairs",
      int((th[0] > 0).sum().item()))
