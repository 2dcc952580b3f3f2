"""Profiling driver (one GPU; run plain or under ncu): one layer of a bench
config built exactly as bench.py does (bench.make_layer), a few fused decodes
plus the split select / attend calls; with PQKV_PHASES=1 the per-CTA phase
timeline of the fused kernel.
Usage: python tools/prof_decode.py [config=northstar] [kind=gaussian] [reps=3]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2407_12820_b200 as pq  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "northstar"
kind = sys.argv[2] if len(sys.argv) > 2 else "gaussian"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
cfgd = bench.CONFIGS[name]
G, B, K = cfgd["g"], cfgd["b"], bench.cfg_k(cfgd)
SM = cfgd["s"] - bench.N_INIT - bench.N_LOCAL
ctx = pq.Context(0)
layer, q, _ = bench.make_layer(ctx, name, kind, seed=1)
cen, codes, tables = layer.centroids, layer.codes, layer.tables
print(name, kind, ctx.decode_plan(layer, G, K))
for i in range(reps):
    out = ctx.decode(layer, q + 0.01 * i, K)
bm, _ = ctx.pq_search(q, cen, codes, B, K, s=SM, ordered=False, tables=tables)
for i in range(reps):
    ctx.decode_attend(layer, q, bm)
torch.cuda.synchronize()
if os.environ.get("PQKV_PHASES"):
    ctx.set_profiling(True)
    for mode in ("fused", "bitmap"):
        for i in range(3):
            if mode == "fused":
                ctx.decode(layer, q, K)
            else:
                ctx.decode_attend(layer, q, bm)
        torch.cuda.synchronize()
        prof = ctx.last_decode_profile()
        print(mode, {k: (round(v / 1965.0, 2) if k != "ctas" else v) for k, v in prof.items()}, "(us)")
        raw = ctx.decode_profile_raw().astype(np.int64)
        raw = raw[raw[:, 4] > 0]
        t0 = raw[:, 4].min()
        pct = lambda v: [round(float(np.percentile(v, q)) / 1e3, 1) for q in (0, 10, 50, 90, 100)]
        print(f"  {mode} timeline us (p0/p10/p50/p90/p100 over {len(raw)} CTAs):")
        print("    start      ", pct(raw[:, 4] - t0))
        print("    rows ready ", pct(raw[:, 5] - t0))
        print("    gather done", pct(raw[:, 6] - t0))
        print("    exit       ", pct(raw[:, 7] - t0))
        print("    gather span", pct(raw[:, 6] - raw[:, 5]))
        if mode == "fused":
            from collections import Counter
            r0sm = Counter(raw[raw[:, 18] == 1][:, 16].tolist())
            allsm = Counter(raw[:, 16].tolist())
            print("  SMs used", len(allsm), "CTAs/SM", sorted(Counter(allsm.values()).items()),
                  "selector CTAs per SM", sorted(Counter(r0sm.values()).items()))
        if mode == "fused":
            cy = lambda a, b: [round(float(np.percentile(raw[:, b] - raw[:, a], q)) / 1965.0, 2) for q in (10, 50, 90, 100)]
            print("  non-selector phases us (p10/p50/p90/p100): sync->staged", cy(1, 19), "classify", cy(19, 20),
                  "expand", cy(20, 2))
        r0 = raw[raw[:, 8] > 0]
        if len(r0):
            cyc = lambda a, b: round(float(np.median(r0[:, b] - r0[:, a])) / 1965.0, 2)
            print("  pair_select phases, median us over", len(r0), "rank-0 CTAs: start->w+lut", cyc(0, 9),
                  "lut", cyc(8, 9), "keys", cyc(10, 11), "radix", cyc(11, 12), "classify", cyc(12, 13),
                  "chist", cyc(13, 14), "-> cluster.sync", cyc(14, 15), "-> dsmem+sync", cyc(15, 1))
    ctx.set_profiling(False)
print("done", out.abs().sum().item())
