"""Decode / build timing for a BASELINE config.  Default: cfg5 per-GPU shape
(configs[4] at 8 GPUs): 16 (request, kv head) units x 128K context, m=4 b=8
(256 centroids), GQA g=4, top-k 1/10 + 4 init + 64 local.  cfg3 (one
Llama-3-8B layer): `8 131072 4 2 6 5 tables`.  Prints build time and decode
us/step (CUDA events).
  python tools/prof_cfg5.py [units] [s] [g] [m] [b] [ratio] [tables]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2407_12820_b200 as pq  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 16
S = int(sys.argv[2]) if len(sys.argv) > 2 else 131072
G = int(sys.argv[3]) if len(sys.argv) > 3 else 4
M = int(sys.argv[4]) if len(sys.argv) > 4 else 4
B = int(sys.argv[5]) if len(sys.argv) > 5 else 8
RATIO = int(sys.argv[6]) if len(sys.argv) > 6 else 10
TABLES = len(sys.argv) > 7 and sys.argv[7] == "tables"
DH, NI, NL = 128, 4, 64
K = round(S / RATIO)
SM = S - NI - NL
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev)
g.manual_seed(1)
keys = torch.empty((P, S, DH), device=dev)
for h in range(P):
    means = torch.randn((8, DH), generator=g, device=dev)
    keys[h] = means[torch.randint(0, 8, (S,), generator=g, device=dev)] + 0.5 * torch.randn((S, DH), generator=g, device=dev)
vals = torch.randn((P, S, DH), generator=g, device=dev)
q = torch.randn((P, G, DH), generator=g, device=dev)
ctx = pq.Context(0)
torch.cuda.synchronize()
t0 = time.perf_counter()
cen, codes = ctx.pq_build(keys[:, NI:NI + SM].contiguous(), M, B, 10, list(range(P)))
torch.cuda.synchronize()
print(f"build {P}x{SM} m{M}b{B}: {time.perf_counter() - t0:.3f} s")
tabs = ctx.tuple_tables(codes, B) if TABLES else None
layer = pq.DecodeLayer(keys=keys, values=vals, centroids=cen, codes=codes, total=S, n_init=NI, n_local=NL, b=B,
                       tables=tabs)
for i in range(3):
    ctx.decode(layer, q, K)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 50
e0.record()
for i in range(reps):
    ctx.decode(layer, q, K)
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3 / reps
t_att = NI + K + NL
byts = P * (SM * M * B / 8 + (1 << B) * DH * 4 + t_att * DH * 8 + 2 * G * DH * 4)
print(f"decode {P} units x {S} m{M}b{B} g{G} k{K}: {us:.1f} us/step, {byts / us / 1e3:.0f} GB/s algorithmic "
      f"({byts / 1e6:.1f} MB), launches {layer.launches(G)}")
bm, _ = ctx.pq_search(q, cen, codes, B, K, s=SM, ordered=False)
e0.record()
for i in range(reps):
    ctx.pq_search(q, cen, codes, B, K, s=SM, ordered=False)
e1.record()
torch.cuda.synchronize()
print(f"  select alone: {e0.elapsed_time(e1) * 1e3 / reps:.1f} us")
e0.record()
for i in range(reps):
    ctx.decode_attend(layer, q, bm)
e1.record()
torch.cuda.synchronize()
print(f"  attend alone: {e0.elapsed_time(e1) * 1e3 / reps:.1f} us")
import numpy as np  # noqa: E402

ctx.set_profiling(True)
for i in range(3):
    ctx.decode(layer, q, K)
torch.cuda.synchronize()
raw = ctx.decode_profile_raw().astype(np.int64)
ctx.set_profiling(False)
raw = raw[raw[:, 4] > 0]
t0 = raw[:, 4].min()
pct = lambda v: [round(float(np.percentile(v, x)) / 1e3, 1) for x in (0, 10, 50, 90, 100)]
print(f"  timeline us (p0/p10/p50/p90/p100 over {len(raw)} CTAs):")
print("    start      ", pct(raw[:, 4] - t0))
print("    rows ready ", pct(raw[:, 5] - t0))
print("    gather done", pct(raw[:, 6] - t0))
print("    exit       ", pct(raw[:, 7] - t0))
cy = lambda a, b: [round(float(np.percentile(raw[:, b] - raw[:, a], x)) / 1965.0, 2) for x in (10, 50, 90)]
print("    select (clock) us", cy(0, 1), "words->rows", cy(1, 2), "gather", cy(2, 3))
print("    SMs used", len(set(raw[:, 16].tolist())))
names = ["start->lut", "keys", "B0", "hist0", "A0", "merge0", "B0'", "rest passes"]
print("    select phases us (median):", {nm: cy(a_, b_)[1] for nm, a_, b_ in
      [("lut", 0, 8), ("scores+hist0", 8, 9), ("barrier0", 9, 10), ("locate0", 10, 11), ("refine", 11, 12),
       ("words scan", 12, 13), ("cand barrier", 13, 14), ("gather+K*", 14, 15), ("patch", 15, 1)]})
print("    select phases us p10/p50/p90:", {nm: cy(a_, b_) for nm, a_, b_ in
      [("scores+hist0", 8, 9), ("barrier0", 9, 10), ("words scan", 12, 13), ("cand barrier", 13, 14),
       ("gather+K*", 14, 15), ("patch", 15, 1)]})
if os.environ.get("PQKV_PROF_SELECT"):
    nvs = raw[:, 21] & 0xff
    print("    value passes", np.bincount(nvs.astype(np.int64)).tolist(), "cand_ok", int(((raw[:, 21] >> 8) & 1).sum()),
          "of", len(raw), "final-bin count p50/p100", int(np.median(raw[:, 23])), int(raw[:, 23].max()),
          "T p50/p100", int(np.median(raw[:, 22])), int(raw[:, 22].max()))

