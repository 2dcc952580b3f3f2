"""Profiling driver (run under ncu on one GPU): one north-star layer
(32 heads x 128K, m2b6, k=26214), a few fused decodes plus the split
select / attend calls.  Usage: python tools/prof_decode.py [reps] [heads] [s]"""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2407_12820_b200 as pq  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
H = int(sys.argv[2]) if len(sys.argv) > 2 else 32
S = int(sys.argv[3]) if len(sys.argv) > 3 else 131072
DH, G, M, B, NI, NL = 128, 1, 2, 6, 4, 64
K = round(S / 5)
SM = S - NI - NL
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev)
g.manual_seed(1)
keys = torch.empty((H, S, DH), device=dev)
for h in range(H):
    means = torch.randn((8, DH), generator=g, device=dev)
    keys[h] = means[torch.randint(0, 8, (S,), generator=g, device=dev)] + 0.5 * torch.randn((S, DH), generator=g, device=dev)
vals = torch.randn((H, S, DH), generator=g, device=dev)
q = torch.randn((H, G, DH), generator=g, device=dev)
ctx = pq.Context(0)
mode = os.environ.get("PQKV_BUILD", "filtered")
if mode == "exact":
    ctx.set_assign_mode(pq.ASSIGN_EXACT)
cen, codes = ctx.pq_build(keys[:, NI:NI + SM].contiguous(), M, B, 10, list(range(H)))
tables = ctx.tuple_tables(codes, B) if os.environ.get("PQKV_TUPLE", "1") == "1" else None
layer = pq.DecodeLayer(keys=keys, values=vals, centroids=cen, codes=codes, total=S, n_init=NI, n_local=NL, b=B,
                       tables=tables)
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
    ctx.set_profiling(False)
print("done", out.abs().sum().item())
