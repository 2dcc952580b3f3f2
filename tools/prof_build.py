"""Profiling driver for the PQ build: P heads x s tokens (gaussian mixture),
m2b6, T=10.  usage: python tools/prof_build.py [P] [s] [exact]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2407_12820_b200 as pq  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 2
S = int(sys.argv[2]) if len(sys.argv) > 2 else 131004
exact = len(sys.argv) > 3 and sys.argv[3] == "exact"
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev)
g.manual_seed(1)
keys = torch.empty((P, S, 128), device=dev)
for h in range(P):
    means = torch.randn((8, 128), generator=g, device=dev)
    keys[h] = means[torch.randint(0, 8, (S,), generator=g, device=dev)] + 0.5 * torch.randn((S, 128), generator=g, device=dev)
ctx = pq.Context(0)
if exact:
    ctx.set_assign_mode(pq.ASSIGN_EXACT)
torch.cuda.synchronize()
t0 = time.perf_counter()
cen, codes = ctx.pq_build(keys, 2, 6, 10, list(range(P)))
torch.cuda.synchronize()
first = time.perf_counter() - t0
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
cen, codes = ctx.pq_build(keys, 2, 6, 10, list(range(P)))
e1.record()
torch.cuda.synchronize()
print(f"build P={P} s={S} exact={exact}: first {first:.3f} s, warm {e0.elapsed_time(e1) / 1e3:.4f} s (events), "
      f"rechecked/total={ctx.last_build_stats()}")
prof = ctx.last_build_profile()
print("hamerly skipped point-visits:", prof.pop("skipped_points"), "k-means++ triangle-skipped:",
      prof.pop("seed_skipped_points"))
tot = sum(prof.values()) or 1
print("phase ms @1.965GHz:", {k: round(v / 1.965e6, 2) for k, v in prof.items()}, "share:",
      {k: round(v / tot, 3) for k, v in prof.items()})
