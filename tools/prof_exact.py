"""Device time of the fp64 attention path (exact_scores + softmax_weights +
weighted_products + sum_chain, pqkv_attend_rows PQKV_PREC_F64) on one head, warm loop.
Usage: python tools/prof_exact.py [t=6622] [S=32768] [P=1] [g=1]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2407_12820_b200 as pq  # noqa: E402

t = int(sys.argv[1]) if len(sys.argv) > 1 else 6622
S = int(sys.argv[2]) if len(sys.argv) > 2 else 32768
P = int(sys.argv[3]) if len(sys.argv) > 3 else 1
g = int(sys.argv[4]) if len(sys.argv) > 4 else 1
ctx = pq.Context(0)
dev = torch.device("cuda:0")
gen = torch.Generator(device=dev).manual_seed(1)
k = torch.randn((P, S, 128), device=dev, generator=gen)
v = torch.randn((P, S, 128), device=dev, generator=gen)
q = torch.randn((P, g, 128), device=dev, generator=gen)
rows = torch.stack([torch.randperm(S, device=dev, generator=gen)[:t].sort().values for _ in range(P)])
for prec, name in ((pq.PREC_F64, "f64"), (pq.PREC_F32, "f32")):
    for _ in range(20):
        ctx.attend_rows(q, k, v, rows, precision=prec)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 200
    e0.record()
    for _ in range(n):
        ctx.attend_rows(q, k, v, rows, precision=prec)
    e1.record()
    torch.cuda.synchronize()
    print(f"{name}: P={P} g={g} t={t}: {e0.elapsed_time(e1) / n * 1e3:.1f} us/call")
