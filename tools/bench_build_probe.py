import sys, time, torch
sys.path.insert(0, "/root/repo")
import paper_2407_12820_b200 as pq
ctx = pq.Context(0)
S, H = 131072, 32
for li in range(4):
    keys, vals, q = ctx.gen_workload(S, 128, h_kv=H, g=1, kind="gaussian", seed=li)
    mids = keys[:, 4:4 + S - 68].contiguous()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    cen, codes = ctx.pq_build(mids, 2, 6, 10, [7 + h for h in range(H)])
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    tabs = ctx.tuple_tables(codes, 6)
    torch.cuda.synchronize()
    print(li, "build", round(t1 - t0, 4), "tables", round(time.perf_counter() - t1, 4), ctx.last_build_stats(), flush=True)
    del mids
