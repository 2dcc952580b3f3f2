import sys, time, ctypes as C
sys.path.insert(0, "/root/repo")
import torch
import paper_2407_12820_b200 as pq
ctx = pq.Context(0)
k, v, q = ctx.gen_workload(8192, 128, h_kv=2, g=1, seed=1)
cen, codes = ctx.pq_build(k[:, 4:8192-64].contiguous(), 2, 6, 4, [1, 2])
layer = pq.DecodeLayer(keys=k, values=v, centroids=cen, codes=codes, total=8192, n_init=4, n_local=64, b=6)
N = 20000
def t(f):
    t0 = time.perf_counter()
    for _ in range(N): f()
    return (time.perf_counter() - t0) / N * 1e6
print("_stream", t(pq._stream))
print("layer.ref", t(layer.ref))
print("_ptr", t(lambda: pq._ptr(q)))
L = layer.ref()
print("ctypes launches()", t(lambda: pq.lib().pqkv_decode_launches(L, 1, 0)))
print("torch.empty", t(lambda: torch.empty((2, 1, 128), device="cuda")))
hq = q.cpu().pin_memory(); ho = torch.empty_like(hq).pin_memory()
print("decode_host total", t(lambda: ctx.decode_host(layer, hq, ho, 100)))
