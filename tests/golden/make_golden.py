"""Generates tests/golden/pqkv_golden.npz from the REFERENCE library itself
(oracle/_ref/libpqkv_ref.so, the unmodified /root/reference sources compiled
by oracle/Makefile).  Run in the CPU container:  python tests/golden/make_golden.py

The fixtures pin the C restatement (oracle/pqkv_oracle.c) and, through it,
the GPU parity tests; they are small enough to commit."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402


def main():
    ref = oracle.ref()
    out = {}
    for seed in (1, 7, 12345, 2**63 + 11):
        for kind in range(4):
            out[f"rng_{seed}_{kind}"] = ref.rng_stream(seed, 48, kind).view(np.uint64)
    for kind, name in ((oracle.GAUSSIAN, "gauss"), (oracle.POWERLAW, "power")):
        k, v, q = ref.gen_workload(96, 16, 2, 2, kind, seed=5)
        out[f"wl_{name}_k"], out[f"wl_{name}_v"], out[f"wl_{name}_q"] = k, v, q
        for h in range(2):
            cen, codes = ref.pq_construct(k[h], 2, 4, 10, 40 + h)
            out[f"pq_{name}_{h}_cen"], out[f"pq_{name}_{h}_codes"] = cen, codes
            sc = ref.pq_score_gqa(q[h], cen, codes)
            out[f"score_{name}_{h}"] = sc
            ids = ref.top_k_desc(sc, 20)
            out[f"topk_{name}_{h}"] = ids
            sel = ids[(ids >= 4) & (ids < 96 - 8)]
            out[f"sel_{name}_{h}"] = sel
            out[f"attn_{name}_{h}"] = np.stack(
                [ref.selective_attention(q[h, r], k[h], v[h], 4, 8, sel) for r in range(2)])
    rng = np.random.default_rng(0)
    pts = rng.standard_normal((150, 3)).astype(np.float32)
    cen, asg, tr, it = ref.kmeans_fit(pts, 7, 20, 31)
    out.update(km_pts=pts, km_cen=cen, km_asg=asg, km_trace=tr, km_iters=np.array([it]))
    tie = np.array([3, 1, 3, 0, 2, 2, 3, -0.0, 0.0], np.float32)
    out["tie_scores"] = tie
    out["tie_top5"] = ref.top_k_desc(tie, 5)
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "pqkv_golden.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes,", len(out), "arrays")


if __name__ == "__main__":
    main()
