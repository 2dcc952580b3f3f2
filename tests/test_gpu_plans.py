"""Selection-exact parity at the exact geometries bench.py measures.

Each case builds one layer of a bench config the way bench.py does
(`bench.make_layer`: device-generated gaussian-mixture or powerlaw K/V, GPU
PQ build with T = 10, code-pair tables), asserts that pqkv_decode picks the
launch plan the bench runs (mode, CTA chunking, cluster, staging, window),
runs one fused decode with the selection-dump hook on, and checks sampled
heads against the oracle: the selection words equal approx_topk's set
(topk.cpp:17-22 tie rule; pq.cpp:128-161 scores) and every query row's output
is within 1e-3 relative of selective_attention (attention.cpp:62-104) over
init ++ selected ++ local.  One headline head's index is also rebuilt by the
oracle (pq_construct, pq.cpp:42-72) and compared bit for bit."""
import os
import sys

import numpy as np
import pytest
from _util import REL_TOL, rel_err, selected_rows

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

pytestmark = pytest.mark.gpu

# The plan each config runs on one B200 (148 SMs); bench.py reports the same
# dict under plan / configs.<name>.plan.
EXPECT = {
    # g = 1: pair-select launch + attention launch (codes staged while the select runs)
    "northstar": dict(mode="pairs_split", launches=2, chunk_tokens=7296, ctas_per_head=18, cluster=1, staged=1,
                      window=7296),
    "cfg1": dict(mode="pairs_split", launches=2),
    "cfg2": dict(mode="pairs_split", launches=2, chunk_tokens=2048, ctas_per_head=16, cluster=1, staged=1),
    # g > 1: wide plan, one 1024-thread CTA per SM (148 // 8 = 18 per head), each selecting on its own
    "cfg3_layer": dict(mode="pairs_fused", launches=1, chunk_tokens=7296, ctas_per_head=18, cluster=1, staged=0),
    "cfg5_per_gpu": dict(mode="keys_split", launches=2),
}


def _check_layer(ctx, orc, name, kind, seed, heads=4, check_build=False):
    import torch

    c = bench.CONFIGS[name]
    g, k = c["g"], bench.cfg_k(c)
    s_mid = c["s"] - bench.N_INIT - bench.N_LOCAL
    layer, q, _ = bench.make_layer(ctx, name, kind, seed=seed)
    plan = ctx.decode_plan(layer, g, k)
    want_plan = EXPECT[name]
    assert {key: plan[key] for key in want_plan} == want_plan, f"{name}: plan {plan}"
    words = torch.zeros((c["units"], (s_mid + 31) // 32), dtype=torch.int32, device="cuda")
    ctx.set_selection_dump(words)
    try:
        out = ctx.decode(layer, q, k)
    finally:
        ctx.set_selection_dump(None)
    torch.cuda.synchronize()
    out = out.cpu().numpy()
    bits = words.cpu().numpy()
    qh = q.cpu().numpy()
    P = c["units"]
    sample = sorted({0, P // 3, (2 * P) // 3, P - 1})[:heads]
    for p in sample:
        cen = layer.centroids[p].cpu().numpy()
        codes = layer.codes[p].cpu().numpy().view(np.uint16)
        rows = orc.top_k_desc(orc.pq_score_gqa(qh[p], cen, codes), k)
        assert np.array_equal(selected_rows(bits[p], s_mid), np.sort(rows).astype(np.int64)), \
            f"{name}/{kind} head {p}: selection differs"
        kh, vh = layer.keys[p].cpu().numpy(), layer.values[p].cpu().numpy()
        for r in range(g):
            want = orc.selective_attention(qh[p, r], kh, vh, bench.N_INIT, bench.N_LOCAL, rows + bench.N_INIT)
            e = rel_err(out[p, r], want)
            assert e < REL_TOL, f"{name}/{kind} head {p} row {r}: rel err {e}"
    if check_build:
        p = sample[0]
        kh = layer.keys[p].cpu().numpy()
        mids = np.ascontiguousarray(kh[bench.N_INIT:bench.N_INIT + s_mid])
        want_cen, want_codes = orc.pq_construct(mids, c["m"], c["b"], bench.T_ITERS, 7 + 131 * seed + p)
        assert np.array_equal(layer.codes[p].cpu().numpy().view(np.uint16), want_codes), "codes differ"
        assert np.array_equal(layer.centroids[p].cpu().numpy(), want_cen), "centroids differ"
    return plan


@pytest.mark.parametrize("kind", ["gaussian", "powerlaw"])
def test_northstar_plan_selection_exact(ctx, orc, kind):
    _check_layer(ctx, orc, "northstar", kind, seed=3, check_build=(kind == "gaussian"))


@pytest.mark.parametrize("name,kind", [("cfg1", "gaussian"), ("cfg2", "gaussian"), ("cfg2", "powerlaw"),
                                       ("cfg3_layer", "gaussian"), ("cfg3_layer", "powerlaw"),
                                       ("cfg5_per_gpu", "gaussian"), ("cfg5_per_gpu", "powerlaw")])
def test_config_plan_selection_exact(ctx, orc, name, kind):
    _check_layer(ctx, orc, name, kind, seed=4)
