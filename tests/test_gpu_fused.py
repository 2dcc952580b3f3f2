"""GPU parity of the single-launch fused decodes (pqkv_decode without ids):
the code-pair path (m = 2, b <= 6 with pair tables) and the per-token key
path (any m, b with m * 2^b * 8 <= 16 KB, one thread-block cluster per head).
The selection words the kernel gathers from (test hook
pqkv_ctx_set_selection_dump) must equal the oracle's approx_topk set exactly
(topk.cpp tie rule), and the output must match selective_attention within
1e-3 relative (north star)."""
import numpy as np
from _util import rel_err
import pytest

import oracle

pytestmark = pytest.mark.gpu


_rel = rel_err


def _run(ctx, orc, cen, codes, keys, vals, qs, b, n_init, n_local, k, tables):
    import torch

    import paper_2407_12820_b200 as pq

    P, s_mid, m = codes.shape
    S = keys.shape[1]
    dc = torch.from_numpy(np.ascontiguousarray(codes).view(np.int16)).cuda()
    tabs = ctx.tuple_tables(dc, b) if tables else None
    layer = pq.DecodeLayer(keys=torch.from_numpy(keys).cuda(), values=torch.from_numpy(vals).cuda(),
                           centroids=torch.from_numpy(cen).cuda(), codes=dc, total=S, n_init=n_init,
                           n_local=n_local, b=b, tables=tabs)
    words = (s_mid + 31) // 32
    dump = torch.zeros((P, words), dtype=torch.int32, device="cuda")
    ctx.set_selection_dump(dump)
    try:
        out = ctx.decode(layer, torch.from_numpy(qs).cuda(), k).cpu().numpy()
    finally:
        ctx.set_selection_dump(None)
    pair_path = m == 2 and b <= 6 and tables
    g = qs.shape[1]
    # pair path: one launch for g > 1, a pair-select launch + the attention
    # for g = 1; key path: select + attention for g > 1 or when the per-head
    # cluster grid is too small for the gather, else one launch
    if pair_path:
        assert layer.launches(g) == (1 if g > 1 else 2)
    else:
        assert layer.launches(g) == 2 if g > 1 else layer.launches(g) in (1, 2)
    bits = dump.cpu().numpy().view(np.uint32)
    for p in range(P):
        rows = orc.top_k_desc(orc.pq_score_gqa(qs[p], cen[p], codes[p]), k)
        got = np.flatnonzero(np.unpackbits(bits[p].view(np.uint8), bitorder="little")[:s_mid])
        assert np.array_equal(got, np.sort(rows).astype(np.int64)), f"head {p}: selection differs"
        for r in range(g):
            want = orc.selective_attention(qs[p, r], keys[p], vals[p], n_init, n_local, rows + n_init)
            assert _rel(out[p, r], want) < 1e-3


@pytest.mark.parametrize("m,b,tables,s,P,g,k", [
    (2, 6, True, 20000, 3, 1, 4000),     # pair path
    (4, 8, False, 20000, 2, 4, 2000),    # cfg5 geometry (key path)
    (2, 7, True, 9000, 2, 2, 900),       # b = 7: key path even with tables
    (2, 6, False, 6000, 2, 1, 1200),     # no tables: key path
    (8, 4, False, 5000, 2, 1, 700),      # m = 8
    (4, 8, False, 131072, 1, 4, 13107),  # 16-CTA cluster, 128K
    (4, 8, False, 800, 2, 1, 5),         # one CTA per head, tiny k
    (4, 8, False, 131072, 2, 1, 65536),  # key path g = 1, 16K chunks: two gather windows per CTA
])
def test_fused_decode_selection_exact(ctx, orc, m, b, tables, s, P, g, k):
    import torch

    n_init, n_local = 4, 64
    keys, vals, qs = orc.gen_workload(s, 128, P, g, oracle.POWERLAW, seed=s + m)
    s_mid = s - n_init - n_local
    cen, codes = ctx.pq_build(torch.from_numpy(np.ascontiguousarray(keys[:, n_init:n_init + s_mid])).cuda(), m, b,
                              6, list(range(P)))
    _run(ctx, orc, cen.cpu().numpy(), codes.cpu().numpy().view(np.uint16), keys, vals, qs, b, n_init, n_local, k,
         tables)


@pytest.mark.parametrize("m,b,c_used", [(4, 8, 1), (4, 8, 3), (4, 8, 6), (4, 8, 12), (2, 6, 2)])
def test_fused_decode_heavy_ties(ctx, orc, m, b, c_used):
    """Few distinct codes: thousands of tokens share the threshold score (1 or
    3 of 256 codes used: the key path's value bins cannot split the threshold
    score's ties -- with one code every score is equal and the refined bin
    has zero width -- so its radix fallback runs); 6 or 12 codes: a handful
    of ties at K* inside a small final bin (the candidate path's tie order)."""
    rng = np.random.default_rng(c_used)
    P, s, n_init, n_local, k = 2, 12000, 4, 64, 3000
    s_mid = s - n_init - n_local
    C = 1 << b
    cen = rng.standard_normal((P, m, C, 128 // m)).astype(np.float32)
    codes = rng.integers(0, c_used, size=(P, s_mid, m)).astype(np.uint16)
    keys = rng.standard_normal((P, s, 128)).astype(np.float32)
    vals = rng.standard_normal((P, s, 128)).astype(np.float32)
    qs = rng.standard_normal((P, 1, 128)).astype(np.float32)
    _run(ctx, orc, cen, codes, keys, vals, qs, b, n_init, n_local, k, m == 2)


@pytest.mark.parametrize("g,ratio", [(1, 5), (2, 5), (1, 2)])
def test_fused_decode_many_heads_windowed(ctx, orc, g, ratio):
    """Many heads (80 x 64K): the plan picks chunks above 8192 tokens, so the
    pair path classifies from L2 and expands + gathers its rows in windows."""
    import torch

    import paper_2407_12820_b200 as pq

    P, S, n_init, n_local, m, b = 80, 65536, 4, 64, 2, 6
    k = S // ratio  # ratio 2: more selected rows per CTA than one window holds
    s_mid = S - n_init - n_local
    gen = torch.Generator(device="cuda")
    gen.manual_seed(7)
    keys = torch.randn((P, S, 128), generator=gen, device="cuda")
    keys[:, :, :8] += 2.0 * torch.randn((P, 1, 8), generator=gen, device="cuda")
    vals = torch.randn((P, S, 128), generator=gen, device="cuda")
    qs = torch.randn((P, g, 128), generator=gen, device="cuda")
    cen, codes = ctx.pq_build(keys[:, n_init:n_init + s_mid].contiguous(), m, b, 4, list(range(P)))
    tabs = ctx.tuple_tables(codes, b)
    layer = pq.DecodeLayer(keys=keys, values=vals, centroids=cen, codes=codes, total=S, n_init=n_init,
                           n_local=n_local, b=b, tables=tabs)
    words = (s_mid + 31) // 32
    dump = torch.zeros((P, words), dtype=torch.int32, device="cuda")
    ctx.set_selection_dump(dump)
    try:
        out = ctx.decode(layer, qs, k).cpu().numpy()
    finally:
        ctx.set_selection_dump(None)
    assert layer.launches(g) == (1 if g > 1 else 2)
    bits = dump.cpu().numpy().view(np.uint32)
    cen_h = cen.cpu().numpy()
    codes_h = codes.cpu().numpy().view(np.uint16)
    q_h = qs.cpu().numpy()
    for p in (0, 41, P - 1):
        rows = orc.top_k_desc(orc.pq_score_gqa(q_h[p], cen_h[p], codes_h[p]), k)
        got = np.flatnonzero(np.unpackbits(bits[p].view(np.uint8), bitorder="little")[:s_mid])
        assert np.array_equal(got, np.sort(rows).astype(np.int64)), f"head {p}: selection differs"
        kh, vh = keys[p].cpu().numpy(), vals[p].cpu().numpy()
        for r in range(g):
            want = orc.selective_attention(q_h[p, r], kh, vh, n_init, n_local, rows + n_init)
            assert _rel(out[p, r], want) < 1e-3
