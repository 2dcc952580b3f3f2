"""GPU parity: decode retrieval (ADC scores, top-k, fused search, attention,
fused decode) against the CPU oracle on the same seeded inputs.

Bars (BASELINE.json north_star): scores, top-k index sets and their order
bit-exact; attention within 1e-3 relative on the fp32 fast path and within
1e-6 (doctest-style mixed abs/rel, attention tests in the reference) on the
fp64 path."""
import numpy as np
from _util import rel_err
import pytest

import oracle

pytestmark = pytest.mark.gpu


def _t(a, dtype=None):
    import torch

    t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.cuda()


def _u16_as_i16(codes):
    return np.ascontiguousarray(codes).view(np.int16)


@pytest.fixture(scope="module")
def index4k(orc):
    """cfg1-like head set: 3 heads x 4096 keys, m2b6, T=10 (oracle-built)."""
    k, v, q = orc.gen_workload(4096, 128, 3, 4, oracle.POWERLAW, seed=7)
    cen, codes = [], []
    for h in range(3):
        c, cd = orc.pq_construct(k[h], 2, 6, 10, 100 + h)
        cen.append(c)
        codes.append(cd)
    return k, v, q, np.stack(cen), np.stack(codes)


@pytest.mark.parametrize("g", [1, 4])
def test_pq_score_bit_exact(ctx, orc, index4k, g):
    k, v, q, cen, codes = index4k
    got = ctx.pq_score(_t(q[:, :g]), _t(cen), _t(_u16_as_i16(codes)), 6).cpu().numpy()
    for h in range(3):
        want = orc.pq_score_gqa(q[h, :g], cen[h], codes[h])
        assert np.array_equal(got[h].view(np.uint32), want.view(np.uint32))


@pytest.mark.parametrize("m,b,d_h,s", [(4, 8, 128, 2048), (1, 3, 16, 300), (8, 2, 32, 777), (2, 10, 64, 1500)])
def test_pq_score_geometries(ctx, orc, m, b, d_h, s):
    rng = np.random.default_rng(m * 100 + b)
    C = 1 << b
    cen = rng.standard_normal((1, m, C, d_h // m)).astype(np.float32)
    codes = rng.integers(0, C, size=(1, s, m)).astype(np.uint16)
    q = rng.standard_normal((1, 3, d_h)).astype(np.float32)
    got = ctx.pq_score(_t(q), _t(cen), _t(_u16_as_i16(codes)), b).cpu().numpy()[0]
    want = orc.pq_score_gqa(q[0], cen[0], codes[0])
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


def test_hand_worked_score_and_cancellation(ctx, orc):
    # test_pq.cpp:61-72: identity codebooks, q = 1 -> score 2.0
    cen = np.array([1, 0, 0, 1, 1, 0, 0, 1], np.float32).reshape(1, 2, 2, 2)
    codes = np.array([[[0, 1]]], np.uint16)
    q = np.ones((1, 1, 4), np.float32)
    assert ctx.pq_score(_t(q), _t(cen), _t(_u16_as_i16(codes)), 1).cpu().numpy()[0, 0] == 2.0
    # test_pq.cpp:108-118: opposed queries in one group cancel to exactly 0
    rng = np.random.default_rng(19)
    cen = rng.standard_normal((1, 2, 8, 4)).astype(np.float32)
    codes = rng.integers(0, 8, size=(1, 32, 2)).astype(np.uint16)
    q1 = rng.standard_normal(8).astype(np.float32)
    q = np.stack([q1, -q1])[None]
    sc = ctx.pq_score(_t(q), _t(cen), _t(_u16_as_i16(codes)), 3).cpu().numpy()
    assert np.all(sc == 0.0)


@pytest.mark.parametrize("n,k,levels", [(100, 50, 17), (4096, 819, 5), (131, 131, 3), (5000, 1, 1000),
                                        (40000, 8000, 64), (1, 1, 2)])
def test_topk_ties_bit_exact(ctx, orc, n, k, levels):
    rng = np.random.default_rng(n + k)
    scores = rng.integers(0, levels, size=(3, n)).astype(np.float32) - levels / 2
    scores[0, ::7] = -0.0  # -0.0 == +0.0 must tie (topk.cpp:17-22)
    got = ctx.topk(_t(scores), k).cpu().numpy()
    for r in range(3):
        want = orc.top_k_desc(scores[r], k)
        assert np.array_equal(got[r].astype(np.uint64), want)


def test_topk_exclusions_and_errors(ctx, orc):
    # test_model.cpp:160-167 / test_pq.cpp:198-202
    scores = np.array([[5, 4, 3, 2, 1]], np.float32)
    ex = np.zeros((1, 5), np.uint8)
    ex[0, [0, 2]] = 1
    got = ctx.topk(_t(scores), 2, _t(ex)).cpu().numpy()[0]
    assert list(got) == [1, 3]
    with pytest.raises(ValueError):
        ctx.topk(_t(scores), 4, _t(ex))
    with pytest.raises(ValueError):
        ctx.topk(_t(scores), 6)
    assert ctx.topk(_t(scores), 0).shape == (1, 0)
    sc = np.array([[0.1, 0.9, 0.5, 0.9]], np.float32)
    assert list(ctx.topk(_t(sc), 2).cpu().numpy()[0]) == [1, 3]
    ex = np.array([[0, 1, 0, 0]], np.uint8)
    assert list(ctx.topk(_t(sc), 2, _t(ex)).cpu().numpy()[0]) == [3, 2]


@pytest.mark.parametrize("k", [1, 205, 819, 4096])
def test_fused_search_matches_score_then_topk(ctx, orc, index4k, k):
    k_, v, q, cen, codes = index4k
    bm, ids = ctx.pq_search(_t(q), _t(cen), _t(_u16_as_i16(codes)), 6, k)
    ids = ids.cpu().numpy()
    bm = bm.cpu().numpy().view(np.uint32)
    for h in range(3):
        want = orc.top_k_desc(orc.pq_score_gqa(q[h], cen[h], codes[h]), k)
        assert np.array_equal(ids[h].astype(np.uint64), want)
        bits = np.unpackbits(bm[h].view(np.uint8), bitorder="little")[:4096]
        assert np.array_equal(np.flatnonzero(bits), np.sort(want).astype(np.int64))


@pytest.mark.parametrize("k", [1, 205, 819, 4096])
def test_tuple_search_matches_score_then_topk(ctx, orc, index4k, k):
    """m == 2 code-pair path: weighted pair radix select + chunked bitmap."""
    k_, v, q, cen, codes = index4k
    dc = _t(_u16_as_i16(codes))
    tables = ctx.tuple_tables(dc, 6)
    bm, ids = ctx.pq_search(_t(q), _t(cen), dc, 6, k, tables=tables)
    ids = ids.cpu().numpy()
    bm = bm.cpu().numpy().view(np.uint32)
    for h in range(3):
        want = orc.top_k_desc(orc.pq_score_gqa(q[h], cen[h], codes[h]), k)
        assert np.array_equal(ids[h].astype(np.uint64), want)
        bits = np.unpackbits(bm[h].view(np.uint8), bitorder="little")[:4096]
        assert np.array_equal(np.flatnonzero(bits), np.sort(want).astype(np.int64))


@pytest.mark.parametrize("s,k,b,C_used", [(37, 10, 6, 64), (20000, 4000, 6, 3), (9000, 8999, 4, 16),
                                          (32700, 6554, 6, 64), (12345, 100, 7, 128), (5000, 2500, 1, 2)])
def test_tuple_search_ties_and_chunks(ctx, orc, s, k, b, C_used):
    """Heavy ties (few distinct pairs), boundaries spanning chunks, incremental tables."""
    rng = np.random.default_rng(s + k)
    C = 1 << b
    cen = rng.standard_normal((2, 2, C, 64)).astype(np.float32)
    codes = rng.integers(0, C_used, size=(2, s, 2)).astype(np.uint16)
    q = rng.standard_normal((2, 2, 128)).astype(np.float32)
    dc = _t(_u16_as_i16(codes))
    half = s // 2
    tables = ctx.tuple_tables(dc, b, s=half)
    tables = ctx.tuple_tables(dc, b, s=s, tables=tables, row_begin=half)  # append path
    bm, ids = ctx.pq_search(_t(q), _t(cen), dc, b, k, tables=tables)
    ids = ids.cpu().numpy()
    for h in range(2):
        want = orc.top_k_desc(orc.pq_score_gqa(q[h], cen[h], codes[h]), k)
        assert np.array_equal(ids[h].astype(np.uint64), want)


def test_fused_search_ragged_and_large(ctx, orc):
    """s not a multiple of 32 or of the cluster slice; 32K tokens, tie-heavy m2b6."""
    rng = np.random.default_rng(5)
    for s, k in [(37, 10), (1000, 999), (32700, 6554)]:
        cen = rng.standard_normal((2, 2, 64, 64)).astype(np.float32)
        codes = rng.integers(0, 64, size=(2, s, 2)).astype(np.uint16)
        q = rng.standard_normal((2, 1, 128)).astype(np.float32)
        bm, ids = ctx.pq_search(_t(q), _t(cen), _t(_u16_as_i16(codes)), 6, k)
        ids = ids.cpu().numpy()
        for h in range(2):
            want = orc.top_k_desc(orc.pq_score_gqa(q[h], cen[h], codes[h]), k)
            assert np.array_equal(ids[h].astype(np.uint64), want)


_rel = rel_err


@pytest.mark.parametrize("d_h,t,g", [(8, 50, 1), (128, 1000, 1), (128, 5000, 4), (6, 30, 3), (64, 300, 2)])
def test_attend_rows_f64_matches_reference(ctx, orc, d_h, t, g):
    rng = np.random.default_rng(d_h + t)
    S = t + 17
    keys = rng.standard_normal((1, S, d_h)).astype(np.float32)
    vals = rng.standard_normal((1, S, d_h)).astype(np.float32)
    q = rng.standard_normal((1, g, d_h)).astype(np.float32)
    rows = np.sort(rng.choice(S, size=t, replace=False)).astype(np.int64)[None]
    got = ctx.attend_rows(_t(q), _t(keys), _t(vals), _t(rows), precision=1).cpu().numpy()
    for r in range(g):
        want = orc.softmax_attention(q[0, r], keys[0], vals[0], rows[0].astype(np.uint64))
        np.testing.assert_allclose(got[0, r], want, rtol=1e-6, atol=1e-6)
    # scores are bit-identical to exact_scores (attention.cpp:11-26)
    sc = ctx.exact_scores(_t(q), _t(keys), _t(rows)).cpu().numpy()
    want_sc = orc.exact_scores(q[0, 0], keys[0][rows[0]])
    assert np.array_equal(sc[0, 0].view(np.uint32), want_sc.view(np.uint32))


@pytest.mark.parametrize("t,g", [(1, 1), (3000, 1), (10000, 4), (9000, 2)])
def test_attend_rows_f32_fast_path(ctx, orc, t, g):
    rng = np.random.default_rng(t)
    S = t + 100
    keys = rng.standard_normal((2, S, 128)).astype(np.float32)
    vals = rng.standard_normal((2, S, 128)).astype(np.float32)
    q = rng.standard_normal((2, g, 128)).astype(np.float32)
    rows = np.stack([np.sort(rng.choice(S, size=t, replace=False)) for _ in range(2)]).astype(np.int64)
    got = ctx.attend_rows(_t(q), _t(keys), _t(vals), _t(rows), precision=0).cpu().numpy()
    for p in range(2):
        for r in range(g):
            want = orc.softmax_attention(q[p, r], keys[p], vals[p], rows[p].astype(np.uint64))
            assert _rel(got[p, r], want) < 1e-3


def _decode_case(orc, s, h, g, n_init, n_local, k, m=2, b=6, seed=3, T=6, tuple_tables=False, ctx=None):
    import paper_2407_12820_b200 as pq

    kk, vv, qq = orc.gen_workload(s, 128, h, g, oracle.POWERLAW, seed=seed)
    s_mid = s - n_init - n_local
    cen = np.zeros((h, m, 1 << b, 128 // m), np.float32)
    codes = np.zeros((h, s_mid, m), np.uint16)
    for p in range(h):
        c, cd = orc.pq_construct(kk[p, n_init:n_init + s_mid], m, b, T, 11 + p)
        cen[p], codes[p] = c, cd
    dc = _t(_u16_as_i16(codes))
    tables = ctx.tuple_tables(dc, b) if tuple_tables else None
    layer = pq.DecodeLayer(keys=_t(kk), values=_t(vv), centroids=_t(cen), codes=dc,
                           total=s, n_init=n_init, n_local=n_local, b=b, tables=tables)
    return kk, vv, qq, cen, codes, layer


@pytest.mark.parametrize("tup", [False, True])
@pytest.mark.parametrize("s,h,g,n_init,n_local,k", [(4096, 3, 1, 4, 64, 819), (2000, 2, 4, 16, 64, 300),
                                                    (700, 2, 2, 0, 1, 50), (9000, 2, 1, 4, 64, 1800),
                                                    (24000, 1, 1, 4, 64, 4800), (20000, 1, 4, 16, 64, 100)])
def test_fused_decode_matches_reference_pipeline(ctx, orc, s, h, g, n_init, n_local, k, tup):
    kk, vv, qq, cen, codes, layer = _decode_case(orc, s, h, g, n_init, n_local, k, tuple_tables=tup, ctx=ctx)
    out, ids = ctx.decode(layer, _t(qq), k, want_ids=True)
    out, ids = out.cpu().numpy(), ids.cpu().numpy()
    for p in range(h):
        # experiments.cpp:218-260: score -> approx_topk -> token ids -> selective_attention
        rows = orc.top_k_desc(orc.pq_score_gqa(qq[p], cen[p], codes[p]), k)
        assert np.array_equal(ids[p].astype(np.uint64), rows)
        for r in range(g):
            want = orc.selective_attention(qq[p, r], kk[p], vv[p], n_init, n_local, rows + n_init)
            assert _rel(out[p, r], want) < 1e-3


def test_decode_host_buffers(ctx, orc):
    import torch

    kk, vv, qq, cen, codes, layer = _decode_case(orc, 3000, 2, 1, 4, 64, 500, tuple_tables=True, ctx=ctx)
    hq = torch.from_numpy(qq).pin_memory()
    ho = torch.zeros_like(hq).pin_memory()
    ctx.decode_host(layer, hq, ho, 500)
    dev = ctx.decode(layer, _t(qq), 500).cpu().numpy()
    assert np.array_equal(ho.numpy(), dev)


def test_encode_matches_reference(ctx, orc, index4k):
    import torch

    k_, v, q, cen, codes = index4k
    keys = k_[:, 123].copy()
    out = torch.zeros((3, 5, 2), dtype=torch.int16, device="cuda")
    ctx.pq_encode(_t(keys), _t(cen), 6, out, 2)
    got = out.cpu().numpy().view(np.uint16)
    for h in range(3):
        assert np.array_equal(got[h, 2], orc.pq_encode_one(keys[h], cen[h]))
        assert np.all(got[h, [0, 1, 3, 4]] == 0)
