"""GPU parity: prefill PQ build (kmeans_fit, pq_construct, assign_nearest)
against the CPU oracle.  Codes / assignments / iteration counts / inertia
traces are bit-exact; centroids are the reference's fp64 means rounded once
to f32, so they are compared bit-exactly as well (north star allows 1e-3)."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

MODES = ["filtered", "exact", "filtered_v1"]


def _t(a):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.fixture(params=MODES)
def mode_ctx(ctx, request):
    """filtered: cluster-split v2 kernel (default); filtered_v1: one CTA per
    problem; exact: fp64 assign everywhere (v1)."""
    import os

    import paper_2407_12820_b200 as pq

    ctx.set_assign_mode(pq.ASSIGN_EXACT if request.param == "exact" else pq.ASSIGN_FILTERED)
    if request.param == "filtered_v1":
        os.environ["PQKV_KMEANS_V1"] = "1"
    yield ctx
    os.environ.pop("PQKV_KMEANS_V1", None)
    ctx.set_assign_mode(pq.ASSIGN_FILTERED)


def _check_kmeans(ctx, orc, pts, k, T, seed):
    cen, asg, its, inr = ctx.kmeans_fit(_t(pts[None]), k, T, [seed], inertia=True)
    wc, wa, wt, wi = orc.kmeans_fit(pts, k, T, seed)
    assert int(its[0]) == wi
    assert np.array_equal(asg[0].cpu().numpy().astype(np.uint64), wa)
    assert np.array_equal(cen[0].cpu().numpy().view(np.uint32), wc.view(np.uint32))
    got_tr = inr[0, :wi].cpu().numpy()
    assert np.array_equal(got_tr.view(np.uint64), wt.view(np.uint64))


@pytest.mark.parametrize("n,dim,k", [(200, 4, 8), (300, 5, 10), (64, 3, 16), (500, 6, 7), (1000, 2, 33),
                                     (2000, 16, 64), (777, 32, 20), (4096, 64, 64), (1024, 8, 256)])
def test_kmeans_fit_bit_exact(mode_ctx, orc, n, dim, k):
    rng = np.random.default_rng(n * 7 + dim)
    pts = rng.standard_normal((n, dim)).astype(np.float32)
    _check_kmeans(mode_ctx, orc, pts, k, 25, n + k)


def test_kmeans_small_and_degenerate(mode_ctx, orc):
    # kmeans.cpp:44-57 seed_from_distinct (n <= k), duplicates, ties
    _check_kmeans(mode_ctx, orc, np.array([[0, 0], [5, 1], [-2, 4]], np.float32), 4, 10, 99)
    _check_kmeans(mode_ctx, orc, np.array([[2.0], [2.0], [7.0], [7.0]], np.float32), 2, 10, 5)
    _check_kmeans(mode_ctx, orc, np.zeros((50, 3), np.float32), 4, 5, 1)  # all coincide
    pts = np.repeat(np.random.default_rng(1).standard_normal((6, 4)).astype(np.float32), 40, axis=0)
    _check_kmeans(mode_ctx, orc, pts, 10, 8, 3)  # fewer distinct points than clusters -> repair
    pts = np.array([[-0.0, 1.0], [0.0, 1.0], [3.0, 3.0]], np.float32)  # memcmp: -0.0 != +0.0
    _check_kmeans(mode_ctx, orc, pts, 3, 4, 2)
    _check_kmeans(mode_ctx, orc, np.array([[1.0, 2.0]], np.float32), 1, 3, 7)


def test_kmeans_blobs_and_batch(mode_ctx, orc):
    rng = np.random.default_rng(4242)
    Q, n, dim = 5, 400, 8
    pts = np.concatenate([1.5 + 0.5 * rng.standard_normal((Q, n // 2, dim)),
                          -1.5 + 0.5 * rng.standard_normal((Q, n // 2, dim))], axis=1).astype(np.float32)
    seeds = [7 + q for q in range(Q)]
    cen, asg, its, _ = mode_ctx.kmeans_fit(_t(pts), 2, 50, seeds)
    for q in range(Q):
        wc, wa, wt, wi = orc.kmeans_fit(pts[q], 2, 50, seeds[q])
        assert np.array_equal(asg[q].cpu().numpy().astype(np.uint64), wa)
        assert np.array_equal(cen[q].cpu().numpy(), wc)
        assert int(its[q]) == wi


@pytest.mark.parametrize("s,d_h,m,b,T", [(4096, 128, 2, 6, 10), (2048, 128, 4, 8, 10), (256, 32, 1, 4, 8),
                                         (96, 32, 4, 4, 10), (16, 8, 2, 4, 10), (1, 8, 2, 4, 5),
                                         (70, 16, 4, 5, 12), (300, 12, 3, 3, 10), (500, 64, 2, 9, 4)])
def test_pq_construct_bit_exact(mode_ctx, orc, s, d_h, m, b, T):
    kind = oracle.POWERLAW if s % 2 == 0 else oracle.GAUSSIAN
    k, _, _ = orc.gen_workload(s, d_h, 2, 1, kind, seed=s + m)
    seeds = [1234 + s, 99 + b]
    cen, codes = mode_ctx.pq_build(_t(k), m, b, T, seeds)
    cen, codes = cen.cpu().numpy(), codes.cpu().numpy().view(np.uint16)
    for h in range(2):
        wc, wcd = orc.pq_construct(k[h], m, b, T, seeds[h])
        assert np.array_equal(codes[h], wcd)
        assert np.array_equal(cen[h].view(np.uint32), wc.view(np.uint32))


@pytest.mark.parametrize("s,kind", [(32768, oracle.POWERLAW), (20000, oracle.GAUSSIAN)])
def test_pq_construct_cluster_split_large(ctx, orc, s, kind):
    """v2 with an 8-CTA cluster per problem on realistic keys (gaussian mixture
    of the e2e workload and the powerlaw profile), m2b6 and m4b8."""
    k, _, _ = orc.gen_workload(s, 128, 1, 1, kind, seed=s)
    for m, b in [(2, 6), (4, 8)]:
        cen, codes = ctx.pq_build(_t(k), m, b, 10, [s + m])
        wc, wcd = orc.pq_construct(k[0], m, b, 10, s + m)
        assert np.array_equal(codes[0].cpu().numpy().view(np.uint16), wcd)
        assert np.array_equal(cen[0].cpu().numpy(), wc)


def test_pq_construct_32k_powerlaw(ctx, orc):
    """The survey's hard case: at 32K an uncertified fp32 assign flips codes;
    the certified filter must not (SURVEY.md 8(a'))."""
    k, _, _ = orc.gen_workload(32768, 128, 1, 1, oracle.POWERLAW, seed=7)
    cen, codes = ctx.pq_build(_t(k), 2, 6, 10, [77])
    wc, wcd = orc.pq_construct(k[0], 2, 6, 10, 77)
    assert np.array_equal(codes[0].cpu().numpy().view(np.uint16), wcd)
    assert np.array_equal(cen[0].cpu().numpy(), wc)
    rechecked, total = ctx.last_build_stats()
    assert total > 0 and rechecked < 0.01 * total


def test_assign_nearest(ctx, orc):
    rng = np.random.default_rng(3)
    pts = rng.standard_normal((3000, 5)).astype(np.float32)
    cen = rng.standard_normal((17, 5)).astype(np.float32)
    cen[5] = cen[3]  # duplicate centroid -> ties to the lower index
    got = ctx.assign_nearest(_t(pts), _t(cen)).cpu().numpy()
    assert np.array_equal(got.astype(np.uint64), orc.assign_nearest(pts, cen))
    # kmeans.cpp:192-220 tie example from test_kmeans.cpp:146-156
    got = ctx.assign_nearest(_t(np.array([[1.0], [3.0]], np.float32)),
                             _t(np.array([[0.0], [2.0], [2.0]], np.float32))).cpu().numpy()
    assert list(got) == [0, 1]


def test_build_errors(ctx):
    import torch

    k = torch.zeros((1, 10, 128), device="cuda")
    with pytest.raises(ValueError):
        ctx.pq_build(k, 3, 6, 10, [1])  # 128 % 3 != 0
    with pytest.raises(ValueError):
        ctx.pq_build(k, 2, 17, 10, [1])
    with pytest.raises(ValueError):
        ctx.pq_build(k, 2, 6, 0, [1])
    pts = torch.zeros((1, 4, 2), device="cuda")
    with pytest.raises(ValueError):
        ctx.kmeans_fit(pts, 0, 5, [1])


def test_pq_construct_many_heads_cluster_of_four(ctx, orc):
    """The bench geometry's cluster split: 32 heads x 2 subspaces at 2 CTAs/SM
    -> 4-CTA clusters per problem; sampled heads vs the oracle."""
    import torch

    P, s = 32, 16384
    keys, _, _ = orc.gen_workload(s, 128, P, 1, oracle.GAUSSIAN, seed=31)
    cen, codes = ctx.pq_build(torch.from_numpy(keys).cuda(), 2, 6, 6, [100 + p for p in range(P)])
    cen, codes = cen.cpu().numpy(), codes.cpu().numpy().view(np.uint16)
    for p in (0, 13, 31):
        wc, wcd = orc.pq_construct(keys[p], 2, 6, 6, 100 + p)
        assert np.array_equal(codes[p], wcd), f"head {p}: codes"
        assert np.array_equal(cen[p], wc), f"head {p}: centroids"
