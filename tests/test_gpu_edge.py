"""GPU edge cases of the decode entry points.

* PqConfig allows b up to 16: with m * 2^b * 8 above 64 KB (b = 13 at
  m = 2) the ADC table does not fit shared memory; the selection then
  materialises the scores and selects over them -- the ordered ids must
  still equal approx_topk's (pq.cpp:113-177, topk.cpp tie rule).
* A rejected pqkv_decode_step (k beyond the grown middle segment) leaves
  the device state untouched: no K/V row written, no code row appended, no
  pair-table count added, total unchanged."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_decode_large_codebook_b13(ctx, orc):
    import torch

    import paper_2407_12820_b200 as pq

    rng = np.random.default_rng(13)
    P, S, n_init, n_local, m, b, k = 2, 9000, 4, 64, 2, 13, 900
    C = 1 << b
    s_mid = S - n_init - n_local
    cen = rng.standard_normal((P, m, C, 128 // m)).astype(np.float32)
    codes = rng.integers(0, C, size=(P, s_mid, m)).astype(np.uint16)
    keys = rng.standard_normal((P, S, 128)).astype(np.float32)
    vals = rng.standard_normal((P, S, 128)).astype(np.float32)
    qs = rng.standard_normal((P, 1, 128)).astype(np.float32)
    layer = pq.DecodeLayer(keys=torch.from_numpy(keys).cuda(), values=torch.from_numpy(vals).cuda(),
                           centroids=torch.from_numpy(cen).cuda(),
                           codes=torch.from_numpy(codes.view(np.int16)).cuda(), total=S, n_init=n_init,
                           n_local=n_local, b=b)
    out, ids = ctx.decode(layer, torch.from_numpy(qs).cuda(), k, want_ids=True)
    ids = ids.cpu().numpy()
    out = out.cpu().numpy()
    for p in range(P):
        want = orc.top_k_desc(orc.pq_score_gqa(qs[p], cen[p], codes[p]), k)
        assert np.array_equal(ids[p].astype(np.uint64), want)
        ref = orc.selective_attention(qs[p, 0], keys[p], vals[p], n_init, n_local, want + n_init)
        assert np.abs(out[p, 0] - ref).max() <= 1e-3 * np.abs(ref).max()


def test_rejected_decode_step_leaves_state(ctx):
    import torch

    import paper_2407_12820_b200 as pq

    P, S0, n_init, n_local, b = 2, 6000, 4, 64, 6
    keys, vals, q = ctx.gen_workload(S0 + 4, 128, h_kv=P, g=1, kind="gaussian", seed=3)
    s_mid = S0 - n_init - n_local
    cen, codes0 = ctx.pq_build(keys[:, n_init:n_init + s_mid].contiguous(), 2, b, 4, [1, 2])
    codes = torch.zeros((P, s_mid + 4, 2), dtype=torch.int16, device="cuda")
    codes[:, :s_mid] = codes0
    tabs = ctx.tuple_tables(codes, b, s=s_mid)
    keys[:, S0:] = 0
    vals[:, S0:] = 0
    layer = pq.DecodeLayer(keys=keys, values=vals, centroids=cen, codes=codes, total=S0, n_init=n_init,
                           n_local=n_local, b=b, tables=tabs)
    snap = [t.clone() for t in (keys, vals, codes, tabs[0], tabs[1])]
    nk = torch.randn((P, 128), device="cuda")
    with pytest.raises(ValueError):
        ctx.decode_step(layer, nk, nk, q, s_mid + 2)  # k > the grown middle segment (s_mid + 1)
    torch.cuda.synchronize()
    assert layer.total == S0
    for before, after in zip(snap, (keys, vals, codes, tabs[0], tabs[1])):
        assert torch.equal(before, after)
    # and a valid step afterwards appends exactly one token
    ctx.decode_step(layer, nk, nk, q, 500)
    torch.cuda.synchronize()
    assert layer.total == S0 + 1
    assert torch.equal(keys[:, S0], nk)


@pytest.mark.parametrize("g", [1, 4])
def test_decode_host_graph_replay(ctx, orc, g):
    """pqkv_decode_host replays a captured graph from the second call of the
    same (layer, buffers, g, k): new query contents in the same pinned buffer
    and a grown layer (decode step) must still give the plain decode's
    result."""
    import torch

    import paper_2407_12820_b200 as pq

    P, S, n_init, n_local, k = 2, 12000, 4, 64, 1500
    keys, vals, q0 = orc.gen_workload(S, 128, P, g, oracle_kind(), seed=29 + g)
    s_mid = S - n_init - n_local
    cen, codes = ctx.pq_build(torch.from_numpy(np.ascontiguousarray(keys[:, n_init:n_init + s_mid])).cuda(), 2, 6,
                              4, list(range(P)))
    cap = S + 8
    dk = torch.zeros((P, cap, 128), device="cuda")
    dv = torch.zeros((P, cap, 128), device="cuda")
    dk[:, :S] = torch.from_numpy(keys).cuda()
    dv[:, :S] = torch.from_numpy(vals).cuda()
    dcodes = torch.zeros((P, cap, 2), dtype=torch.int16, device="cuda")
    dcodes[:, :s_mid] = codes
    layer = pq.DecodeLayer(keys=dk, values=dv, centroids=cen, codes=dcodes, total=S, n_init=n_init,
                           n_local=n_local, b=6, tables=ctx.tuple_tables(dcodes, 6, s=s_mid))
    hq = torch.empty((P, g, 128)).pin_memory()
    ho = torch.empty((P, g, 128)).pin_memory()
    rng = np.random.default_rng(g)
    for step in range(5):
        q = torch.from_numpy(q0 + 0.05 * rng.standard_normal(q0.shape).astype(np.float32))
        hq.copy_(q)
        ctx.decode_host(layer, hq, ho, k)
        want = ctx.decode(layer, q.cuda(), k).cpu()
        assert torch.equal(ho, want), f"step {step}"
        if step == 2:  # grow the layer by one token: the graph key changes
            ctx.decode_step(layer, torch.randn((P, 128), device="cuda"), torch.randn((P, 128), device="cuda"),
                            q.cuda(), k)


def test_decode_host_graph_replay_key_path(ctx, orc):
    """The split key path (m4b8, g = 4: cluster select -> gather polling each
    unit's select-done counter) replayed as a graph by pqkv_decode_host: the
    counters reset by each decode must leave every replay equal to the plain
    decode, and the oracle's selection."""
    import torch

    P, S, n_init, n_local, g, k = 3, 9000, 4, 64, 4, 900
    keys, vals, q0 = orc.gen_workload(S, 128, P, g, oracle_kind(), seed=41)
    s_mid = S - n_init - n_local
    cen, codes = ctx.pq_build(torch.from_numpy(np.ascontiguousarray(keys[:, n_init:n_init + s_mid])).cuda(), 4, 8,
                              4, list(range(P)))
    import paper_2407_12820_b200 as pq

    layer = pq.DecodeLayer(keys=torch.from_numpy(keys).cuda(), values=torch.from_numpy(vals).cuda(), centroids=cen,
                           codes=codes, total=S, n_init=n_init, n_local=n_local, b=8)
    assert ctx.decode_plan(layer, g, k)["mode"] == "keys_split"
    hq = torch.empty((P, g, 128)).pin_memory()
    ho = torch.empty((P, g, 128)).pin_memory()
    rng = np.random.default_rng(7)
    cen_h, codes_h = cen.cpu().numpy(), codes.cpu().numpy().view(np.uint16)
    for step in range(4):
        q = q0 + 0.05 * rng.standard_normal(q0.shape).astype(np.float32)
        hq.copy_(torch.from_numpy(q))
        ctx.decode_host(layer, hq, ho, k)
        want = ctx.decode(layer, torch.from_numpy(q).cuda(), k).cpu()
        assert torch.equal(ho, want), f"step {step}"
        p = step % P
        rows = orc.top_k_desc(orc.pq_score_gqa(q[p], cen_h[p], codes_h[p]), k)
        ref = orc.selective_attention(q[p, 0], keys[p], vals[p], n_init, n_local, rows + n_init)
        assert np.abs(ho[p, 0].numpy() - ref).max() / np.abs(ref).max() < 1e-3, f"step {step}"


def oracle_kind():
    import oracle

    return oracle.GAUSSIAN
