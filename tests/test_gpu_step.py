"""GPU parity of the on-device e2e decode step:
pqkv_decode_step = evict_local_append (kv_store.cpp:77-90: encode + append of
the oldest local token, fresh K/V as the newest) + the decode of run_e2e's
per-head loop (experiments.cpp:197-260), checked step by step against the
oracle running the same sequence on the host.  Codes and selected ids
bit-exact, attention within 1e-3 relative (north star)."""
import numpy as np
from _util import rel_err
import pytest

import oracle

pytestmark = pytest.mark.gpu


_rel = rel_err


@pytest.mark.parametrize("g,kind,tables,m,b", [(1, oracle.GAUSSIAN, True, 2, 6), (4, oracle.POWERLAW, True, 2, 6),
                                               (2, oracle.GAUSSIAN, False, 2, 6), (4, oracle.GAUSSIAN, False, 4, 8)])
def test_decode_step_matches_e2e_loop(ctx, orc, g, kind, tables, m, b):
    import torch

    import paper_2407_12820_b200 as pq

    P, n_init, n_local, steps, k = 2, 4, 64, 6, 700
    s_mid0 = 4093  # the middle segment crosses a code-pair chunk (4096 rows) during the steps
    S0 = s_mid0 + n_init + n_local
    keys, vals, qs = orc.gen_workload(S0, 128, P, g, kind, seed=21)
    rng = np.random.default_rng(g)
    cap_tok = S0 + steps
    kh = np.zeros((P, cap_tok, 128), np.float32)
    vh = np.zeros((P, cap_tok, 128), np.float32)
    kh[:, :S0], vh[:, :S0] = keys, vals
    dk, dv = torch.from_numpy(kh).cuda(), torch.from_numpy(vh).cuda()
    cap = s_mid0 + steps
    cen, codes0 = ctx.pq_build(dk[:, n_init:n_init + s_mid0].contiguous(), m, b, 10, [5, 6])
    codes = torch.zeros((P, cap, m), dtype=torch.int16, device="cuda")
    codes[:, :s_mid0] = codes0
    tabs = ctx.tuple_tables(codes, b, s=s_mid0) if tables else None
    layer = pq.DecodeLayer(keys=dk, values=dv, centroids=cen, codes=codes, total=S0, n_init=n_init,
                           n_local=n_local, b=b, tables=tabs)
    cen_h = cen.cpu().numpy()
    codes_h = [list(codes0[p].cpu().numpy().view(np.uint16)) for p in range(P)]
    total = S0
    for step in range(steps):
        nk = rng.standard_normal((P, 128)).astype(np.float32)
        nv = rng.standard_normal((P, 128)).astype(np.float32)
        q = (qs + 0.25 / np.sqrt(128) * rng.standard_normal(qs.shape)).astype(np.float32)
        want_ids = step % 2 == 0
        res = ctx.decode_step(layer, torch.from_numpy(nk).cuda(), torch.from_numpy(nv).cuda(),
                              torch.from_numpy(q).cuda(), k, want_ids=want_ids)
        out, ids = res if want_ids else (res, None)
        torch.cuda.synchronize()
        # host replay of evict_local_append
        for p in range(P):
            ev = total - n_local
            codes_h[p].append(orc.pq_encode_one(kh[p, ev], cen_h[p]))
            kh[p, total], vh[p, total] = nk[p], nv[p]
        total += 1
        assert layer.total == total
        got_codes = codes[:, :total - n_init - n_local].cpu().numpy().view(np.uint16)
        for p in range(P):
            cd = np.asarray(codes_h[p], np.uint16).reshape(-1, m)
            assert np.array_equal(got_codes[p], cd), f"step {step}: appended code differs"
            rows = orc.top_k_desc(orc.pq_score_gqa(q[p], cen_h[p], cd), k)
            if ids is not None:
                assert np.array_equal(ids[p].cpu().numpy().astype(np.uint64), rows), f"step {step}: top-k"
            for r in range(g):
                want = orc.selective_attention(q[p, r], kh[p, :total], vh[p, :total], n_init, n_local,
                                               rows + n_init)
                assert _rel(out[p, r].cpu().numpy(), want) < 1e-3, f"step {step}: attention"
    if tables:  # the incrementally counted tables equal a rebuild over the grown codes
        th, ch = ctx.tuple_tables(codes, b, s=total - n_init - n_local)
        assert torch.equal(th, tabs[0]) and torch.equal(ch, tabs[1])


def test_decode_step_errors(ctx, orc):
    import torch

    import paper_2407_12820_b200 as pq

    keys, vals, qs = orc.gen_workload(600, 128, 1, 1, oracle.GAUSSIAN, seed=2)
    dk, dv = torch.from_numpy(keys).cuda(), torch.from_numpy(vals).cuda()
    cen, codes = ctx.pq_build(dk[:, 4:536].contiguous(), 2, 6, 4, [1])
    layer = pq.DecodeLayer(keys=dk, values=dv, centroids=cen, codes=codes, total=600, n_init=4, n_local=64, b=6)
    nk = torch.zeros((1, 128), device="cuda")
    with pytest.raises(ValueError):  # no room for token 600 in a 600-row cache
        ctx.decode_step(layer, nk, nk, torch.from_numpy(qs).cuda(), 10)
    assert layer.total == 600
