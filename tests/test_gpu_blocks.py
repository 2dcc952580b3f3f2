"""GPU: per-request block-cache accounting (pqkv_block_rank) -- distinct
tokens, distinct tokens per block and the top-k_cache ranking (count desc,
block id asc: kv_store.cpp:158-166) -- against a numpy restatement of
fetch_topk's by_block map.  The full LRU/LFU state machine is checked against
the reference library in tests/cpp/test_api.cpp (kv_cache suite)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _want(ids, n_tokens, bs, k_cache):
    d = np.unique(ids[(ids >= 0) & (ids < n_tokens)])
    nb = max(1, -(-n_tokens // bs))
    counts = np.bincount(d // bs, minlength=nb)[:nb]
    touched = np.flatnonzero(counts)
    order = sorted(touched, key=lambda b: (-counts[b], b))[:k_cache]
    ranked = np.full(k_cache, -1, np.int64)
    ranked[:len(order)] = order
    return d, counts, ranked, len(touched)


@pytest.mark.parametrize("n_tokens,bs,n,k_cache", [(131072, 128, 26214, 32), (5000, 7, 900, 5), (300, 1000, 50, 3),
                                                   (70000, 64, 1, 4), (4096, 16, 0, 2),
                                                   # bitmap + sort keys beyond shared memory: the global-memory
                                                   # path (block size 1 over 100K tokens; 16 over 600K)
                                                   (100000, 1, 30000, 40), (600000, 16, 50000, 64)])
def test_block_rank_matches_by_block_map(ctx, n_tokens, bs, n, k_cache):
    import torch

    rng = np.random.default_rng(n_tokens + bs)
    P = 3
    ids = np.stack([rng.integers(0, n_tokens, n) for _ in range(P)]).astype(np.int64)
    if n > 10:
        ids[:, :5] = ids[:, 5:10]  # repeated ids count once
    bm, counts, ranked, touched = ctx.block_rank(torch.from_numpy(ids).cuda(), n_tokens, bs, k_cache)
    bm = bm.cpu().numpy().view(np.uint32)
    for p in range(P):
        d, wc, wr, wt = _want(ids[p], n_tokens, bs, k_cache)
        bits = np.flatnonzero(np.unpackbits(bm[p].view(np.uint8), bitorder="little"))
        assert np.array_equal(bits, d)
        assert np.array_equal(counts[p].cpu().numpy(), wc)
        assert np.array_equal(ranked[p].cpu().numpy(), wr)
        assert int(touched[p]) == wt
