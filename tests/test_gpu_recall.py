"""GPU: device-resident recall metrics.

* pqkv_exact_topk / pqkv_overlap_fraction / pqkv_relative_error /
  pqkv_attend_dense against the oracle on the same inputs (exact ids,
  bit-identical error values on identical outputs).
* paper_2407_12820_b200.recall.run_recall on acceptance criterion 9's grid
  (powerlaw keys from the reference's generator, s = 4096, m2b6,
  k = 205/410/819, seeds 1..10, T = 15) prints the same CSV as the
  reference's run_recall + write_recall_csv, byte for byte."""
import os
import subprocess

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _t(a):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def test_metric_ops_match_oracle(ctx, orc):
    import torch

    P, s, g, k = 3, 5000, 4, 700
    keys, vals, qs = orc.gen_workload(s, 128, P, g, oracle.POWERLAW, seed=5)
    ids = ctx.exact_topk(_t(qs), _t(keys), k).cpu().numpy()
    for p in range(P):
        qsum = np.zeros(128, np.float32)
        for r in range(g):
            qsum = (qsum + qs[p, r]).astype(np.float32)
        want = orc.top_k_desc(orc.exact_scores(qsum, keys[p]), k)
        assert np.array_equal(ids[p].astype(np.uint64), want)
    # overlap: a shifted copy of the exact ids
    got = torch.from_numpy(np.concatenate([ids[:, : k // 2], ids[:, : k - k // 2] + 1], 1)).cuda()
    ov = ctx.overlap_fraction(got, _t(ids), s).cpu().numpy()
    for p in range(P):
        want = len(set(got[p].cpu().tolist()) & set(ids[p].tolist())) / k
        assert ov[p] == want
    # full attention (fp64 path) + relative_error
    full = ctx.attend_dense(_t(qs), _t(keys), _t(vals)).cpu().numpy()
    for p in range(P):
        for r in range(g):
            want = orc.softmax_attention(qs[p, r], keys[p], vals[p])
            assert np.abs(full[p, r] - want).max() <= 1e-6 * np.abs(want).max()
    noisy = full + 1e-3 * np.random.default_rng(1).standard_normal(full.shape).astype(np.float32)
    re = ctx.relative_error(_t(noisy), _t(full)).cpu().numpy()
    for p in range(P):
        a, b = noisy[p].astype(np.float64).ravel(), full[p].astype(np.float64).ravel()
        num = den = 0.0
        for i in range(a.size):
            num += (a[i] - b[i]) * (a[i] - b[i])
            den += b[i] * b[i]
        assert re[p] == np.sqrt(num / den)


def test_run_recall_csv_equals_reference(ctx, orc):
    from paper_2407_12820_b200 import recall

    exe = os.path.join(ROOT, "oracle", "_ref", "dropin", "dropin_csv_ref")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/dropin not built")
    ref = subprocess.run([exe, "recall9"], capture_output=True, text=True, timeout=600)
    assert ref.returncode == 0
    wl = {}
    for seed in range(1, 11):
        k, v, q = orc.gen_workload(4096, 128, 1, 1, oracle.POWERLAW, n_components=8, spread=0.5, zipf=1.0, seed=seed)
        wl[seed] = (_t(k), _t(v), _t(q))
    rows = recall.run_recall(ctx, wl, [2], [6], [205, 410, 819], max_iter=15)
    got = recall.recall_csv(rows)
    if got != ref.stdout:
        diff = [(a, b) for a, b in zip(got.splitlines(), ref.stdout.splitlines()) if a != b]
        pytest.fail(f"{len(diff)} CSV lines differ, first: {diff[:3]}")
