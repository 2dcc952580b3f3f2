"""GPU: device-side synthetic workloads (pqkv_gen_workload) follow the
reference generator's distributions (workload.cpp:39-79): gaussian-mixture
keys around n_components shared means with the given spread, N(0,1) values
and queries; powerlaw keys whose scaled exact scores against the head's unit
query direction are 8/(rank+1)^zipf over a permutation of ranks."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_gaussian_mixture(ctx):
    k, v, q = ctx.gen_workload(20000, 128, h_kv=2, g=3, kind="gaussian", n_components=8, spread=0.5, seed=5)
    k, v, q = k.cpu().numpy(), v.cpu().numpy(), q.cpu().numpy()
    assert k.shape == (2, 20000, 128) and q.shape == (2, 3, 128)
    for h in range(2):
        # 8 clusters: same-component keys are ~spread*sqrt(2d) = 8 apart,
        # different components ~sqrt(2d(1 + spread^2)) = 17.9
        rows = k[h]
        centres = []
        for x in rows[:2000]:
            if all(np.linalg.norm(x - c) > 12.0 for c in centres):
                centres.append(x)
        assert len(centres) == 8
        lab = np.stack([((rows - c) ** 2).sum(1) for c in centres]).argmin(0)
        means = np.stack([rows[lab == j].mean(0) for j in range(8)])
        resid = rows - means[lab]
        assert abs(resid.std() - 0.5) < 0.01  # spread
        assert abs(means.std() - 1.0) < 0.15  # means ~ N(0, 1)
    assert abs(v.mean()) < 0.01 and abs(v.std() - 1) < 0.01
    assert abs(q.std() - 1) < 0.2
    k2, _, _ = ctx.gen_workload(20000, 128, h_kv=2, g=3, kind="gaussian", seed=5)
    assert np.array_equal(k, k2.cpu().numpy())  # a pure function of the seed


def test_powerlaw_scores(ctx):
    s, d, zipf = 5000, 128, 1.0
    k, v, q = ctx.gen_workload(s, d, h_kv=2, g=2, kind="powerlaw", zipf=zipf, seed=9)
    k, q = k.cpu().numpy().astype(np.float64), q.cpu().numpy().astype(np.float64)
    for h in range(2):
        assert np.allclose(q[h, 0], q[h, 1]) and abs(np.linalg.norm(q[h, 0]) - 1) < 1e-6
        scores = k[h] @ q[h, 0] / np.sqrt(d)
        want = 8.0 / np.arange(1, s + 1) ** zipf
        assert np.allclose(np.sort(scores)[::-1], want, rtol=1e-4, atol=1e-5)  # ranks are a permutation
        # the orthogonal part is a unit vector's remainder: |key - (key.q)q| <= 1
        orth = k[h] - np.outer(k[h] @ q[h, 0], q[h, 0])
        assert np.all(np.linalg.norm(orth, axis=1) <= 1 + 1e-5)


def test_bad_arguments(ctx):
    with pytest.raises(ValueError):
        ctx.gen_workload(100, 128, kind="gaussian", n_components=0)
    with pytest.raises(ValueError):
        ctx.gen_workload(100, 128, kind="powerlaw", zipf=0.0)
