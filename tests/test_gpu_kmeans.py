"""k-means EAMC construction on device vs the reference's own results
(tests/golden/kmeans_cases.npz from make_kmeans_golden.py): identical
assignments, centroids within 1e-12 (the distance GEMM's summation order is
the only difference; centroid means are bit-identical for identical
assignments), the same objective history; plus the reference's property
tests (monotone objective, Lloyd fixed point, determinism)."""
import os

import numpy as np
import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def z():
    with np.load(os.path.join(ROOT, "tests", "golden", "kmeans_cases.npz")) as f:
        return {k: f[k] for k in f.files}


@pytest.fixture(scope="module")
def m():
    import paper_2508_17137_b200 as m
    m.load_library()
    return m


def _check(res, cent, assign, hist):
    assert np.array_equal(res.assignments, assign)
    assert res.centroids.shape == cent.shape
    assert np.allclose(res.centroids, cent, rtol=0, atol=1e-12)
    assert len(res.objective_history) == len(hist)
    assert np.allclose(res.objective_history, hist, rtol=1e-12, atol=1e-12)


def test_reference_cases(m, z):
    exact_cent = 0
    for i in range(int(z["n_cases"][0])):
        k, seed, it, keff = (int(v) for v in z[f"c{i}_meta"])
        res = m.kmeans(z[f"c{i}_x"], k, seed=seed, max_iters=it)
        assert res.effective_k == keff
        _check(res, z[f"c{i}_cent"], z[f"c{i}_assign"], z[f"c{i}_hist"])
        assert res.objective == pytest.approx(float(z[f"c{i}_obj"][0]), rel=1e-12, abs=1e-12)
        exact_cent += int(np.array_equal(res.centroids, z[f"c{i}_cent"]))
    # centroid means follow numpy's accumulation order: most cases bit-equal
    assert exact_cent >= int(z["n_cases"][0]) // 2


def test_large_case(m, z):
    k, seed, it, n, d, s = (int(v) for v in z["big_meta"])
    x = np.random.default_rng(s).random((n, d)) ** 4
    res = m.kmeans(x, k, seed=seed, max_iters=it)
    _check(res, z["big_cent"], z["big_assign"], z["big_hist"])


def test_properties(m):
    rng = np.random.default_rng(5)
    for trial in range(30):
        n = int(rng.integers(3, 40))
        d = int(rng.integers(2, 9))
        k = int(rng.integers(1, n + 1))
        v = rng.random((n, d))
        res = m.kmeans(v, k, seed=trial)
        h = res.objective_history
        assert all(b <= a + 1e-9 for a, b in zip(h, h[1:]))
        d2 = ((v[:, None, :] - res.centroids[None, :, :]) ** 2).sum(axis=2)
        own = d2[np.arange(n), res.assignments]
        assert (own <= d2.min(axis=1) + 1e-9).all()
        again = m.kmeans(v, k, seed=trial)
        assert np.array_equal(again.centroids, res.centroids)


def test_eamc_kmeans(m, z):
    shape = m.ModelShape(26, 64, 6)
    packed = m.generate_packed(m.GeneratorConfig(120, 24, shape, 8, 0.9, 3))
    for j in range(2):
        cap, binz, seed = (int(v) for v in z[f"eamc{j}_meta"])
        coll = m.build_eamc(packed, m.EamcConfig(mode="kmeans", capacity=cap,
                                                 binarize=bool(binz), seed=seed))
        assert np.allclose(coll.sketches, z[f"eamc{j}_sketches"], rtol=0, atol=1e-12)


def test_sqnorms_bit_exact(m):
    from paper_2508_17137_b200 import sketches as sk
    rng = np.random.default_rng(2)
    for d in (1, 5, 8, 100, 129, 1664, 9000, 14848):
        x = rng.random((7, d)) * rng.random((7, d))
        got = sk._sqnorms(torch.from_numpy(x).cuda()).cpu().numpy()
        assert np.array_equal(got, (x * x).sum(axis=1)), d


def test_activation_report(m):
    """K8 counts -> activation_report == a numpy restatement of
    metrics.activation_report (metrics.py:95-119) on the same traces."""
    from conftest import load_case
    c = load_case("v2lite_small")
    shape = m.ModelShape(26, 64, 6)
    truth = c["truth"].astype(np.uint64)
    off = c["row_off"]
    packed = m.PackedTraces(shape, torch.from_numpy(truth.view(np.int64)).cuda(),
                            torch.from_numpy(off).cuda(), off, np.arange(len(off) - 1))
    rep = m.activation_report(packed, shape)
    L, E = 26, 64
    counts = np.zeros((L, E), dtype=np.int64)
    distinct = []
    for p in range(len(off) - 1):
        seen = np.zeros((L, E), dtype=bool)
        for r in range(off[p], off[p + 1]):
            l = (r - off[p]) % L
            for e in range(E):
                if (int(truth[r, 0]) >> e) & 1:
                    counts[l, e] += 1
                    seen[l, e] = True
        distinct.append(seen.sum(axis=1))
    assert np.array_equal(rep.layer_expert_counts, counts)
    assert np.array_equal(rep.prompt_layer_distinct, np.stack(distinct))
    assert rep.prompt_ids == list(range(len(off) - 1))
