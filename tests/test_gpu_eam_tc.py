"""EAM matching at scale on tensor cores (BASELINE C4 shape, reduced library):
the tcgen05 row-argmax GEMM + fp64 re-rank must return exactly numpy's fp64
first argmax of unit . (q / |q|) (SketchCollection.match_nearest,
sketches.py:165-184) for every per-token layer-0 query."""
import numpy as np
import pytest
import torch

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(600)]


def test_tc_matcher_exact_argmax():
    import paper_2508_17137_b200 as m
    from paper_2508_17137_b200 import sketches as SK
    shape = m.ModelShape(26, 64, 6)
    lib_traces = m.generate_packed(m.GeneratorConfig(3000, 32, shape, 8, 0.9, 11,
                                                     first_prompt_id=10**6))
    coll = SK.build_eamc(lib_traces, SK.EamcConfig(mode="recent", capacity=3000))
    queries = m.generate_packed(m.GeneratorConfig(16, 40, shape, 8, 0.9, 7))
    counts = SK.token_query_counts(queries, warmup=8)
    assert counts.shape == (16 * 32, 26 * 64)
    # query counts restated on the host from the packed truth
    truth = queries.truth.cpu().numpy().view(np.uint64).reshape(16, 40, 26)
    bits = ((truth[..., None] >> np.arange(64, dtype=np.uint64)) & np.uint64(1)).astype(np.int64)
    cum = np.cumsum(bits, axis=1) - bits  # tokens < t
    want_counts = cum[:, 8:].reshape(16 * 32, 26 * 64)
    assert np.array_equal(counts.cpu().numpy(), want_counts)
    tc = SK.TensorCoreMatcher(coll)
    idx, sim, nrr = tc.match_counts(counts)
    sk = coll.sketches
    unit = sk / np.where(np.linalg.norm(sk, axis=1) > 0, np.linalg.norm(sk, axis=1), 1.0)[:, None]
    q = want_counts.astype(np.float64)
    qn = np.linalg.norm(q, axis=1)
    sims = unit @ (q / qn[:, None]).T
    want = np.argmax(sims, axis=0)
    got = idx.cpu().numpy()
    assert np.array_equal(got, want), np.nonzero(got != want)[0][:10]
    np.testing.assert_allclose(sim.cpu().numpy(), sims[want, np.arange(len(want))], atol=1e-12)
    print(f"re-ranked tiles per query: mean {nrr.float().mean().item():.2f} max {nrr.max().item()}")
    # zero query -> index 0
    z = torch.zeros((2, 26 * 64), dtype=torch.int32, device="cuda")
    zi, zs, _ = tc.match_counts(z)
    assert zi.tolist() == [0, 0] and zs.tolist() == [0.0, 0.0]
