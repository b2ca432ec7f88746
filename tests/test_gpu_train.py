"""learned_linear training on device vs the reference's own train()
(tests/golden/train_cases.npz from make_train_golden.py): identical
features (bit-exact), same number of epochs (early stop), loss history and
final weights within 1e-10 (the per-example dot product sums in a different
order than numpy's BLAS; every other operation follows numpy's order)."""
import os

import numpy as np
import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu
NAMES = ["rule10", "rule5", "v2lite", "e100", "stop"]


@pytest.fixture(scope="module")
def z():
    with np.load(os.path.join(ROOT, "tests", "golden", "train_cases.npz")) as f:
        return {k: f[k] for k in f.files}


def _packed(m, z, name):
    L, E, k = (int(x) for x in z[f"{name}_shape"])
    shape = m.ModelShape(L, E, k)
    truth = z[f"{name}_truth"]
    off = z[f"{name}_off"]
    return shape, m.PackedTraces(shape, torch.from_numpy(truth.view(np.int64)).cuda(),
                                 torch.from_numpy(off).cuda(), off,
                                 np.arange(len(off) - 1, dtype=np.int64))


@pytest.mark.parametrize("name", NAMES)
def test_train_matches_reference(z, name):
    import paper_2508_17137_b200 as m
    m.load_library()
    shape, packed = _packed(m, z, name)
    lr, ep, decay, seed = z[f"{name}_cfg"]
    cfg = m.LearnerConfig(learning_rate=float(lr), epochs=int(ep), decay=float(decay),
                          seed=int(seed))
    model = m.train(packed, shape, cfg)
    want_loss = z[f"{name}_loss"]
    assert len(model.loss_history) == len(want_loss)
    np.testing.assert_allclose(model.loss_history, want_loss, rtol=1e-10, atol=0)
    np.testing.assert_allclose(model.weights, z[f"{name}_weights"], rtol=0, atol=1e-10)
    again = m.train(packed, shape, cfg)
    assert np.array_equal(again.weights, model.weights)  # deterministic


def test_features_bit_exact(z):
    import paper_2508_17137_b200 as m
    from paper_2508_17137_b200 import _native as nat
    m.load_library()
    shape, packed = _packed(m, z, "v2lite")
    hist = torch.empty((packed.rows, shape.num_experts), dtype=torch.float64, device="cuda")
    nat.call("moeb_linear_features", nat.ptr(packed.truth), nat.ptr(packed.row_off),
             packed.num_prompts, shape.num_layers, shape.num_experts, 0.9, nat.ptr(hist),
             nat.stream_ptr())
    assert np.array_equal(hist.cpu().numpy(), z["v2lite_hist"])
