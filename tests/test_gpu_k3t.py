"""K3t (tensor-core column sums, fp32 scores with a rigorous error bound,
exact fp64 re-evaluation of undecidable rows) gives exactly the masks and
fused replay counters of the fp64 K3 kernel -- and through it the
reference's (test_gpu_parity / test_gpu_acceptance compare those with the
reference's own outputs).

Cases: the bench shape and others (L up to 32, budgets 1..16, threshold
mode, decays 0 .. 0.99), ragged prompts, weights with exact ties (dyadic
values: most rows undecidable in fp32, all of them re-evaluated), and a
workspace too small for the re-evaluation list (the whole call is redone by
the gated fp64 kernel)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def m():
    import paper_2508_17137_b200 as m
    m.load_library()
    return m


def _packed(m, L, k, prompts, tokens, seed, ragged=False):
    shape = m.ModelShape(L, 64, k)
    packed = m.generate_packed(m.GeneratorConfig(prompts, tokens, shape, 8, 0.9, seed))
    if not ragged:
        return shape, packed
    truth = packed.truth.reshape(-1)
    rows, off = [], [0]
    for p in range(prompts):
        T = 1 + (p * 13) % tokens
        r0 = int(packed.row_off_host[p])
        rows.append(truth[r0:r0 + T * L])
        off.append(off[-1] + T * L)
    off = np.array(off, dtype=np.int64)
    return shape, m.PackedTraces(shape, torch.cat(rows).reshape(-1, 1).contiguous(),
                                 torch.from_numpy(off).cuda(), off,
                                 np.arange(prompts, dtype=np.int64))


def _both(m, monkeypatch, shape, packed, w, decay, budget, threshold, warmup=8):
    model = m.LinearModel(shape, m.LearnerConfig(epochs=0, decay=decay), w, trained=True)
    pred = m.make_predictor("learned_linear", shape, model=model, threshold=threshold)
    L = shape.num_layers
    out = []
    for mode in ("tc", "fp64"):
        if mode == "fp64":
            monkeypatch.setenv("MOEB_K3", "fp64")
        else:
            monkeypatch.delenv("MOEB_K3", raising=False)
        cnt = torch.zeros(2 + 2 * L, dtype=torch.int64, device="cuda")
        masks = pred.predict_masks(packed, budget, warmup, counts=cnt)
        amb = pred.ambiguous_rows() if mode == "tc" else None
        out.append((masks.clone(), cnt.clone(), amb))
    monkeypatch.delenv("MOEB_K3", raising=False)
    return out


@pytest.mark.parametrize("L,k,budget,threshold,decay", [
    (26, 6, 6, False, 0.9), (26, 6, 8, False, 0.9), (3, 2, 2, False, 0.9),
    (32, 8, 8, False, 0.5), (26, 6, 1, False, 0.9), (26, 6, 16, False, 0.9),
    (26, 6, 6, True, 0.9), (5, 4, 3, False, 0.0), (26, 6, 6, False, 0.99),
    (17, 6, 5, False, 0.75)])
@pytest.mark.parametrize("ragged", [False, True])
def test_k3t_equals_fp64_kernel(m, monkeypatch, L, k, budget, threshold, decay, ragged):
    shape, packed = _packed(m, L, k, 70, 150, 11 + L, ragged)
    w = np.random.default_rng(L * 7 + budget).normal(0.0, 0.01, (64, L + 65))
    if threshold:
        w[:, -1] -= 0.02  # a mix of positive and negative scores
    (tm, tc_cnt, amb), (fm, f_cnt, _) = _both(m, monkeypatch, shape, packed, w, decay, budget,
                                             threshold)
    assert torch.equal(tm, fm)
    assert torch.equal(tc_cnt, f_cnt)
    assert amb is not None and amb < max(50, packed.rows // 100)


def test_k3t_exact_ties(m, monkeypatch):
    """Dyadic weights: many exactly tied scores -- the fp32 path must hand
    every undecidable row to the fp64 re-evaluation (ties to the lower id)."""
    shape, packed = _packed(m, 26, 6, 40, 120, 5)
    rng = np.random.default_rng(3)
    w = rng.integers(-4, 5, (64, 91)).astype(np.float64) / 64.0
    (tm, tc_cnt, amb), (fm, f_cnt, _) = _both(m, monkeypatch, shape, packed, w, 0.5, 6, False)
    assert amb > 0
    assert torch.equal(tm, fm) and torch.equal(tc_cnt, f_cnt)


def test_k3t_list_overflow(m, monkeypatch):
    """A workspace whose re-evaluation list is too small: the gated fp64
    kernel redoes the call; masks and counters unchanged."""
    from paper_2508_17137_b200 import _native as nat
    shape, packed = _packed(m, 26, 6, 40, 120, 5)
    w = np.random.default_rng(3).integers(-4, 5, (64, 91)).astype(np.float64) / 64.0
    (fm_tc, f_cnt_tc, amb), _ = _both(m, monkeypatch, shape, packed, w, 0.5, 6, False)
    lib = nat.load_library()
    full = lib.moeb_linear_workspace_bytes(packed.rows, 26, 64)
    cap_bytes = 8 * 65536
    small = full - cap_bytes + 8 * 4  # room for 4 list entries
    assert amb > 4
    ws = torch.empty(small, dtype=torch.uint8, device="cuda")
    out = torch.empty_like(packed.truth)
    cnt = torch.zeros(54, dtype=torch.int64, device="cuda")
    wt = torch.from_numpy(w).cuda()
    nat.call("moeb_linear_predict_counts", nat.ptr(packed.truth), nat.ptr(packed.row_off),
             packed.num_prompts, 26, 64, nat.ptr(wt), 0.5, 6, 0, 8, 6, nat.ptr(out), None, None,
             nat.ptr(cnt), packed.rows, nat.ptr(ws), small, nat.stream_ptr())
    assert torch.equal(out, fm_tc) and torch.equal(cnt, f_cnt_tc)


def test_k3t_c2_scale_ambiguity(m, monkeypatch):
    """Bench weights on 1,000 C2 prompts x 363 tokens: identical to the fp64
    kernel, and the fp32 bound leaves only a small fraction of rows to fp64."""
    shape, packed = _packed(m, 26, 6, 1000, 363, 7)
    w = np.random.default_rng(0).normal(0.0, 0.01, (64, 91))
    (tm, tc_cnt, amb), (fm, f_cnt, _) = _both(m, monkeypatch, shape, packed, w, 0.9, 6, False)
    print(f"ambiguous rows: {amb} of {packed.rows} ({amb / packed.rows:.2e})")
    assert torch.equal(tm, fm) and torch.equal(tc_cnt, f_cnt)
    assert amb < packed.rows * 2e-3
