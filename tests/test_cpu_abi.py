"""CPU-only checks: the C-ABI library loads and exports every symbol that
include/moeb.h declares (no compute calls), and the host-side API mirrors the
reference's configuration semantics."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_symbols():
    src = open(os.path.join(ROOT, "include", "moeb.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*|size_t)\s+(moeb_\w+)\s*\(", src,
                                 re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_2508_17137_b200 import build
    path = build.build()
    return ctypes.CDLL(path)


def test_library_exports_header(lib):
    syms = _header_symbols()
    assert len(syms) >= 12
    for s in syms:
        assert hasattr(lib, s), s


def test_python_binding_covers_header():
    from paper_2508_17137_b200 import _native
    assert set(_header_symbols()) == set(_native.EXPORTS)


def test_version_without_gpu(lib):
    lib.moeb_version.restype = ctypes.c_int
    assert lib.moeb_version() == 100


def test_no_cpu_fallback():
    import torch
    import paper_2508_17137_b200 as m
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(m.NativeUnavailable):
        m.load_library()


def test_config_semantics():
    import paper_2508_17137_b200 as m
    shape = m.ModelShape(4, 8, 2)
    assert m.CacheConfig(capacity_fraction=0.1).resolve_capacity(shape) == 3
    assert m.CacheConfig(capacity_fraction=1.0).resolve_capacity(shape) == 32
    assert m.CacheConfig(capacity_fraction=0.001).resolve_capacity(shape) == 1
    v2 = m.ModelShape(26, 64, 6)
    caps = [m.CacheConfig(capacity_fraction=f).resolve_capacity(v2)
            for f in (0.05, 0.1, 0.15, 0.2, 0.25, 0.3, 0.4, 0.5)]
    assert caps == [83, 166, 249, 332, 416, 499, 665, 832]
    for bad in (dict(), dict(capacity_fraction=0.5, capacity_entries=3),
                dict(capacity_fraction=0.0), dict(capacity_fraction=1.5)):
        with pytest.raises(m.ConfigError):
            m.CacheConfig(**bad)
    with pytest.raises(m.ConfigError):
        m.ReplayConfig(shape, m.CacheConfig(capacity_entries=2), warmup_tokens=-1)
    with pytest.raises(m.ConfigError):
        m.ModelShape(1, 4, 5)
    with pytest.raises(m.ConfigError):
        m.make_predictor("nonsense", shape)
    for kind in ("oracle", "global_frequency", "eam_cosine", "external", "learned_linear"):
        with pytest.raises(m.ConfigError):
            m.make_predictor(kind, shape)


def test_seeded_init_matches_reference_rule():
    import paper_2508_17137_b200 as m
    shape = m.ModelShape(26, 64, 6)
    model = m.train(None, shape, m.LearnerConfig(epochs=0, seed=0))
    want = np.random.default_rng(0).normal(0.0, 0.01, (64, 91))
    assert np.array_equal(model.weights, want) and model.trained


def test_shard_bounds_cover_all_prompts():
    import torch
    import paper_2508_17137_b200 as m
    shape = m.ModelShape(3, 8, 2)
    lens = np.array([5, 1, 9, 2, 7, 3, 3, 8])
    off = np.concatenate([[0], np.cumsum(lens * 3)]).astype(np.int64)
    packed = m.PackedTraces(shape, torch.zeros((off[-1], 1), dtype=torch.int64),
                            torch.from_numpy(off), off, np.arange(8))
    for world in (1, 2, 3, 4, 8):
        got = []
        for r in range(world):
            s = packed.shard(r, world)
            got.extend(s.prompt_ids.tolist())
            assert s.row_off_host[0] == 0
        assert got == list(range(8))
