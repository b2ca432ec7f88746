"""Sketch collections (EAMC) for the MoE-Infinity cosine matcher (sketches.py
in the reference, :26-255).

Sketches are row-normalised, layer-major flattened rEAMs. Building them from
traces (counts + normalisation), k-means EAMC construction
(sketches.py:62-139; csrc/kmeans.cu) and every match run on device; the raw
sketches also stay on the host for JSON persistence.
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as nat
from .core import ActivationMatrix, ConfigError, DimensionError, ModelShape


@dataclass(frozen=True)
class EamcConfig:
    mode: str = "recent"
    capacity: int = 100
    binarize: bool = False
    kmeans_max_iters: int = 100
    seed: int = 0

    def __post_init__(self):
        if self.mode not in ("recent", "kmeans"):
            raise ConfigError(f"mode must be 'recent' or 'kmeans', got {self.mode!r}")
        if self.capacity < 1:
            raise ConfigError(f"capacity must be >= 1, got {self.capacity}")
        if self.kmeans_max_iters < 1:
            raise ConfigError(f"kmeans_max_iters must be >= 1, got {self.kmeans_max_iters}")


class SketchCollection:
    """Stored sketches with device-resident matching tables."""

    def __init__(self, sketches, config: EamcConfig, shape: ModelShape):
        if isinstance(sketches, torch.Tensor):
            dev = sketches.to(torch.float64)
            host = dev.cpu().numpy()
        else:
            host = np.asarray(sketches, dtype=np.float64)
            dev = None
        if host.ndim != 2 or host.shape[1] != shape.total_experts:
            raise DimensionError(f"sketches must be 2-D with row length {shape.total_experts}")
        if host.shape[0] > config.capacity:
            raise ConfigError(f"{host.shape[0]} sketches exceed capacity {config.capacity}")
        self.sketches = host
        self.config = config
        self.shape = shape
        self._dev = dev
        self._unit_t = None
        self._topw: dict[int, torch.Tensor] = {}

    def __len__(self) -> int:
        return self.sketches.shape[0]

    def device_tables(self, budget: int, device=None):
        """(unit_t [D][S] fp64, topw [S][L][W]) on device (moeb_eam_prepare)."""
        dev = torch.device("cuda") if device is None else torch.device(device)
        if self._dev is None or self._dev.device != dev:
            self._dev = torch.from_numpy(np.ascontiguousarray(self.sketches)).to(dev)
            self._unit_t = None
            self._topw = {}
        if self._unit_t is None or budget not in self._topw:
            S, L, E = len(self), self.shape.num_layers, self.shape.num_experts
            unit_t = torch.empty((L * E, S), dtype=torch.float64, device=dev)
            topw = torch.empty((S, L, self.shape.mask_words), dtype=torch.int64, device=dev)
            nat.call("moeb_eam_prepare", nat.ptr(self._dev), S, L, E, int(budget),
                     nat.ptr(unit_t), nat.ptr(topw), nat.stream_ptr())
            self._unit_t = unit_t
            self._topw[budget] = topw
        return self._unit_t, self._topw[budget]

    def match_nearest_batch(self, queries) -> tuple[np.ndarray, np.ndarray]:
        """Batched match_nearest for explicit query vectors [M][D] (device fp64 scan)."""
        q = torch.as_tensor(np.ascontiguousarray(queries, dtype=np.float64)).cuda()
        if q.ndim != 2 or q.shape[1] != self.sketches.shape[1]:
            raise DimensionError(f"query length {tuple(q.shape)} != sketch length "
                                 f"{self.sketches.shape[1]}")
        unit_t, _ = self.device_tables(1, q.device)
        M = q.shape[0]
        idx = torch.empty(max(M, 1), dtype=torch.int32, device=q.device)
        sim = torch.empty(max(M, 1), dtype=torch.float64, device=q.device)
        nat.call("moeb_match_queries", nat.ptr(q), M, q.shape[1], nat.ptr(unit_t), len(self),
                 nat.ptr(idx), nat.ptr(sim), nat.stream_ptr())
        return idx[:M].cpu().numpy(), sim[:M].cpu().numpy()

    def match_nearest(self, query) -> tuple[int, float]:
        """Index and cosine of the nearest sketch (sketches.py:165-184)."""
        if len(self) == 0:
            raise ConfigError("no sketches in collection")
        q = np.asarray(query, dtype=np.float64)
        if q.shape != (self.sketches.shape[1],):
            raise DimensionError(f"query length {q.shape} != sketch length "
                                 f"{self.sketches.shape[1]}")
        idx, sim = self.match_nearest_batch(q[None, :])
        return int(idx[0]), float(sim[0])

    def layer_block(self, index: int, layer_id: int) -> np.ndarray:
        e = self.shape.num_experts
        return self.sketches[index, layer_id * e:(layer_id + 1) * e]


def ream_counts(packed, max_tokens: int | None = None) -> torch.Tensor:
    """Per-prompt activation counts [P][L*E] int32 on device (core.py:196-205)."""
    shape = packed.shape
    P = packed.num_prompts
    counts = torch.empty((P, shape.total_experts), dtype=torch.int32, device=packed.device)
    nat.call("moeb_ream_counts", nat.ptr(packed.truth), nat.ptr(packed.row_off), P,
             shape.num_layers, shape.num_experts, -1 if max_tokens is None else int(max_tokens),
             nat.ptr(counts), nat.stream_ptr())
    return counts


def normalize_counts(counts: torch.Tensor, shape: ModelShape, binarize: bool = False):
    """Sketches [n][L*E] fp64 from counts (core.normalize), on device."""
    counts = counts.to(torch.int32).contiguous()
    n = counts.shape[0]
    out = torch.empty((n, shape.total_experts), dtype=torch.float64, device=counts.device)
    nat.call("moeb_sketch_normalize", nat.ptr(counts), n, shape.num_layers, shape.num_experts,
             int(bool(binarize)), nat.ptr(out), nat.stream_ptr())
    return out


@dataclass
class KMeansResult:
    """sketches.KMeansResult (sketches.py:53-59)."""

    centroids: np.ndarray
    assignments: np.ndarray
    objective: float
    objective_history: list[float] = field(default_factory=list)
    effective_k: int = 0


def _sqnorms(X: torch.Tensor) -> torch.Tensor:
    out = torch.empty(X.shape[0], dtype=torch.float64, device=X.device)
    nat.call("moeb_row_sqnorms", nat.ptr(X), X.shape[0], X.shape[1], nat.ptr(out),
             nat.stream_ptr())
    return out


def _assign(X, xn, C):
    """First nearest centroid per vector and its squared distance (K9)."""
    n, D = X.shape
    cn = _sqnorms(C)
    idx = torch.empty(n, dtype=torch.int64, device=X.device)
    d2 = torch.empty(n, dtype=torch.float64, device=X.device)
    nat.call("moeb_sqdist_argmin", nat.ptr(X), nat.ptr(xn), nat.ptr(C), nat.ptr(cn), n,
             C.shape[0], D, nat.ptr(idx), nat.ptr(d2), nat.stream_ptr())
    return idx, d2


def _plusplus_init(X, xn, k: int, rng: np.random.Generator) -> torch.Tensor:
    """sketches._plusplus_init (sketches.py:72-86): distances on device, the
    seeded draws (rng.integers / rng.choice over d2 / total) on the host with
    the reference's own numpy calls so the chosen indices follow its stream."""
    n, D = X.shape
    C = torch.empty((k, D), dtype=torch.float64, device=X.device)
    d2 = torch.empty(n, dtype=torch.float64, device=X.device)
    first = int(rng.integers(0, n))
    C[0] = X[first]
    for j in range(k):
        if j > 0:
            d2h = d2.cpu().numpy()
            total = d2h.sum()
            if total <= 0.0:
                idx = int(rng.integers(0, n))
            else:
                idx = int(rng.choice(n, p=d2h / total))
            C[j] = X[idx]
            if j == k - 1:
                break
        cn = _sqnorms(C[j:j + 1])
        nat.call("moeb_sqdist_update", nat.ptr(X), nat.ptr(xn), nat.ptr(C[j]), nat.ptr(cn), n,
                 D, int(j == 0), nat.ptr(d2), nat.stream_ptr())
    return C


def kmeans(vectors, k: int, seed: int = 0, max_iters: int = 100, device=None) -> KMeansResult:
    """sketches.kmeans (sketches.py:89-139): Lloyd's algorithm with seeded
    k-means++ initialisation, on device. Assignment = fused distance GEMM +
    argmin (K9); centroid update = per-cluster means in member index order
    (bit-identical to numpy for identical assignments); empty clusters are
    re-seeded from the farthest points (stable order). Returns numpy arrays
    like the reference."""
    if isinstance(vectors, torch.Tensor):
        X = vectors.to(torch.float64)
    else:
        arr = np.asarray(vectors, dtype=np.float64)
        if arr.ndim != 2 or arr.shape[0] < 1:
            raise DimensionError("kmeans needs a non-empty 2-D array of vectors")
        nat.load_library()
        X = torch.from_numpy(np.ascontiguousarray(arr)).to(
            device if device is not None else torch.device("cuda", torch.cuda.current_device()))
    if X.dim() != 2 or X.shape[0] < 1:
        raise DimensionError("kmeans needs a non-empty 2-D array of vectors")
    X = X.contiguous()
    n, D = X.shape
    k = min(k, n)
    if k < 1:
        raise ConfigError(f"k must be >= 1, got {k}")
    rng = np.random.default_rng(seed)
    xn = _sqnorms(X)
    C = _plusplus_init(X, xn, k, rng)
    assignments = None
    history: list[float] = []
    for _ in range(max_iters):
        idx, pd2 = _assign(X, xn, C)
        counts = torch.bincount(idx, minlength=k)
        empty = torch.nonzero(counts == 0).flatten().tolist()
        if empty:
            order = np.argsort(-pd2.cpu().numpy(), kind="stable")
            for taken, j in enumerate(empty):
                C[j] = X[int(order[taken])]
            idx, pd2 = _assign(X, xn, C)
        history.append(float(pd2.cpu().numpy().sum()))
        if assignments is not None and torch.equal(idx, assignments):
            break
        assignments = idx
        counts = torch.bincount(idx, minlength=k)
        members = torch.argsort(idx, stable=True)
        offs = torch.zeros(k + 1, dtype=torch.int64, device=X.device)
        offs[1:] = torch.cumsum(counts, 0)
        nat.call("moeb_cluster_means", nat.ptr(X), nat.ptr(members), nat.ptr(offs), k, D,
                 nat.ptr(C), nat.stream_ptr())
    idx, pd2 = _assign(X, xn, C)
    objective = float(pd2.cpu().numpy().sum())
    return KMeansResult(C.cpu().numpy(), idx.cpu().numpy(), objective, history, k)


def build_eamc(matrices, config: EamcConfig, shape: ModelShape | None = None) -> SketchCollection:
    """Collection from rEAMs (sketches.py:200-216): ActivationMatrix list or
    PackedTraces (one rEAM per prompt). Recent mode keeps the last `capacity`."""
    from .traces import PackedTraces

    if isinstance(matrices, PackedTraces):
        shape = matrices.shape
        counts = ream_counts(matrices)
    else:
        if not matrices:
            raise ConfigError("at least one activation matrix is required")
        shape = matrices[0].shape
        counts = torch.as_tensor(np.stack([m.counts for m in matrices]).reshape(len(matrices), -1)
                                 .astype(np.int32)).cuda()
    if config.mode == "recent":
        counts = counts[-config.capacity:]
        return SketchCollection(normalize_counts(counts, shape, config.binarize), config, shape)
    vectors = normalize_counts(counts, shape, config.binarize)
    result = kmeans(vectors, config.capacity, seed=config.seed, max_iters=config.kmeans_max_iters)
    return SketchCollection(result.centroids, config, shape)


def save_eamc(collection: SketchCollection, path) -> None:
    payload = {
        "mode": collection.config.mode,
        "capacity": collection.config.capacity,
        "binarize": collection.config.binarize,
        "kmeans_max_iters": collection.config.kmeans_max_iters,
        "seed": collection.config.seed,
        "num_layers": collection.shape.num_layers,
        "num_experts": collection.shape.num_experts,
        "top_k": collection.shape.top_k,
        "sketches": [[float(v) for v in row] for row in collection.sketches],
    }
    with open(path, "w", encoding="utf-8") as fh:
        json.dump(payload, fh)
        fh.write("\n")


def load_eamc(path) -> SketchCollection:
    """Same file format and checks as the reference (sketches.py:237-255)."""
    with open(path, encoding="utf-8") as fh:
        payload = json.load(fh)
    try:
        config = EamcConfig(mode=payload["mode"], capacity=payload["capacity"],
                            binarize=payload["binarize"],
                            kmeans_max_iters=payload["kmeans_max_iters"], seed=payload["seed"])
        shape = ModelShape(payload["num_layers"], payload["num_experts"], payload["top_k"])
        sketches = np.asarray(payload["sketches"], dtype=np.float64)
    except (KeyError, TypeError) as exc:
        raise ConfigError(f"bad sketch collection file {path}: {exc}") from None
    if sketches.size == 0:
        raise ConfigError(f"no sketches in {path}")
    return SketchCollection(sketches, config, shape)


class TensorCoreMatcher:
    """SketchCollection.match_nearest for many count-vector queries at once on
    tensor cores (BASELINE C4; K6b): one tcgen05 GEMM over the
    fp16-split unit sketches with a fused per-tile max/argmax epilogue, then
    an fp64 re-rank of near-tie tiles. Exact first-argmax semantics."""

    EPS_REL = 3e-5  # bound on split + fp32-accumulation error, relative to the max score

    def __init__(self, collection: SketchCollection, device=None):
        dev = torch.device("cuda") if device is None else torch.device(device)
        S, D = collection.sketches.shape
        if D % 32:
            raise DimensionError("sketch length must be a multiple of 32")
        self.S, self.D, self.S_pad = S, D, (S + 255) // 256 * 256
        self.sketches = torch.from_numpy(np.ascontiguousarray(collection.sketches)).to(dev)
        self.uu = torch.empty((self.S_pad, 2 * D), dtype=torch.float16, device=dev)
        self.norms = torch.empty(S, dtype=torch.float64, device=dev)
        nat.call("moeb_eam_pack_library", nat.ptr(self.sketches), S, D, self.S_pad,
                 nat.ptr(self.uu), nat.ptr(self.norms), nat.stream_ptr())
        self.device = dev

    def match_counts(self, counts: torch.Tensor, timing: dict | None = None):
        """counts [M][D] int32 (partial rEAM counts with equal per-layer row sums,
        e.g. layer-0 queries) -> (idx int32 [M], cosine fp64 [M], tiles re-ranked)."""
        from .transformer import gemm
        counts = counts.to(torch.int32).contiguous()
        M = counts.shape[0]
        dev = self.device
        cc = torch.empty((max(M, 1), 2 * self.D), dtype=torch.float16, device=dev)
        nat.call("moeb_eam_pack_queries", nat.ptr(counts), M, self.D, nat.ptr(cc),
                 nat.stream_ptr())
        nt = self.S_pad // 256
        pval = torch.empty((max(M, 1), nt), dtype=torch.float32, device=dev)
        pidx = torch.empty((max(M, 1), nt), dtype=torch.int32, device=dev)
        e0 = e1 = None
        if timing is not None:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
        gemm(cc, self.uu, M, self.S_pad, 2 * self.D, 5, out32=pval, out16=pidx, fp16=True)
        if timing is not None:
            e1.record()
            timing.setdefault("gemm_rowmax", []).append((e0, e1, 2.0 * M * self.S * self.D))
        idx = torch.empty(max(M, 1), dtype=torch.int32, device=dev)
        sim = torch.empty(max(M, 1), dtype=torch.float64, device=dev)
        nrr = torch.empty(max(M, 1), dtype=torch.int32, device=dev)
        nat.call("moeb_eam_rerank", nat.ptr(pval), nat.ptr(pidx), nt, nat.ptr(counts),
                 nat.ptr(self.sketches), nat.ptr(self.norms), M, self.S, self.D,
                 float(self.EPS_REL), nat.ptr(idx), nat.ptr(sim), nat.ptr(nrr), nat.stream_ptr())
        return idx[:M], sim[:M], nrr[:M]


def token_query_counts(packed, warmup: int) -> torch.Tensor:
    """Layer-0 partial rEAM counts for every prompt token >= warmup (C4 queries)."""
    L, E = packed.shape.num_layers, packed.shape.num_experts
    per = np.maximum(packed.num_tokens - warmup, 0)
    qoff = np.concatenate([[0], np.cumsum(per)]).astype(np.int64)
    out = torch.empty((max(int(qoff[-1]), 1), L * E), dtype=torch.int32, device=packed.device)
    qd = torch.from_numpy(qoff).to(packed.device)
    nat.call("moeb_token_prefix_counts", nat.ptr(packed.truth), nat.ptr(packed.row_off),
             nat.ptr(qd), packed.num_prompts, L, E, int(warmup), nat.ptr(out), nat.stream_ptr())
    return out[:int(qoff[-1])]
