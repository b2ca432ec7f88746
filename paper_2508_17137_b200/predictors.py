"""Expert-set predictors as device mask producers (predictors.py in the reference).

The reference protocol is per step: ``predict(ctx) -> frozenset`` called from
the replay loop. Here every predictor turns a whole ``PackedTraces`` batch
into one bitmask row per trace row in a single device pass
(``predict_masks``); predictions never depend on the cache
(engine.py:244-246), so this is exactly the sequence of sets the reference
loop would produce. The optional flags the reference engine reads with
getattr (engine.py:128-141) keep their meaning: ``unbounded_prefetch``,
``history_decay``, and coverage for the external predictor.

Kinds: oracle, lru_only, next_layer_all, global_frequency, eam_cosine,
external, learned_linear (predictors.py:29-37), plus ``transformer`` (the
paper's predictor, transformer.py).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _native as nat
from .core import ActivationMatrix, ConfigError, ModelShape
from .learner import LinearModel
from .sketches import SketchCollection, ream_counts
from .traces import PackedTraces, pack_traces

PREDICTOR_KINDS = ("oracle", "lru_only", "next_layer_all", "global_frequency", "eam_cosine",
                   "external", "learned_linear", "transformer")


@dataclass
class PredictionContext:
    """One (token, layer) query of the reference's per-step protocol
    (predictors.py:40-54). The device predictors here work on whole traces
    (predict_masks); the type is kept for API compatibility."""

    prompt_id: int
    token_index: int
    target_layer: int
    partial_ream: ActivationMatrix
    history: np.ndarray
    budget: int


def _empty(packed: PackedTraces) -> torch.Tensor:
    return torch.empty((packed.rows, packed.shape.mask_words), dtype=torch.int64,
                       device=packed.device)


def _policy(kind_code: int, packed: PackedTraces, budget: int, truth=None, table=None):
    out = _empty(packed)
    nat.call("moeb_policy_masks", kind_code, nat.ptr(truth), packed.rows,
             packed.shape.num_layers, packed.shape.num_experts, int(budget), nat.ptr(table),
             nat.ptr(out), nat.stream_ptr())
    return out


class DevicePredictor:
    kind = "base"
    unbounded_prefetch = False
    #: True when the predictor's masks are all-empty (lru_only): the cache sim
    #: then runs without reading a prediction stream at all.
    empty = False

    def predict_masks(self, packed: PackedTraces, budget: int, warmup: int = 0,
                      metrics: torch.Tensor | None = None) -> torch.Tensor:
        raise NotImplementedError

    def coverage(self, packed: PackedTraces):
        return None


class OraclePredictor(DevicePredictor):
    """Ground truth truncated to the budget lowest ids (predictors.py:57-82)."""

    kind = "oracle"

    def __init__(self, traces, shape: ModelShape):
        self.shape = shape
        self._packed = pack_traces(traces, shape)

    def _truth_for(self, packed: PackedTraces) -> torch.Tensor:
        mine = self._packed
        if (np.array_equal(mine.prompt_ids, packed.prompt_ids)
                and np.array_equal(mine.row_off_host, packed.row_off_host)):
            return mine.truth.to(packed.device)
        pos = {int(p): i for i, p in enumerate(mine.prompt_ids)}
        idx = []
        for i, pid in enumerate(packed.prompt_ids):
            if int(pid) not in pos:
                raise ConfigError(f"oracle has no trace for prompt {int(pid)}")
            j = pos[int(pid)]
            n = int(packed.row_off_host[i + 1] - packed.row_off_host[i])
            if n > mine.row_off_host[j + 1] - mine.row_off_host[j]:
                raise ConfigError(f"oracle trace for prompt {int(pid)} is shorter than replayed")
            idx.append(np.arange(n) + mine.row_off_host[j])
        gather = torch.from_numpy(np.concatenate(idx)).to(mine.truth.device)
        return mine.truth.index_select(0, gather).to(packed.device).contiguous()

    def predict_masks(self, packed, budget, warmup=0, metrics=None):
        return _policy(1, packed, budget, truth=self._truth_for(packed))


class LruOnlyPredictor(DevicePredictor):
    kind = "lru_only"
    empty = True

    def __init__(self, shape: ModelShape):
        self.shape = shape

    def predict_masks(self, packed, budget, warmup=0, metrics=None):
        return _policy(0, packed, budget)


class NextLayerAllPredictor(DevicePredictor):
    kind = "next_layer_all"
    unbounded_prefetch = True

    def __init__(self, shape: ModelShape):
        self.shape = shape

    def predict_masks(self, packed, budget, warmup=0, metrics=None):
        return _policy(2, packed, budget)


class GlobalFrequencyPredictor(DevicePredictor):
    """Top experts per layer by training-workload counts, ties to the lower id
    (predictors.py:111-139). Counting runs on device over the packed workload."""

    kind = "global_frequency"

    def __init__(self, train_traces, shape: ModelShape):
        if train_traces is None or (not isinstance(train_traces, PackedTraces)
                                    and not train_traces):
            raise ConfigError("global_frequency needs a training workload")
        self.shape = shape
        packed = pack_traces(train_traces, shape)
        per_prompt = ream_counts(packed)
        self.counts = per_prompt.to(torch.int64).sum(0).cpu().numpy().reshape(
            shape.num_layers, shape.num_experts)
        E = shape.num_experts
        # order[l] = ids by (-count, id): a stable argsort of -count
        self._order = np.argsort(-self.counts, axis=1, kind="stable")
        self._tables: dict[tuple, torch.Tensor] = {}  # (budget, device) -> table

    def _table(self, budget: int, device) -> torch.Tensor:
        key = (budget, str(device))
        if key not in self._tables:
            L, W = self.shape.num_layers, self.shape.mask_words
            m = min(budget, self.shape.num_experts)
            tab = np.zeros((L, W), dtype=np.uint64)
            for l in range(L):
                for e in self._order[l, :m]:
                    tab[l, e >> 6] |= np.uint64(1) << np.uint64(e & 63)
            self._tables[key] = torch.from_numpy(tab.view(np.int64)).to(device)
        return self._tables[key]

    def predict_masks(self, packed, budget, warmup=0, metrics=None):
        return _policy(3, packed, budget, table=self._table(budget, packed.device))


class EamCosinePredictor(DevicePredictor):
    """Nearest stored sketch by cosine over the partial rEAM; top-budget
    positive weights of its block (predictors.py:151-219). Kernel K6."""

    kind = "eam_cosine"
    uses_partial_ream = True

    def __init__(self, collection: SketchCollection):
        if len(collection) == 0:
            raise ConfigError("eam_cosine needs a non-empty sketch collection")
        self.collection = collection
        self.shape = collection.shape

    def predict_masks(self, packed, budget, warmup=0, metrics=None, idx_out=None):
        unit_t, topw = self.collection.device_tables(budget, packed.device)
        out = _empty(packed)
        s = self.shape
        nat.call("moeb_eam_predict", nat.ptr(packed.truth), nat.ptr(packed.row_off),
                 packed.num_prompts, s.num_layers, s.num_experts, int(warmup), nat.ptr(unit_t),
                 nat.ptr(topw), len(self.collection), nat.ptr(idx_out), nat.ptr(out),
                 nat.stream_ptr())
        return out


class ExternalPredictor(DevicePredictor):
    """Lookup into an external prediction table; missing keys predict nothing
    and count as uncovered (predictors.py:222-242, engine.py:175-176)."""

    kind = "external"

    def __init__(self, table: dict, shape: ModelShape):
        self.shape = shape
        self.table = table      # as given: a dict (reference form) or a PredictionTable
        self._tables = {}       # device -> PredictionTable
        self._last = None       # (packed, (masks, coverage)) of the last join

    def covers(self, prompt_id: int, token_index: int, layer_id: int) -> bool:
        return (prompt_id, token_index, layer_id) in self.table

    def _table_on(self, device):
        from .traceio import PredictionTable
        if isinstance(self.table, PredictionTable) and self.table.prompt_id.device == device:
            return self.table
        key = str(device)
        if key not in self._tables:
            self._tables[key] = (self.table.to(device) if isinstance(self.table, PredictionTable)
                                 else PredictionTable.from_dict(self.table, self.shape, device))
        return self._tables[key]

    def _build(self, packed: PackedTraces):
        """Masks + coverage per trace row: the table (key-sorted device
        arrays, one copy per device) joined onto the rows on device
        (moeb_predictions_join). The last join is reused only for the very
        same PackedTraces object (predict_masks + coverage of one replay)."""
        from .traceio import join_predictions
        if self._last is not None and self._last[0] is packed:
            return self._last[1]
        res = join_predictions(self._table_on(packed.device), packed)
        self._last = (packed, res)
        return res

    def predict_masks(self, packed, budget, warmup=0, metrics=None):
        return self._build(packed)[0]

    def coverage(self, packed):
        return self._build(packed)[1]


class LearnedLinearPredictor(DevicePredictor):
    """Linear model over decayed-history features (predictors.py:245-268).
    Kernel K3 with the selection head and (optionally) metrics fused."""

    kind = "learned_linear"
    uses_history = True

    def __init__(self, model: LinearModel, threshold: bool = False):
        if not model.trained:
            raise ConfigError("learned_linear needs a trained model")
        self.model = model
        self.shape = model.shape
        self.threshold = threshold
        self._w = {}

    @property
    def history_decay(self) -> float:
        return self.model.config.decay

    def weights_on(self, device) -> torch.Tensor:
        key = str(device)
        if key not in self._w:
            self._w[key] = torch.from_numpy(
                np.ascontiguousarray(self.model.weights, dtype=np.float64)).to(device)
        return self._w[key]

    def tables_on(self, device) -> torch.Tensor:
        """Wide-kernel tables (moeb_linear_prepare) for E > 64."""
        key = ("tab", str(device))
        if key not in self._w:
            s = self.shape
            lib = nat.load_library()
            n = lib.moeb_linear_table_doubles(s.num_layers, s.num_experts)
            tab = torch.empty(n, dtype=torch.float64, device=device)
            nat.call("moeb_linear_prepare", nat.ptr(self.weights_on(device)), s.num_layers,
                     s.num_experts, float(self.history_decay), nat.ptr(tab), nat.stream_ptr())
            self._w[key] = tab
        return self._w[key]

    def _workspace(self, nbytes: int, device):
        """K3t's scratch, kept per (device, stream) and grown when needed:
        calls on one stream are ordered, so reusing it is safe, and a fresh
        600 MB allocation per call could make the caching allocator fall back
        to cudaMalloc (and its implicit synchronisation) in a pipeline."""
        if nbytes <= 0:
            return None
        key = (str(device), torch.cuda.current_stream(device).cuda_stream)
        cache = self.__dict__.setdefault("_ws", {})
        ws = cache.get(key)
        if ws is None or ws.numel() < nbytes:
            ws = cache[key] = nat.workspace(nbytes, device)
        return ws

    def ambiguous_rows(self) -> int | None:
        """Rows of the last predict_masks call that the tensor-core kernel
        (K3t) handed to the exact fp64 re-evaluation (None: K3t not used)."""
        ws = getattr(self, "last_workspace", None)
        if ws is None:
            return None
        out = torch.zeros(1, dtype=torch.int64, device=ws.device)
        nat.call("moeb_linear_ambiguous_rows", nat.ptr(ws), self.shape.num_layers, nat.ptr(out),
                 nat.stream_ptr())
        return int(out.item())

    @property
    def supports_counts(self) -> bool:
        """predict_masks(counts=...) fills the replay's cache-independent
        counters (E <= 64 kernel only)."""
        return self.shape.num_experts <= 64

    # predict_masks(out=...) writes into a caller-owned [rows][W] int64 buffer
    # (pipelines keep one per batch slot instead of allocating 528 MB a step)
    supports_out = True

    def predict_masks(self, packed, budget, warmup=0, metrics=None, logits=None, counts=None,
                      out=None):
        s = self.shape
        if out is None:
            out = _empty(packed)
        elif tuple(out.shape) != (packed.rows, s.mask_words) or out.dtype != torch.int64:
            raise ConfigError("out must be int64 [rows][mask words]")
        if counts is not None and s.num_experts > 64:
            raise ConfigError("fused replay counts need E <= 64")
        if s.num_experts > 64:
            nat.call("moeb_linear_predict_wide", nat.ptr(packed.truth), nat.ptr(packed.row_off),
                     packed.num_prompts, s.num_layers, s.num_experts,
                     nat.ptr(self.tables_on(packed.device)), float(self.history_decay),
                     int(budget), int(bool(self.threshold)), int(warmup), nat.ptr(out),
                     nat.ptr(logits), nat.ptr(metrics), nat.stream_ptr())
            return out
        ws_bytes = 0 if logits is not None else nat.load_library().moeb_linear_workspace_bytes(
            packed.rows, s.num_layers, s.num_experts)
        ws = self._workspace(ws_bytes, packed.device)
        self.last_workspace = ws
        nat.call("moeb_linear_predict_counts", nat.ptr(packed.truth), nat.ptr(packed.row_off),
                 packed.num_prompts, s.num_layers, s.num_experts,
                 nat.ptr(self.weights_on(packed.device)), float(self.history_decay),
                 int(budget), int(bool(self.threshold)), int(warmup), s.top_k, nat.ptr(out),
                 nat.ptr(logits), nat.ptr(metrics), nat.ptr(counts), packed.rows, nat.ptr(ws),
                 ws_bytes, nat.stream_ptr())
        return out


def make_predictor(kind: str, shape: ModelShape, *, traces=None, train_traces=None,
                   eamc: SketchCollection | None = None, model: LinearModel | None = None,
                   predictions: dict | None = None, threshold: bool = False,
                   transformer=None):
    """Build a predictor, checking its required state (predictors.py:271-303)."""
    if kind == "oracle":
        if traces is None:
            raise ConfigError("oracle predictor needs the replayed traces")
        return OraclePredictor(traces, shape)
    if kind == "lru_only":
        return LruOnlyPredictor(shape)
    if kind == "next_layer_all":
        return NextLayerAllPredictor(shape)
    if kind == "global_frequency":
        if train_traces is None:
            raise ConfigError("global_frequency predictor needs training traces")
        return GlobalFrequencyPredictor(train_traces, shape)
    if kind == "eam_cosine":
        if eamc is None:
            raise ConfigError("eam_cosine predictor needs a sketch collection")
        return EamCosinePredictor(eamc)
    if kind == "external":
        if predictions is None:
            raise ConfigError("external predictor needs a prediction table")
        return ExternalPredictor(predictions, shape)
    if kind == "learned_linear":
        if model is None:
            raise ConfigError("learned_linear predictor needs a trained model")
        return LearnedLinearPredictor(model, threshold=threshold)
    if kind == "transformer":
        from .transformer import TransformerPredictor
        if transformer is None:
            raise ConfigError("transformer predictor needs weights (TransformerWeights)")
        return TransformerPredictor(transformer, shape, threshold=threshold)
    raise ConfigError(f"unknown predictor kind {kind!r}")
