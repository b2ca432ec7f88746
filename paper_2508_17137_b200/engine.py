"""Trace replay under a predictor and an expert cache (engine.py in the reference).

Same configuration objects, report type and call signatures as
``moesim.engine``; the work runs on the GPU in three stream-ordered launches
per batch: predictor masks (predictors.py), the fused metrics counters, and
the cache replay K1 (moeb_cache_sim) for every requested capacity at once.
``jobs`` is accepted for signature compatibility; parallelism is the GPU's
(multi-GPU sharding: distributed.py).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import os

import numpy as np
import torch

from . import _native as nat
from .cache import POLICIES, CacheConfig
from .core import ConfigError, ModelShape, RangeError
from .metrics import MetricCounts, mask_metrics, metric_vector
from .traces import (PackedTraces, ids6_to_masks, ids_to_masks, idpairs_to_masks, pack_traces,
                     ranks_to_masks)


@dataclass(frozen=True)
class ReplayConfig:
    shape: ModelShape
    cache: CacheConfig
    warmup_tokens: int = 8
    history_decay: float = 0.9

    def __post_init__(self):
        if self.warmup_tokens < 0:
            raise ConfigError(f"warmup_tokens must be >= 0, got {self.warmup_tokens}")
        if not 0.0 <= self.history_decay < 1.0:
            raise ConfigError(f"history_decay must be in [0, 1), got {self.history_decay}")


@dataclass
class PromptCounters:
    measured_accesses: int = 0
    cache_hits: int = 0
    prediction_opportunities: int = 0
    prediction_hits: int = 0


def _rate(hits: int, denom: int):
    return hits / denom if denom else None


@dataclass
class SimReport:
    """Aggregate and per-prompt counters for one replay run (engine.py:62-110)."""

    shape: ModelShape
    measured_accesses: int = 0
    cache_hits: int = 0
    prediction_opportunities: int = 0
    prediction_hits: int = 0
    uncovered_queries: int = 0
    layer_accesses: np.ndarray = None
    layer_cache_hits: np.ndarray = None
    layer_prediction_hits: np.ndarray = None
    per_prompt: dict = field(default_factory=dict)

    def __post_init__(self):
        L = self.shape.num_layers
        if self.layer_accesses is None:
            self.layer_accesses = np.zeros(L, dtype=np.int64)
        if self.layer_cache_hits is None:
            self.layer_cache_hits = np.zeros(L, dtype=np.int64)
        if self.layer_prediction_hits is None:
            self.layer_prediction_hits = np.zeros(L, dtype=np.int64)

    @property
    def cache_hit_rate(self):
        return _rate(self.cache_hits, self.measured_accesses)

    @property
    def prediction_hit_rate(self):
        return _rate(self.prediction_hits, self.prediction_opportunities)

    def merge(self, other: "SimReport") -> None:
        self.measured_accesses += other.measured_accesses
        self.cache_hits += other.cache_hits
        self.prediction_opportunities += other.prediction_opportunities
        self.prediction_hits += other.prediction_hits
        self.uncovered_queries += other.uncovered_queries
        self.layer_accesses += other.layer_accesses
        self.layer_cache_hits += other.layer_cache_hits
        self.layer_prediction_hits += other.layer_prediction_hits
        self.per_prompt.update(other.per_prompt)

    @classmethod
    def aggregate(cls, shape: ModelShape, reports) -> "SimReport":
        total = cls(shape)
        for r in reports:
            total.merge(r)
        return total

    @classmethod
    def from_counters(cls, shape: ModelShape, vec, per_prompt=None, prompt_ids=None):
        """From the K1 counter vector [4+3L] (and per-prompt [P,4])."""
        v = np.asarray(vec, dtype=np.int64)
        L = shape.num_layers
        rep = cls(shape, int(v[0]), int(v[1]), int(v[0]), int(v[2]), int(v[3]),
                  v[4:4 + L].copy(), v[4 + L:4 + 2 * L].copy(), v[4 + 2 * L:4 + 3 * L].copy())
        if per_prompt is not None:
            pp = np.asarray(per_prompt, dtype=np.int64)
            for pid, row in zip(prompt_ids, pp):
                rep.per_prompt[int(pid)] = PromptCounters(int(row[0]), int(row[1]), int(row[0]),
                                                          int(row[2]))
        return rep


def _packed(traces, shape: ModelShape) -> PackedTraces:
    return traces if isinstance(traces, PackedTraces) else pack_traces(traces, shape)


def _check_lengths(packed: PackedTraces, warmup: int) -> None:
    """replay_prompt refuses prompts not longer than the warm-up (engine.py:123-127)."""
    short = np.nonzero(packed.num_tokens <= warmup)[0]
    if len(short):
        i = int(short[0])
        raise ConfigError(f"prompt {int(packed.prompt_ids[i])} has {int(packed.num_tokens[i])} "
                          f"tokens, not more than warmup_tokens={warmup}")


def _stack_multi_caps(packed, streams, capacities, budget, policy, want_hits):
    """Indices of the capacities K1m takes (see cache_replay). MOEB_K1M=0
    disables it, MOEB_K1M=all uses it for every capacity it is exact for."""
    mode = os.environ.get("MOEB_K1M", "")
    shape = packed.shape
    if mode == "0" or policy != "lru" or want_hits or shape.num_experts > 64:
        return []
    if any(c is not None for _, c, _ in streams) or not packed.num_prompts:
        return []
    if int(np.max(np.diff(packed.row_off_host))) > 32768:
        return []
    kmax = shape.num_experts if any(u for _, _, u in streams) else budget
    if mode == "all":
        return [j for j, c in enumerate(capacities) if c > kmax]
    # K1s decides the small capacities of predicted streams in ~1 ms; K1m's
    # one pass costs about as much as 5 capacities of the exact kernel, so it
    # takes over when it replaces at least 6 of them
    keys = shape.num_layers * shape.num_experts
    with_preds = all(mk is not None for mk, _, _ in streams)
    lo = max(kmax, int(0.12 * keys)) if with_preds else kmax
    idx = [j for j, c in enumerate(capacities) if c > lo]
    return idx if len(idx) >= 6 else []


def _stack_multi(packed, streams, capacities, idx, warmup, budget, counters, per_prompt):
    shape = packed.shape
    L = shape.num_layers
    rmax = int(np.max(np.diff(packed.row_off_host)))
    idx = sorted(idx, key=lambda j: capacities[j])  # the kernel takes ascending capacities
    # the per-key last-access tables in caller-owned global memory (more
    # prompts resident per SM than with them in shared memory)
    ws_bytes = nat.load_library().moeb_cache_replay_stack_workspace_bytes(
        len(streams), packed.num_prompts, L)
    ws = nat.workspace(ws_bytes, packed.device)
    for g in range(0, len(idx), 16):
        sel = idx[g:g + 16]
        sc = torch.zeros((len(streams), len(sel), 4 + 3 * L), dtype=torch.int64,
                         device=packed.device)
        sp = (torch.zeros((len(streams), len(sel), packed.num_prompts, 4), dtype=torch.int64,
                          device=packed.device) if per_prompt is not None else None)
        nat.call("moeb_cache_replay_stack", nat.ptr(packed.truth),
                 nat.ptr_array([m for m, _, _ in streams]),
                 nat.i32_array([int(bool(u)) for _, _, u in streams]), len(streams),
                 nat.ptr(packed.row_off), packed.num_prompts, L, shape.num_experts, int(warmup),
                 nat.i64_array([capacities[j] for j in sel]), len(sel), int(budget), rmax,
                 shape.top_k, nat.ptr(sc), nat.ptr(sp), nat.ptr(ws), ws_bytes, nat.stream_ptr())
        counters[:, sel] += sc
        if per_prompt is not None:
            per_prompt[:, sel] += sp


def cache_replay(packed: PackedTraces, streams, capacities, warmup: int, budget: int,
                 policy: str = "lru", want_per_prompt: bool = True, want_hits: bool = False,
                 counters=None, given_counts=None, _per_prompt=None, _no_multi=False):
    """Run K1 for every (prediction stream, capacity) pair in one call.

    ``streams`` is a list of (masks | None, coverage | None, unbounded).
    Returns device tensors counters [n][C][4+3L], per_prompt [n][C][P][4] or
    None, hit masks [n][C][rows][W] or None. ``counters`` (optional, int64
    [n][C][4+3L]) is accumulated into instead of a fresh zero tensor.
    ``given_counts`` (optional, int64 [n][2+2L], e.g. from the learned_linear
    predictor's fused counts) supplies the cache-independent counters so the
    replay kernel skips them (moeb_cache_sim_counted); results are identical.
    """
    shape = packed.shape
    L = shape.num_layers
    n, C, P = len(streams), len(capacities), packed.num_prompts
    dev = packed.device
    if P and int(np.max(np.diff(packed.row_off_host))) >= 2**31 - 64:
        raise RangeError("a prompt has >= 2^31 - 64 trace rows (cache replay limit)")
    if counters is None:
        counters = torch.zeros((n, C, 4 + 3 * L), dtype=torch.int64, device=dev)
    elif tuple(counters.shape) != (n, C, 4 + 3 * L) or counters.dtype != torch.int64:
        raise ConfigError("counters must be int64 [streams][capacities][4+3L]")
    per_prompt = (torch.zeros((n, C, P, 4), dtype=torch.int64, device=dev)
                  if want_per_prompt else _per_prompt)
    hits = (torch.zeros((n, C, packed.rows, shape.mask_words), dtype=torch.int64, device=dev)
            if want_hits else None)
    # K1m (moeb_cache_replay_stack): every capacity above the K1s range
    # (and above the keys a row can prefetch, so no pin binds) in one exact
    # stack-distance pass; the others take K1s / the exact kernel below
    multi = ([] if _no_multi else
             _stack_multi_caps(packed, streams, capacities, budget, policy, want_hits))
    if multi:
        _stack_multi(packed, streams, capacities, multi, warmup, budget, counters, per_prompt)
        rest = [j for j in range(C) if j not in multi]
        if not rest:
            return counters, per_prompt, hits
        sub_c = counters[:, rest].contiguous()
        sub_p = per_prompt[:, rest].contiguous() if per_prompt is not None else None
        cache_replay(packed, streams, [capacities[j] for j in rest], warmup, budget, policy,
                     want_per_prompt=False, counters=sub_c, given_counts=given_counts,
                     _per_prompt=sub_p, _no_multi=True)
        counters[:, rest] = sub_c
        if per_prompt is not None:
            per_prompt[:, rest] = sub_p
        return counters, per_prompt, hits
    lib = nat.load_library()
    ws_bytes = lib.moeb_cache_sim_workspace_bytes_shape(min(n, 16), P, L, shape.num_experts)
    ws = nat.workspace(ws_bytes, dev)
    for lo in range(0, n, 16):
        chunk = streams[lo:lo + 16]
        nat.call("moeb_cache_sim_counted", nat.ptr(packed.truth),
                 nat.ptr_array([m for m, _, _ in chunk]),
                 nat.ptr_array([c for _, c, _ in chunk]),
                 nat.i32_array([int(bool(u)) for _, _, u in chunk]), len(chunk),
                 nat.ptr(packed.row_off), P, L, shape.num_experts, int(warmup),
                 nat.i64_array(capacities), C, int(budget), POLICIES[policy],
                 nat.ptr(counters[lo:lo + 16]),
                 nat.ptr(None if per_prompt is None else per_prompt[lo:lo + 16]),
                 nat.ptr(None if hits is None else hits[lo:lo + 16]),
                 nat.ptr(None if given_counts is None else given_counts[lo:lo + 16]),
                 packed.rows, nat.ptr(ws), ws_bytes, nat.stream_ptr())
    return counters, per_prompt, hits


def predict_stream(predictor, packed: PackedTraces, config: ReplayConfig, metrics=None):
    """(masks, coverage, unbounded) of one predictor over a packed batch."""
    budget = config.cache.prefetch_budget
    if getattr(predictor, "empty", False) and metrics is None:
        return None, None, False
    masks = predictor.predict_masks(packed, budget, config.warmup_tokens, metrics=metrics)
    return masks, predictor.coverage(packed), bool(getattr(predictor, "unbounded_prefetch", False))


def _group_world() -> int:
    import torch.distributed as dist
    return dist.get_world_size() if dist.is_available() and dist.is_initialized() else 1


def _job_devices(jobs: int, packed: PackedTraces) -> list:
    """``jobs`` -> GPUs: the reference fans prompts out over
    `jobs` worker processes (engine.py:222-238); here over up to `jobs`
    visible GPUs of this process (the caller's device first)."""
    n = min(max(1, int(jobs)), torch.cuda.device_count(), max(1, packed.num_prompts))
    first = packed.device.index if packed.device.type == "cuda" else torch.cuda.current_device()
    return [torch.device("cuda", (first + i) % torch.cuda.device_count()) for i in range(n)]


def _replay_on_devices(packed: PackedTraces, predictor, config: ReplayConfig, caps, policy: str,
                       per_prompt: bool, devices):
    """Row-balanced prompt shards, one per device, launched asynchronously on
    each device's current stream; counters summed (integer, order-free) and
    per-prompt counters concatenated in prompt order on the host."""
    budget, warmup = config.cache.prefetch_budget, config.warmup_tokens
    launched = []
    for i, dev in enumerate(devices):
        shard = packed.shard(i, len(devices)).to(dev)
        with torch.cuda.device(dev):
            stream = predict_stream(predictor, shard, config)
            counters, pp, _ = cache_replay(shard, [stream], caps, warmup, budget, policy,
                                           per_prompt)
        launched.append((shard, counters, pp))
    vec = sum(c[0].cpu().numpy() for _, c, _ in launched)
    pp = (np.concatenate([p[0].cpu().numpy() for _, _, p in launched], axis=1)
          if per_prompt else None)
    ids = np.concatenate([s.prompt_ids for s, _, _ in launched])
    return vec, pp, ids


def replay_traces(traces, predictor, config: ReplayConfig, jobs: int = 1, policy: str = "lru",
                  per_prompt: bool = True) -> SimReport:
    """Replay every prompt; counters identical to the reference for any batch
    split and any ``jobs`` (engine.py:222-238; results are integer sums).

    ``jobs`` maps to GPUs: with an initialised torch.distributed group of
    more than one rank (one process per GPU, torchrun) every rank passes the
    same traces, replays its row-balanced prompt shard and the counters are
    all-reduced (``distributed.replay_sharded``; every rank returns the whole
    report); otherwise ``jobs`` > 1 spreads the prompts over up to ``jobs``
    GPUs visible to this process."""
    packed = _packed(traces, config.shape)
    _check_lengths(packed, config.warmup_tokens)
    if _group_world() > 1:
        from .distributed import replay_sharded
        return replay_sharded(packed, predictor, config, policy=policy, per_prompt=per_prompt)
    cap = config.cache.resolve_capacity(config.shape)
    devices = _job_devices(jobs, packed)
    if len(devices) > 1:
        vec, pp, ids = _replay_on_devices(packed, predictor, config, [cap], policy, per_prompt,
                                          devices)
        return SimReport.from_counters(config.shape, vec[0], None if pp is None else pp[0], ids)
    stream = predict_stream(predictor, packed, config)
    counters, pp, _ = cache_replay(packed, [stream], [cap], config.warmup_tokens,
                                   config.cache.prefetch_budget, policy, per_prompt)
    return SimReport.from_counters(
        config.shape, counters[0, 0].cpu().numpy(),
        None if pp is None else pp[0, 0].cpu().numpy(), packed.prompt_ids)


class PipelinedReplay:
    """Prediction + cache replay over prompt chunks on overlapping streams.

    Prompts are independent (``engine.py:94-110`` fans them out to a process
    pool), so a batch is cut into ``chunks`` row-balanced prompt ranges and
    issued as a three-stage pipeline: [copy stream] host->device copy of the
    chunk's truth rows (only when ``host_truth`` is given: pinned uint64 rows
    of the whole batch), [predict stream] the predictor's masks (+ fused metric
    counters), [replay stream] K1 for the chunk. Chunk c's replay runs while
    chunk c+1 is predicted and chunk c+2 copied. All counters are integer sums
    accumulated with atomics, so results are identical to one unchunked call.
    The chunk views are built once (construction does host work that would
    otherwise serialise the streams).
    """

    def __init__(self, packed: PackedTraces, chunks: int = 4, overlap_steps: bool = False):
        """``overlap_steps``: consecutive ``run`` calls overlap -- call i+1's
        predictor runs while call i's replay and metrics finish (two mask
        buffers used alternately; the predictor stream has the highest
        priority so its persistent kernel is placed first and the replay fills
        the resources it leaves). ``run`` then returns without ordering the
        caller's stream after the work: call ``join()`` before reading any
        result."""
        self.packed = packed
        self.overlap = bool(overlap_steps)
        self._slot = 0
        self._slot_done = {}
        P = packed.num_prompts
        chunks = max(1, min(int(chunks), P))
        targets = np.arange(1, chunks) * (packed.rows / chunks)
        cuts = np.searchsorted(packed.row_off_host, targets)
        bounds = sorted(set([0] + [int(c) for c in cuts] + [P]))
        self.bounds = [(a, b) for a, b in zip(bounds[:-1], bounds[1:]) if b > a]
        self.views = [packed.select(a, b) for a, b in self.bounds]
        self._host_off = None
        dev = packed.device
        self._mbufs = {}  # persistent masks per chunk (predictors with out=)
        self.s_copy = torch.cuda.Stream(dev)
        self.s_pred = torch.cuda.Stream(dev, priority=-2 if self.overlap else 0)
        self.s_sim = torch.cuda.Stream(dev, priority=-1)
        self.s_met = torch.cuda.Stream(dev, priority=0)

    def host_offsets(self):
        """Pinned host copies of each chunk's rebased row offsets (copied with
        the truth rows when the batch comes from host memory)."""
        if self._host_off is None:
            self._host_off = [torch.from_numpy(np.ascontiguousarray(v.row_off_host)).pin_memory()
                              for v in self.views]
        return self._host_off

    @property
    def h2d_offset_bytes(self) -> int:
        return sum(8 * (b - a + 1) for a, b in self.bounds)

    def run(self, predictor, capacities, warmup: int, budget: int, policy: str = "lru",
            metrics=None, host_truth=None, counters=None, timing=None, per_prompt: bool = False):
        """Enqueue the pipeline; returns counters [1][C][4+3L] (device, ordered
        on the caller's current stream). ``metrics`` (int64 [3E+3]) receives the
        fused prediction metrics when the predictor supports them. ``timing``
        (a list) receives (stage, start_event, end_event, rows) per launch,
        recorded on the launching stream."""
        ev = (lambda: torch.cuda.Event(enable_timing=True)) if timing is not None else None
        shape, packed = self.packed.shape, self.packed
        main = torch.cuda.current_stream(packed.device)
        if counters is None:
            counters = torch.zeros((1, len(capacities), 4 + 3 * shape.num_layers),
                                   dtype=torch.int64, device=packed.device)
        for s in (self.s_copy, self.s_pred, self.s_sim, self.s_met):
            s.wait_stream(main)
        slot = self._slot
        if self.overlap:
            # this slot's mask buffers were last read by the replay / metrics
            # of the call before the previous one
            for done in self._slot_done.get(slot, ()):
                self.s_pred.wait_event(done)
            self._slot ^= 1
        unbounded = bool(getattr(predictor, "unbounded_prefetch", False))
        pps = []
        for ci, ((a, b), view) in enumerate(zip(self.bounds, self.views)):
            if host_truth is not None:
                r0, r1 = int(packed.row_off_host[a]), int(packed.row_off_host[b])
                with torch.cuda.stream(self.s_copy):
                    view.truth.copy_(host_truth[r0:r1], non_blocking=True)
                    view.row_off.copy_(self.host_offsets()[ci],
                                       non_blocking=True)
                self.s_pred.wait_stream(self.s_copy)
            with torch.cuda.stream(self.s_pred):
                gc = None
                if getattr(predictor, "empty", False) and metrics is None:
                    masks, cov = None, None
                else:
                    if ev:
                        e0, e1 = ev(), ev()
                        e0.record(self.s_pred)
                    gc = _counts_buffer(predictor, shape, packed.device)
                    masks = predictor.predict_masks(view, budget, warmup, **_counts_kw(gc),
                                                    **_out_kw(predictor, self._mbufs, (slot, ci), view))
                    if ev:
                        e1.record(self.s_pred)
                        timing.append(("predict", e0, e1, view.rows))
                    cov = predictor.coverage(view)
            masks_ready = torch.cuda.Event()
            masks_ready.record(self.s_pred)
            self.s_sim.wait_event(masks_ready)
            for t in (masks, cov, gc):
                if t is not None:
                    t.record_stream(self.s_sim)
            with torch.cuda.stream(self.s_sim):
                if ev:
                    e2, e3 = ev(), ev()
                    e2.record(self.s_sim)
                _, pp, _ = cache_replay(view, [(masks, cov, unbounded)], capacities, warmup,
                                        budget, policy, want_per_prompt=per_prompt,
                                        counters=counters, given_counts=gc)
                if ev:
                    e3.record(self.s_sim)
                    timing.append(("replay", e2, e3, view.rows))
                if per_prompt:
                    pps.append(pp)
            if metrics is not None and masks is not None:
                _overlapped_metrics(self.s_met, masks_ready, masks, view, warmup, metrics)
        # per-prompt counters [1][C][P][4] (SimReport.per_prompt, engine.py:75)
        self.last_per_prompt = None
        if per_prompt:
            with torch.cuda.stream(self.s_sim):
                self.last_per_prompt = pps[0] if len(pps) == 1 else torch.cat(pps, dim=2)
            self.last_per_prompt.record_stream(self.s_sim)
        if self.overlap:
            done = (torch.cuda.Event(), torch.cuda.Event())
            done[0].record(self.s_sim)
            done[1].record(self.s_met)
            self._slot_done[slot] = done
        else:
            self.join()
        counters.record_stream(self.s_sim)
        if metrics is not None:
            metrics.record_stream(self.s_met)
        return counters

    def join(self):
        """Order the caller's stream after every launched call."""
        main = torch.cuda.current_stream(self.packed.device)
        main.wait_stream(self.s_sim)
        main.wait_stream(self.s_pred)
        main.wait_stream(self.s_met)


def _counts_buffer(predictor, shape, device):
    """[1][2+2L] zeros when the predictor fuses the replay's cache-independent
    counters (measured accesses, prediction hits) into its kernel, else None."""
    if not getattr(predictor, "supports_counts", False):
        return None
    return torch.zeros((1, 2 + 2 * shape.num_layers), dtype=torch.int64, device=device)


def _counts_kw(gc):
    return {} if gc is None else {"counts": gc[0]}


def _out_kw(predictor, bufs: dict, key, packed: PackedTraces):
    """A persistent masks buffer per pipeline slot for predictors that take
    out= (a fresh 528 MB tensor per step makes the caching allocator fall
    back to cudaMalloc / cudaFree, which synchronise, inside the pipeline)."""
    if not getattr(predictor, "supports_out", False):
        return {}
    b = bufs.get(key)
    if b is None or b.shape[0] != packed.rows:
        b = bufs[key] = torch.empty((packed.rows, packed.shape.mask_words), dtype=torch.int64,
                                    device=packed.device)
    return {"out": b}


def _overlapped_metrics(s_met, masks_ready, masks, view, warmup, out):
    """K7 on a low-priority stream, issued after the replay (K1) launch on the
    high-priority one: K1's blocks are placed first (one resident wave), and
    the HBM-streaming metrics pass fills the resources they leave free
    instead of running between the predictor and the replay."""
    s_met.wait_event(masks_ready)
    masks.record_stream(s_met)
    view.truth.record_stream(s_met)
    with torch.cuda.stream(s_met):
        mask_metrics(masks, view.truth, view.row_off, view.shape.num_layers,
                     view.shape.num_experts, warmup, out=out)


class StreamingReplay:
    """Predict + replay over a sequence of host-resident batches of one prompt
    geometry (same row offsets), double-buffered: batch i+1's host->device
    copy runs on a copy stream while batch i is predicted and replayed on the
    compute stream (three device buffers), and each batch's counters (plus
    prediction metrics) go back to pinned host memory asynchronously. Throughput is
    max(copy, compute) per batch instead of their sum. The first batch has no
    compute to hide its copy behind, so it is copied in ``first_chunks``
    row-balanced prompt ranges and the predictor starts on each range as it
    lands (the replay needs the whole batch's masks).

    A host batch is either the int64 mask rows [rows][W] or, for E <= 64, a
    compact wire format decoded into masks on the copy stream: the u8 expert
    ids of ``masks_to_ids`` ([rows][k], 6 B/row at k = 6; ``ids_bad`` turns 1
    if an id was >= E) or the int32 combinatorial ranks of ``masks_to_ranks``
    ([rows], 4 B/row; ``ids_bad`` turns 1 for a rank >= C(E, k)).

    ``run`` returns, per batch, pinned host tensors (counters [C][4+3L],
    metrics [3E+3] or None, and with ``per_prompt`` the per-prompt counters
    [C][P][4]), valid after ``torch.cuda.synchronize()``."""

    # device batch buffers: batch i+1 is copied while batch i computes, and a
    # buffer is refilled only after the metrics pass (a low-priority stream
    # that trails the compute stream) of the batch that used it two batches
    # earlier, so the copy engine never waits for it
    NBUF = 3

    def __init__(self, shape: ModelShape, row_off_host: np.ndarray, prompt_ids, device=None,
                 token_ids=None, first_chunks: int = 4):
        dev = torch.device(device) if device is not None else torch.device(
            "cuda", torch.cuda.current_device())
        self.shape = shape
        rows = int(row_off_host[-1])
        off_d = torch.from_numpy(np.ascontiguousarray(row_off_host, dtype=np.int64)).to(dev)
        self.bufs = [PackedTraces(shape, torch.empty((rows, shape.mask_words), dtype=torch.int64,
                                                     device=dev), off_d,
                                  np.asarray(row_off_host, dtype=np.int64),
                                  np.asarray(prompt_ids, dtype=np.int64), token_ids)
                     for _ in range(self.NBUF)]
        self.ids_bufs = [None] * self.NBUF  # device staging for compact (id / rank) batches
        self.ids_bad = torch.zeros(1, dtype=torch.int32, device=dev)
        self._mbufs = {}  # persistent masks per buffer slot (predictors with out=)
        self.s_copy = torch.cuda.Stream(dev)
        self.s_dec = torch.cuda.Stream(dev)
        self.s_comp = torch.cuda.Stream(dev, priority=-1)
        # MOEB_STREAM_OVERLAP=1: batch i's replay on its own stream, beside
        # batch i+1's predictor (measured: no end-to-end gain -- the batch
        # decode and the predictor already fill the GPU -- so off by default)
        self.s_rep = (torch.cuda.Stream(dev, priority=-1)
                      if os.environ.get("MOEB_STREAM_OVERLAP") == "1" else self.s_comp)
        self.s_met = torch.cuda.Stream(dev, priority=0)
        self.device = dev
        P = len(prompt_ids)
        n = max(1, min(int(first_chunks), P))
        cuts = np.searchsorted(self.bufs[0].row_off_host, np.arange(1, n) * (rows / n))
        b = sorted(set([0] + [int(c) for c in cuts] + [P]))
        self.first_views = [self.bufs[0].select(lo, hi) for lo, hi in zip(b[:-1], b[1:]) if hi > lo]

    @property
    def rows(self) -> int:
        return self.bufs[0].rows

    def run(self, predictor, capacities, warmup: int, budget: int, host_batches,
            policy: str = "lru", metrics: bool = False, timing=None, per_prompt: bool = False,
            wire: str | None = None):
        """``wire="ids6"`` / ``"idpairs"``: the host batches are packed
        6-bit id / id-pair streams (``masks_to_ids6`` / ``masks_to_idpairs``);
        otherwise the format follows the batch's dtype / shape (masks, u8 ids,
        ranks)."""
        shape, dev = self.shape, self.device
        L, E = shape.num_layers, shape.num_experts
        main = torch.cuda.current_stream(dev)
        self.s_copy.wait_stream(main)
        self.s_dec.wait_stream(main)
        self.s_comp.wait_stream(main)
        self.s_rep.wait_stream(main)
        self.s_met.wait_stream(main)
        copied = [torch.cuda.Event() for _ in range(self.NBUF)]
        freed = [None] * self.NBUF
        out = []
        host_batches = list(host_batches)
        # every batch's pinned read-back buffers up front, before any work is
        # enqueued (a host allocation between launches would stall the pipeline)
        P = self.bufs[0].num_prompts
        outs = [(torch.empty((len(capacities), 4 + 3 * L), dtype=torch.int64, pin_memory=True),
                 torch.empty(3 * E + 3, dtype=torch.int64, pin_memory=True) if metrics else None,
                 torch.empty((len(capacities), P, 4), dtype=torch.int64, pin_memory=True)
                 if per_prompt else None)
                for _ in host_batches]
        unbounded = bool(getattr(predictor, "unbounded_prefetch", False))
        for i, hb in enumerate(host_batches):
            b = i % self.NBUF
            buf = self.bufs[b]
            empty = getattr(predictor, "empty", False) and not metrics
            ids6 = wire in ("ids6", "idpairs")  # packed ids / id pairs (a bit stream)
            ranked = not ids6 and hb.dtype == torch.int32 and hb.dim() == 1  # combinatorial ranks:
            packed_ranks = ranked and hb.shape[0] != buf.rows    # as a bit stream
            compact = ids6 or ranked or hb.dtype == torch.uint8  # or [rows][k] expert ids
            # the first batch lands in prompt ranges (not splittable: a bit stream)
            split = (i == 0 and len(self.first_views) > 1 and not empty and not packed_ranks
                     and not ids6)
            parts = []
            with torch.cuda.stream(self.s_copy):
                if freed[b] is not None:
                    for e in freed[b]:
                        if e is not None:
                            self.s_copy.wait_event(e)
                if compact:
                    ib = self.ids_bufs[b]
                    if ib is None or ib.shape != hb.shape or ib.dtype != hb.dtype:
                        ib = self.ids_bufs[b] = torch.empty(hb.shape, dtype=hb.dtype,
                                                            device=dev)

                def land(dst, r0, r1):
                    """copy rows [r0, r1) (copy stream); compact rows are decoded
                    into masks on the decode stream, so the copy engine goes on
                    to the next range / batch meanwhile. Returns the event
                    after which dst holds the masks."""
                    done = torch.cuda.Event()
                    if compact:
                        if packed_ranks or ids6:  # the whole stream (no split for it)
                            ib.copy_(hb, non_blocking=True)
                        else:
                            ib[r0:r1].copy_(hb[r0:r1], non_blocking=True)
                        landed = torch.cuda.Event()
                        landed.record(self.s_copy)
                        self.s_dec.wait_event(landed)
                        with torch.cuda.stream(self.s_dec):
                            if wire == "idpairs":
                                idpairs_to_masks(ib, shape.top_k, r1 - r0, dst, self.ids_bad)
                            elif ids6:
                                ids6_to_masks(ib, shape.top_k, r1 - r0, dst, self.ids_bad)
                            elif packed_ranks:
                                ranks_to_masks(ib, shape.top_k, E, dst, self.ids_bad, rows=r1 - r0)
                            elif ranked:
                                ranks_to_masks(ib[r0:r1], shape.top_k, E, dst, self.ids_bad)
                            else:
                                ids_to_masks(ib[r0:r1], E, dst, self.ids_bad)
                            done.record(self.s_dec)
                    else:
                        dst.copy_(hb[r0:r1], non_blocking=True)
                        done.record(self.s_copy)
                    return done

                if split:  # first batch: copy range by range, predict as each lands
                    r0 = 0
                    for v in self.first_views:
                        r1 = r0 + v.rows
                        parts.append(land(v.truth, r0, r1))
                        r0 = r1
                    copied[b] = parts[-1]
                else:
                    copied[b] = land(buf.truth, 0, buf.rows)
            with torch.cuda.stream(self.s_comp):
                if not split:
                    self.s_comp.wait_event(copied[b])
                if timing is not None:
                    e0 = torch.cuda.Event(enable_timing=True)
                    e0.record(self.s_comp)
                vec = (torch.zeros(3 * E + 3, dtype=torch.int64, device=dev)
                       if metrics else None)
                gc = None
                if empty:
                    masks, cov = None, None
                elif split:
                    gc = _counts_buffer(predictor, shape, dev)
                    pieces = []
                    for v, e in zip(self.first_views, parts):
                        self.s_comp.wait_event(e)
                        pieces.append(predictor.predict_masks(v, budget, warmup, **_counts_kw(gc)))
                    masks = torch.cat(pieces)
                    cov = predictor.coverage(buf)
                else:
                    gc = _counts_buffer(predictor, shape, dev)
                    masks = predictor.predict_masks(buf, budget, warmup, **_counts_kw(gc),
                                                    **_out_kw(predictor, self._mbufs, b, buf))
                    cov = predictor.coverage(buf)
                masks_ready = torch.cuda.Event()
                masks_ready.record(self.s_comp)
            for t in (masks, cov, gc):
                if t is not None:
                    t.record_stream(self.s_rep)
            self.s_rep.wait_event(masks_ready)
            with torch.cuda.stream(self.s_rep):
                cnt, pp, _ = cache_replay(buf, [(masks, cov, unbounded)], capacities, warmup,
                                          budget, policy, want_per_prompt=per_prompt,
                                          given_counts=gc)
                ev = torch.cuda.Event()
                ev.record(self.s_rep)
                c_h, v_h, p_h = outs[i]
                c_h.copy_(cnt[0], non_blocking=True)
                if per_prompt:
                    p_h.copy_(pp[0], non_blocking=True)
                met_ev = None
                if vec is not None:
                    # the metrics pass runs on its own (low-priority) stream and
                    # is not waited for by the next batch's predictor, only by
                    # the refill of this batch's buffer and its read-back
                    _overlapped_metrics(self.s_met, masks_ready, masks, buf, warmup, vec)
                    vec.record_stream(self.s_met)
                    with torch.cuda.stream(self.s_met):
                        v_h.copy_(vec, non_blocking=True)
                        met_ev = torch.cuda.Event()
                        met_ev.record(self.s_met)
                freed[b] = (ev, met_ev)
                if timing is not None:
                    e1 = torch.cuda.Event(enable_timing=True)
                    e1.record(self.s_rep)
                    timing.append((e0, e1))
                out.append((c_h, v_h, p_h) if per_prompt else (c_h, v_h))
        main.wait_stream(self.s_comp)
        main.wait_stream(self.s_rep)
        main.wait_stream(self.s_copy)
        main.wait_stream(self.s_dec)
        main.wait_stream(self.s_met)
        return out


def replay_prompt(trace, predictor, config: ReplayConfig) -> SimReport:
    return replay_traces([trace], predictor, config)


def prediction_metrics(traces, predictor, config: ReplayConfig) -> MetricCounts:
    """Integer metric counters over all measured steps (device), finishing on host."""
    packed = _packed(traces, config.shape)
    E = config.shape.num_experts
    vec = metric_vector(E, packed.device)
    if getattr(predictor, "kind", "") == "learned_linear" and E <= 64:
        predictor.predict_masks(packed, config.cache.prefetch_budget, config.warmup_tokens,
                                metrics=vec)
    else:
        masks = predictor.predict_masks(packed, config.cache.prefetch_budget, config.warmup_tokens)
        mask_metrics(masks, packed.truth, packed.row_off, config.shape.num_layers, E,
                     config.warmup_tokens, vec)
    return MetricCounts.from_vector(vec.cpu().numpy(), E)


def collect_prediction_sets(traces, predictor, config: ReplayConfig):
    """(pred_sets, truth_sets, layer_ids) for every measured step (engine.py:241-272).

    Masks are computed on device; the conversion to Python sets is host-side
    compatibility glue (use prediction_metrics for bulk evaluation)."""
    packed = _packed(traces, config.shape)
    masks = predictor.predict_masks(packed, config.cache.prefetch_budget, config.warmup_tokens)
    pm = masks.cpu().numpy().view(np.uint64)
    tm = packed.truth.cpu().numpy().view(np.uint64)
    L, E = config.shape.num_layers, config.shape.num_experts
    pred_sets, truth_sets, layer_ids = [], [], []
    for i in range(packed.num_prompts):
        r0 = int(packed.row_off_host[i]) + config.warmup_tokens * L
        for r in range(r0, int(packed.row_off_host[i + 1])):
            pred_sets.append(_bits(pm[r], E))
            truth_sets.append(_bits(tm[r], E))
            layer_ids.append((r - int(packed.row_off_host[i])) % L)
    return pred_sets, truth_sets, layer_ids


def _bits(words, E) -> frozenset:
    out = []
    for w, word in enumerate(words):
        word = int(word)
        while word:
            b = word & -word
            out.append(w * 64 + b.bit_length() - 1)
            word ^= b
    return frozenset(e for e in out if e < E)


@dataclass
class SweepPoint:
    capacity_fraction: float
    predictor_kind: str
    report: SimReport


def sweep(traces, predictor_factory, predictor_kind: str, capacities, shape: ModelShape,
          prefetch_budget: int, warmup_tokens: int, history_decay: float = 0.9,
          jobs: int = 1, policy: str = "lru") -> list[SweepPoint]:
    """One report per capacity fraction (engine.py:282-306). Predictions do not
    depend on the cache, so one predictor pass feeds every capacity; all
    capacities replay concurrently in one K1 launch per capacity."""
    if traces is None or (not isinstance(traces, PackedTraces) and not traces):
        raise ConfigError("sweep needs at least one trace")
    if not capacities:
        raise ConfigError("sweep needs at least one capacity")
    packed = _packed(traces, shape)
    _check_lengths(packed, warmup_tokens)
    cfgs = [ReplayConfig(shape, CacheConfig(capacity_fraction=f, prefetch_budget=prefetch_budget),
                         warmup_tokens, history_decay) for f in capacities]
    caps = [c.cache.resolve_capacity(shape) for c in cfgs]
    ids = packed.prompt_ids
    if _group_world() > 1:  # one process per GPU: this rank's shard, counters all-reduced
        import torch.distributed as dist
        from .distributed import _all_reduce_sum
        local = packed if packed.meta.get("presharded") else packed.shard(dist.get_rank(),
                                                                          dist.get_world_size())
        stream = predict_stream(predictor_factory(), local, cfgs[0])
        counters, pp, _ = cache_replay(local, [stream], caps, warmup_tokens, prefetch_budget,
                                       policy)
        counters = _all_reduce_sum(counters).cpu().numpy()
        gathered = [None] * dist.get_world_size()
        dist.all_gather_object(gathered, (pp.cpu().numpy(), local.prompt_ids))
        pp = np.concatenate([g[0] for g in gathered], axis=2)
        ids = np.concatenate([g[1] for g in gathered])
    else:
        devices = _job_devices(jobs, packed)
        if len(devices) > 1:
            counters, pp, ids = _replay_on_devices(packed, predictor_factory(), cfgs[0], caps,
                                                   policy, True, devices)
            counters, pp = counters[None], pp[None]
        else:
            stream = predict_stream(predictor_factory(), packed, cfgs[0])
            counters, pp, _ = cache_replay(packed, [stream], caps, warmup_tokens,
                                           prefetch_budget, policy)
            counters = counters.cpu().numpy()
            pp = pp.cpu().numpy()
    return [SweepPoint(f, predictor_kind,
                       SimReport.from_counters(shape, counters[0, j], pp[0, j], ids))
            for j, f in enumerate(capacities)]


# ---------------------------------------------------------------------------
# CSV reports of the device counters (engine.py:58-59, 309-383), formatted
# exactly as the reference does.
# ---------------------------------------------------------------------------

def format_rate(rate) -> str:
    return "n/a" if rate is None else repr(rate)


def sweep_csv(points) -> bytes:
    out = ["capacity_fraction,predictor,cache_hit_rate,prediction_hit_rate,measured_accesses\n"]
    for p in points:
        out.append(f"{repr(p.capacity_fraction)},{p.predictor_kind},"
                   f"{format_rate(p.report.cache_hit_rate)},"
                   f"{format_rate(p.report.prediction_hit_rate)},"
                   f"{p.report.measured_accesses}\n")
    return "".join(out).encode("utf-8")


def sweep_layers_csv(points) -> bytes:
    out = ["capacity_fraction,predictor,layer_id,measured_accesses,"
           "cache_hits,cache_hit_rate,prediction_hits,prediction_hit_rate\n"]
    for p in points:
        r = p.report
        for layer in range(r.shape.num_layers):
            acc, ch = int(r.layer_accesses[layer]), int(r.layer_cache_hits[layer])
            ph = int(r.layer_prediction_hits[layer])
            out.append(f"{repr(p.capacity_fraction)},{p.predictor_kind},{layer},"
                       f"{acc},{ch},{format_rate(_rate(ch, acc))},"
                       f"{ph},{format_rate(_rate(ph, acc))}\n")
    return "".join(out).encode("utf-8")


def report_summary_csv(report: SimReport, predictor_kind: str, capacity_entries: int) -> bytes:
    return ("predictor,capacity_entries,measured_accesses,cache_hits,"
            "cache_hit_rate,prediction_opportunities,prediction_hits,"
            "prediction_hit_rate,uncovered_queries\n"
            f"{predictor_kind},{capacity_entries},{report.measured_accesses},"
            f"{report.cache_hits},{format_rate(report.cache_hit_rate)},"
            f"{report.prediction_opportunities},{report.prediction_hits},"
            f"{format_rate(report.prediction_hit_rate)},{report.uncovered_queries}\n"
            ).encode("utf-8")


def report_layers_csv(report: SimReport) -> bytes:
    out = ["layer_id,measured_accesses,cache_hits,cache_hit_rate,"
           "prediction_hits,prediction_hit_rate\n"]
    for layer in range(report.shape.num_layers):
        acc, ch = int(report.layer_accesses[layer]), int(report.layer_cache_hits[layer])
        ph = int(report.layer_prediction_hits[layer])
        out.append(f"{layer},{acc},{ch},{format_rate(_rate(ch, acc))},"
                   f"{ph},{format_rate(_rate(ph, acc))}\n")
    return "".join(out).encode("utf-8")


def report_prompts_csv(report: SimReport) -> bytes:
    out = ["prompt_id,measured_accesses,cache_hits,cache_hit_rate,"
           "prediction_hits,prediction_hit_rate\n"]
    for pid in sorted(report.per_prompt):
        c = report.per_prompt[pid]
        out.append(f"{pid},{c.measured_accesses},{c.cache_hits},"
                   f"{format_rate(_rate(c.cache_hits, c.measured_accesses))},"
                   f"{c.prediction_hits},"
                   f"{format_rate(_rate(c.prediction_hits, c.prediction_opportunities))}\n")
    return "".join(out).encode("utf-8")
