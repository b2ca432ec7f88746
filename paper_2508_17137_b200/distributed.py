"""Prompt-sharded replay across GPUs.

Prompts are independent (private cache, rEAM and history per prompt,
engine.py:222-238), so each rank replays a contiguous, row-balanced prompt
range and the only exchange is one SUM all-reduce of the int64 counter
vectors (the analogue of SimReport.merge, engine.py:94-110). Integer sums are
order-independent, so any GPU count gives bit-identical reports. Per-prompt
counters, when requested, are all-gathered (engine.py:75, report_prompts_csv).

With an NCCL group the CUDA counter tensors are reduced in place over NVLink;
with a gloo group (CPU tests) they are staged through host memory.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from .engine import ReplayConfig, SimReport, _check_lengths, cache_replay, predict_stream
from .metrics import MetricCounts, mask_metrics, metric_vector
from .traces import PackedTraces


def _all_reduce_sum(t: torch.Tensor, group=None) -> torch.Tensor:
    if dist.get_backend(group) == "nccl":
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        return t
    host = t.detach().cpu()
    dist.all_reduce(host, op=dist.ReduceOp.SUM, group=group)
    return host.to(t.device)


def combine_reports(shape, counters, per_prompt=None, prompt_ids=None, group=None) -> SimReport:
    """Sum local K1 counter vectors [4+3L] over the group and (optionally)
    gather per-prompt counters [P_local,4] into one SimReport."""
    vec = _all_reduce_sum(torch.as_tensor(counters, dtype=torch.int64).reshape(-1).clone(), group)
    pp_all = ids_all = None
    if per_prompt is not None:
        world = dist.get_world_size(group)
        local = (np.asarray(per_prompt, dtype=np.int64), np.asarray(prompt_ids, dtype=np.int64))
        gathered = [None] * world
        dist.all_gather_object(gathered, local, group=group)
        pp_all = np.concatenate([g[0] for g in gathered])
        ids_all = np.concatenate([g[1] for g in gathered])
    return SimReport.from_counters(shape, vec.cpu().numpy(), pp_all, ids_all)


def combine_metrics(vec, num_experts: int, group=None) -> MetricCounts:
    v = _all_reduce_sum(torch.as_tensor(vec, dtype=torch.int64).reshape(-1).clone(), group)
    return MetricCounts.from_vector(v.cpu().numpy(), num_experts)


def replay_sharded(packed: PackedTraces, predictor, config: ReplayConfig, group=None,
                   policy: str = "lru", per_prompt: bool = False) -> SimReport:
    """replay_traces over all ranks of `group`: this rank's shard on its GPU,
    then one counter all-reduce. `packed` holds every prompt (each rank may
    also pass only its own prompts with `packed.meta['presharded'] = True`)."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    local = packed if packed.meta.get("presharded") else packed.shard(rank, world)
    _check_lengths(local, config.warmup_tokens)
    cap = config.cache.resolve_capacity(config.shape)
    stream = predict_stream(predictor, local, config)
    counters, pp, _ = cache_replay(local, [stream], [cap], config.warmup_tokens,
                                   config.cache.prefetch_budget, policy, per_prompt)
    if world == 1:
        return SimReport.from_counters(config.shape, counters[0, 0].cpu().numpy(),
                                       None if pp is None else pp[0, 0].cpu().numpy(),
                                       local.prompt_ids)
    return combine_reports(config.shape, counters[0, 0],
                           None if pp is None else pp[0, 0].cpu().numpy(),
                           local.prompt_ids, group)


def metrics_sharded(packed: PackedTraces, predictor, config: ReplayConfig,
                    group=None) -> MetricCounts:
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    local = packed if packed.meta.get("presharded") else packed.shard(rank, world)
    E = config.shape.num_experts
    vec = metric_vector(E, local.device)
    masks = predictor.predict_masks(local, config.cache.prefetch_budget, config.warmup_tokens)
    mask_metrics(masks, local.truth, local.row_off, config.shape.num_layers, E,
                 config.warmup_tokens, vec)
    if world == 1:
        return MetricCounts.from_vector(vec.cpu().numpy(), E)
    return combine_metrics(vec, E, group)
