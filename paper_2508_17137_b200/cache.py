"""Cache configuration and the per-call ExpertCache API (cache.py:22-154).

The product path replays whole traces in one kernel (engine.replay_traces ->
moeb_cache_sim). ``ExpertCache`` keeps the reference's per-call interface for
compatibility and known-answer tests: every call is executed on the device
by ``moeb_cache_ops`` (the same LRU/LFU state machines the trace kernel
uses), replaying the recorded op log; it is O(n) per call and meant for
small interactive use, not bulk simulation.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _native as nat
from .core import ConfigError, ModelShape, RangeError

POLICIES = {"lru": 0, "lfu": 1}


@dataclass(frozen=True)
class CacheConfig:
    """Exactly one of a capacity fraction or an entry count (cache.py:22-55)."""

    capacity_fraction: float | None = None
    capacity_entries: int | None = None
    prefetch_budget: int = 6

    def __post_init__(self):
        if (self.capacity_fraction is None) == (self.capacity_entries is None):
            raise ConfigError("exactly one of capacity_fraction or capacity_entries must be set")
        if self.capacity_fraction is not None and not 0.0 < self.capacity_fraction <= 1.0:
            raise ConfigError(f"capacity_fraction must be in (0, 1], got {self.capacity_fraction}")
        if self.capacity_entries is not None and self.capacity_entries < 1:
            raise ConfigError(f"capacity_entries must be >= 1, got {self.capacity_entries}")
        if self.prefetch_budget < 1:
            raise ConfigError(f"prefetch_budget must be >= 1, got {self.prefetch_budget}")

    def resolve_capacity(self, shape: ModelShape) -> int:
        """max(1, floor(fraction * L * E)) with the reference's float product."""
        if self.capacity_entries is not None:
            return self.capacity_entries
        return max(1, int(self.capacity_fraction * shape.total_experts))


def cache_ops(ops, keys, shape: ModelShape, capacity: int, policy: str = "lru",
              device=None) -> np.ndarray:
    """Run an op stream (0 begin_step, 1 touch, 2 prefetch) on one device cache.

    Returns per-op results (touch hit / prefetch inserted) as uint8.
    """
    if capacity < 1:
        raise ConfigError(f"capacity must be >= 1, got {capacity}")
    ops = np.ascontiguousarray(ops, dtype=np.int32)
    keys = np.ascontiguousarray(keys, dtype=np.int32)
    n = len(ops)
    dev = torch.device("cuda") if device is None else torch.device(device)
    res = torch.zeros(max(n, 1), dtype=torch.uint8, device=dev)
    if n:
        o = torch.from_numpy(ops).to(dev)
        k = torch.from_numpy(keys).to(dev)
        nat.call("moeb_cache_ops", nat.ptr(o), nat.ptr(k), n, shape.num_layers,
                 shape.num_experts, int(capacity), POLICIES[policy], nat.ptr(res),
                 nat.stream_ptr())
    return res[:n].cpu().numpy()


class ExpertCache:
    """Per-call ExpertCache API over the device state machine (cache.py:58-154)."""

    def __init__(self, capacity: int, shape: ModelShape, policy: str = "lru"):
        if capacity < 1:
            raise ConfigError(f"capacity must be >= 1, got {capacity}")
        self.capacity = capacity
        self.shape = shape
        self.policy = policy
        self._ops: list[int] = []
        self._keys: list[int] = []

    def _check(self, key) -> int:
        layer, expert = key
        if not 0 <= layer < self.shape.num_layers:
            raise RangeError(f"layer {layer} out of range [0, {self.shape.num_layers})")
        if not 0 <= expert < self.shape.num_experts:
            raise RangeError(f"expert {expert} out of range [0, {self.shape.num_experts})")
        return layer * self.shape.num_experts + expert

    def _run(self) -> np.ndarray:
        return cache_ops(self._ops, self._keys, self.shape, self.capacity, self.policy)

    def begin_step(self) -> None:
        self._ops.append(0)
        self._keys.append(0)

    def touch(self, key) -> bool:
        k = self._check(key)
        self._ops.append(1)
        self._keys.append(k)
        return bool(self._run()[-1])

    def prefetch(self, keys, limit: int | None = None) -> int:
        keys = list(keys)
        if limit is None:
            limit = len(keys)
        ks = [self._check(k) for k in keys[:limit]]
        for k in ks:
            self._ops.append(2)
            self._keys.append(k)
        if not ks:
            return 0
        return int(self._run()[-len(ks):].sum())
