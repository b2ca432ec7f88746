"""Prediction-quality metrics (metrics.py:12-79 in the reference).

The device kernel K7 (moeb_metrics, or fused into moeb_linear_predict)
produces the integer core -- per-expert TP/FP/FN, positions, exact-set
matches, label-correct -- and ``MetricCounts`` finishes with the reference's
own numpy expressions, so the floats are identical given identical masks.
The set-based functions keep the reference signatures.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _native as nat
from .core import DimensionError


@dataclass
class MetricCounts:
    num_experts: int
    tp: np.ndarray
    fp: np.ndarray
    fn: np.ndarray
    positions: int
    exact: int
    label_correct: int

    @classmethod
    def from_vector(cls, vec, num_experts: int) -> "MetricCounts":
        v = np.asarray(vec.cpu() if isinstance(vec, torch.Tensor) else vec, dtype=np.int64)
        E = num_experts
        return cls(E, v[:E].copy(), v[E:2 * E].copy(), v[2 * E:3 * E].copy(), int(v[3 * E]),
                   int(v[3 * E + 1]), int(v[3 * E + 2]))

    def macro_f1(self, include_all: bool = False) -> float:
        tp, fp, fn = self.tp, self.fp, self.fn
        support = tp + fp + fn
        with np.errstate(invalid="ignore"):
            f1 = np.where(support > 0, 2.0 * tp / np.maximum(2 * tp + fp + fn, 1), 0.0)
        if include_all:
            return float(f1.mean()) if self.num_experts else 0.0
        included = support > 0
        if not included.any():
            return 0.0
        return float(f1[included].mean())

    @property
    def position_accuracy(self) -> float:
        return self.exact / self.positions if self.positions else 0.0

    @property
    def label_accuracy(self) -> float:
        return self.label_correct / (self.positions * self.num_experts) if self.positions else 0.0


def metric_vector(num_experts: int, device) -> torch.Tensor:
    return torch.zeros(3 * num_experts + 3, dtype=torch.int64, device=device)


def mask_metrics(pred: torch.Tensor, truth: torch.Tensor, row_off: torch.Tensor, L: int, E: int,
                 warmup: int, out: torch.Tensor | None = None) -> torch.Tensor:
    """K7 over CSR-packed masks; accumulates into (and returns) the int64 vector."""
    if out is None:
        out = metric_vector(E, pred.device)
    nat.call("moeb_metrics", nat.ptr(pred), nat.ptr(truth), nat.ptr(row_off),
             row_off.shape[0] - 1, L, E, int(warmup), nat.ptr(out), nat.stream_ptr())
    return out


def _sets_counts(pred_sets, truth_sets, num_experts: int) -> MetricCounts:
    if len(pred_sets) != len(truth_sets):
        raise DimensionError(f"{len(pred_sets)} predictions vs {len(truth_sets)} truths")
    n = len(truth_sets)
    W = (num_experts + 63) // 64
    pm = np.zeros((max(n, 1), W), dtype=np.uint64)
    tm = np.zeros((max(n, 1), W), dtype=np.uint64)
    for i, (p, t) in enumerate(zip(pred_sets, truth_sets)):
        for e in p:
            pm[i, e >> 6] |= np.uint64(1) << np.uint64(e & 63)
        for e in t:
            tm[i, e >> 6] |= np.uint64(1) << np.uint64(e & 63)
    dev = torch.device("cuda")
    P = torch.from_numpy(pm.view(np.int64)).to(dev)
    T = torch.from_numpy(tm.view(np.int64)).to(dev)
    off = torch.tensor([0, n], dtype=torch.int64, device=dev)
    vec = mask_metrics(P, T, off, 1, num_experts, 0)
    return MetricCounts.from_vector(vec, num_experts)


def position_accuracy(pred_sets, truth_sets) -> float:
    if len(pred_sets) != len(truth_sets):
        raise DimensionError(f"{len(pred_sets)} predictions vs {len(truth_sets)} truths")
    if not truth_sets:
        return 0.0
    E = 1 + max([max(s) for s in list(pred_sets) + list(truth_sets) if s] or [0])
    return _sets_counts(pred_sets, truth_sets, E).position_accuracy


def macro_f1(pred_sets, truth_sets, num_experts: int, include_all: bool = False) -> float:
    return _sets_counts(pred_sets, truth_sets, num_experts).macro_f1(include_all)


def label_accuracy(pred_sets, truth_sets, num_experts: int) -> float:
    if len(pred_sets) != len(truth_sets):
        raise DimensionError(f"{len(pred_sets)} predictions vs {len(truth_sets)} truths")
    if not truth_sets:
        return 0.0
    return _sets_counts(pred_sets, truth_sets, num_experts).label_accuracy


@dataclass
class ActivationReport:
    """Exact activation counts per (layer, expert) plus per-prompt sparsity
    (metrics.py:80-92)."""

    layer_expert_counts: np.ndarray
    prompt_ids: list[int]
    prompt_layer_distinct: np.ndarray

    @property
    def total_activations(self) -> int:
        return int(self.layer_expert_counts.sum())


def activation_report(traces, shape) -> ActivationReport:
    """metrics.activation_report (metrics.py:95-119) from the per-prompt
    activation counts K8 (moeb_ream_counts) computes on device: layer totals
    are their sum over prompts, distinct counts their per-layer support."""
    from .sketches import ream_counts
    from .traces import PackedTraces, pack_traces

    packed = traces if isinstance(traces, PackedTraces) else pack_traces(traces, shape)
    L, E = shape.num_layers, shape.num_experts
    if packed.num_prompts == 0:
        return ActivationReport(np.zeros((L, E), dtype=np.int64), [],
                                np.zeros((0, L), dtype=np.int64))
    counts = ream_counts(packed).view(packed.num_prompts, L, E)
    totals = counts.sum(dim=0, dtype=torch.int64).cpu().numpy()
    distinct = (counts > 0).sum(dim=2, dtype=torch.int64).cpu().numpy()
    return ActivationReport(totals, [int(p) for p in packed.prompt_ids], distinct)


def activation_report_csv(report: ActivationReport) -> bytes:
    """metrics.activation_report_csv (metrics.py:122-128)."""
    lines = ["layer_id,expert_id,count"]
    counts = report.layer_expert_counts
    for layer in range(counts.shape[0]):
        for expert in range(counts.shape[1]):
            lines.append(f"{layer},{expert},{counts[layer, expert]}")
    return ("\n".join(lines) + "\n").encode("utf-8")


def distinct_report_csv(report: ActivationReport) -> bytes:
    """metrics.distinct_report_csv (metrics.py:131-136)."""
    lines = ["prompt_id,layer_id,distinct_experts"]
    for row, pid in enumerate(report.prompt_ids):
        for layer in range(report.prompt_layer_distinct.shape[1]):
            lines.append(f"{pid},{layer},{report.prompt_layer_distinct[row, layer]}")
    return ("\n".join(lines) + "\n").encode("utf-8")
