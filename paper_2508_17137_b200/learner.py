"""Linear learned predictor model container (learner.py:22-224 in the reference).

Inference over whole traces is the device kernel moeb_linear_predict
(predictors.LearnedLinearPredictor); training (the reference's per-example
SGD, learner.py:116-155) runs as moeb_linear_features + one
moeb_linear_sgd_epoch launch per epoch (csrc/learner.cu).
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field

import numpy as np

from .core import ConfigError, ModelShape


@dataclass(frozen=True)
class LearnerConfig:
    learning_rate: float = 0.05
    epochs: int = 10
    decay: float = 0.9
    seed: int = 0

    def __post_init__(self):
        if self.learning_rate <= 0:
            raise ConfigError(f"learning_rate must be > 0, got {self.learning_rate}")
        if self.epochs < 0:
            raise ConfigError(f"epochs must be >= 0, got {self.epochs}")
        if not 0.0 <= self.decay < 1.0:
            raise ConfigError(f"decay must be in [0, 1), got {self.decay}")


@dataclass
class LinearModel:
    """Weights [E][L+E+1] over [layer one-hot | decayed history | bias]."""

    shape: ModelShape
    config: LearnerConfig
    weights: np.ndarray
    trained: bool = False
    loss_history: list[float] = field(default_factory=list)

    @property
    def feature_len(self) -> int:
        return self.shape.num_layers + self.shape.num_experts + 1


def init_weights(shape: ModelShape, seed: int) -> np.ndarray:
    """The reference's initialisation: default_rng(seed).normal(0, 0.01, (E, L+E+1))
    (learner.py:128-129)."""
    rng = np.random.default_rng(seed)
    return rng.normal(0.0, 0.01, size=(shape.num_experts, shape.num_layers + shape.num_experts + 1))


_EARLY_STOP_DELTA = 1e-5
_EARLY_STOP_PATIENCE = 3


def train(traces, shape: ModelShape, config: LearnerConfig = LearnerConfig()) -> LinearModel:
    """learner.train (learner.py:116-155): per-example SGD over seeded-shuffled
    (token, layer) steps with patience-3 early stop, on device.

    The features (decayed histories, bit-identical to training_pairs) come
    from moeb_linear_features; each epoch is one moeb_linear_sgd_epoch launch
    in the permutation the reference's rng draws (same seed, same call
    sequence: normal() init, then permutation() per epoch). epochs = 0
    returns the seeded initialisation, marked trained."""
    import torch

    from . import _native as nat
    from .traces import PackedTraces, pack_traces

    if traces is not None and hasattr(traces, "__len__") and len(traces) == 0:
        raise ConfigError("cannot train on an empty trace list")
    if traces is None and config.epochs > 0:  # None: the seeded init only (epochs = 0)
        raise ConfigError("cannot train on an empty trace list")
    rng = np.random.default_rng(config.seed)
    L, E = shape.num_layers, shape.num_experts
    weights = rng.normal(0.0, 0.01, size=(E, L + E + 1))
    if config.epochs == 0:
        return LinearModel(shape, config, weights, trained=True)
    packed = traces if isinstance(traces, PackedTraces) else pack_traces(traces, shape)
    n = packed.rows
    if n == 0:
        raise ConfigError("no training examples: traces are empty")
    dev = packed.device
    hist = torch.empty((n, E), dtype=torch.float64, device=dev)
    nat.call("moeb_linear_features", nat.ptr(packed.truth), nat.ptr(packed.row_off),
             packed.num_prompts, L, E, float(config.decay), nat.ptr(hist), nat.stream_ptr())
    w_d = torch.from_numpy(np.ascontiguousarray(weights)).to(dev)
    loss_d = torch.zeros(1, dtype=torch.float64, device=dev)
    losses: list[float] = []
    best = np.inf
    stalls = 0
    for _ in range(config.epochs):
        order = torch.from_numpy(rng.permutation(n).astype(np.int64)).to(dev)
        nat.call("moeb_linear_sgd_epoch", nat.ptr(w_d), nat.ptr(hist), nat.ptr(packed.truth),
                 nat.ptr(order), n, L, E, float(config.learning_rate), nat.ptr(loss_d),
                 nat.stream_ptr())
        epoch_loss = float(loss_d.item()) / n
        losses.append(epoch_loss)
        if best - epoch_loss < _EARLY_STOP_DELTA:
            stalls += 1
            if stalls >= _EARLY_STOP_PATIENCE:
                break
        else:
            stalls = 0
        best = min(best, epoch_loss)
    return LinearModel(shape, config, w_d.cpu().numpy(), trained=True, loss_history=losses)


def save_model(model: LinearModel, path) -> None:
    payload = {
        "kind": "linear-multilabel",
        "num_layers": model.shape.num_layers,
        "num_experts": model.shape.num_experts,
        "top_k": model.shape.top_k,
        "learning_rate": model.config.learning_rate,
        "epochs": model.config.epochs,
        "decay": model.config.decay,
        "seed": model.config.seed,
        "trained": model.trained,
        "loss_history": list(model.loss_history),
        "weights": [[float(v) for v in row] for row in model.weights],
    }
    with open(path, "w", encoding="utf-8") as fh:
        json.dump(payload, fh)
        fh.write("\n")


def load_model(path) -> LinearModel:
    """Same file format and checks as the reference (learner.py:204-224)."""
    with open(path, encoding="utf-8") as fh:
        payload = json.load(fh)
    try:
        shape = ModelShape(payload["num_layers"], payload["num_experts"], payload["top_k"])
        config = LearnerConfig(payload["learning_rate"], payload["epochs"], payload["decay"],
                               payload["seed"])
        weights = np.asarray(payload["weights"], dtype=np.float64)
        trained = bool(payload["trained"])
        losses = [float(v) for v in payload.get("loss_history", [])]
    except (KeyError, TypeError) as exc:
        raise ConfigError(f"bad model file {path}: {exc}") from None
    expected = (shape.num_experts, shape.num_layers + shape.num_experts + 1)
    if weights.shape != expected:
        raise ConfigError(f"model weights shape {weights.shape} != {expected}")
    if not np.isfinite(weights).all():
        raise ConfigError("model weights must be finite")
    return LinearModel(shape, config, weights, trained, losses)


# Per-vector helpers of the reference's learner (learner.py:52-72, :158-182).
# They score ONE feature vector on the host, exactly as the reference does;
# whole traces go through K3 (moeb_linear_predict), never through these.

def feature_vector(target_layer: int, layer_history: np.ndarray, shape: ModelShape) -> np.ndarray:
    """[layer one-hot | decayed history for the target layer | 1.0] (learner.py:52-59)."""
    f = np.zeros(shape.num_layers + shape.num_experts + 1, dtype=np.float64)
    f[target_layer] = 1.0
    f[shape.num_layers:shape.num_layers + shape.num_experts] = layer_history
    f[-1] = 1.0
    return f


def update_history(history: np.ndarray, layer_id: int, expert_ids, decay: float) -> None:
    """history[layer] = decay * history[layer] + firings (learner.py:62-72)."""
    history[layer_id] *= decay
    for e in expert_ids:
        history[layer_id, e] += 1.0


def predict_scores(model: LinearModel, features: np.ndarray) -> np.ndarray:
    if not model.trained:
        raise ConfigError("model is untrained")
    return model.weights @ features


def top_k_experts(scores: np.ndarray, k: int) -> frozenset[int]:
    """The k highest-scoring experts, ties to the lower id (learner.py:164-169)."""
    k = min(k, len(scores))
    order = np.lexsort((np.arange(len(scores)), -np.asarray(scores)))
    return frozenset(int(e) for e in order[:k])


def predict_topk(model: LinearModel, features: np.ndarray, k: int,
                 threshold: bool = False) -> frozenset[int]:
    """Top-k experts by logit, or logit > 0 in threshold mode (learner.py:172-182)."""
    scores = predict_scores(model, features)
    if threshold:
        return frozenset(int(e) for e in np.nonzero(scores > 0.0)[0])
    return top_k_experts(scores, k)
