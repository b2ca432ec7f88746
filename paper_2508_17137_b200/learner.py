"""Linear learned predictor model container (learner.py:22-224 in the reference).

Inference over whole traces is the device kernel moeb_linear_predict
(predictors.LearnedLinearPredictor). Training with epochs > 0 (the reference's
per-example SGD, learner.py:116-155) is the step before this hot path and is
listed as a next component in DESIGN.md; ``train`` here reproduces the
reference's seeded initialisation exactly (epochs = 0 returns it, marked
trained, as the reference does).
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


def train(traces, shape: ModelShape, config: LearnerConfig = LearnerConfig()) -> LinearModel:
    """Seeded model. epochs = 0: the reference's random init, marked trained."""
    if traces is not None and hasattr(traces, "__len__") and len(traces) == 0:
        raise ConfigError("cannot train on an empty trace list")
    if config.epochs > 0:
        raise NotImplementedError(
            "SGD training (learner.py:116-155) is not part of this hot path; "
            "use epochs=0 (seeded init) or load_model() with trained weights")
    return LinearModel(shape, config, init_weights(shape, config.seed), trained=True)


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
