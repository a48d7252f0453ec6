"""Standalone model-state containers with the reference's attribute names.

`GPState` carries what `GPModel` (surrogate.py:264-332) exposes - `space, configs, _cho, alpha,
hyperparameters, y_mean, y_std, log_objective, use_transforms, noise, objective_to_model` - so the
device uploader treats it exactly like a reference GPModel.  `GPState.fit` performs the
once-per-iteration setup of GPModel.__init__ (surrogate.py:286-303): optional log, standardise
(population std, sd < 1e-12 -> 1), Gram from the device's bit-exact pairwise distances, noise floor
+ jitter on the diagonal, Cholesky, alpha.  `Forest` mirrors FeasibilityModel's flat arrays.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
from scipy.linalg import cho_factor, cho_solve

SQRT5 = math.sqrt(5.0)
JITTER = 1e-9
NOISE_FLOOR = 1e-6


@dataclass(frozen=True)
class Hyper:
    outputscale: float
    noise_variance: float
    lengthscales: tuple


class GPState:
    def __init__(self, space, configs, hyperparameters, L, alpha, y_mean, y_std, *,
                 log_objective=False, use_transforms=True):
        self.space = space
        self.configs = list(configs)
        self.hyperparameters = hyperparameters
        self._cho = (np.asarray(L, dtype=np.float64), True)
        self.alpha = np.asarray(alpha, dtype=np.float64)
        self.y_mean, self.y_std = float(y_mean), float(y_std)
        self.log_objective = bool(log_objective)
        self.use_transforms = bool(use_transforms)
        self.noise = max(hyperparameters.noise_variance, NOISE_FLOOR)

    def objective_to_model(self, value: float) -> float:
        if self.log_objective:
            if value <= 0:
                raise ValueError("log objective transform requires positive values")
            return math.log(value)
        return float(value)

    @classmethod
    def fit(cls, space, configs, y, hyperparameters, *, log_objective=False, use_transforms=True,
            scorer=None, device=False):
        """GPModel.__init__ numerics with the Gram's squared distances from the device; device=True:
        the Gram, its Cholesky factor and alpha on the device too (bx_gp_factor)."""
        from .device import scorer as _scorer

        sc = scorer or _scorer()
        lay = sc.set_space(space, use_transforms)
        y = np.asarray(y, dtype=np.float64)
        if log_objective:
            y = np.log(y)
        mu = float(np.mean(y))
        sd = float(np.std(y))
        if not np.isfinite(sd) or sd < 1e-12:
            sd = 1.0
        z = (y - mu) / sd
        rows = sc.to_device(lay.encode(configs))
        if device:
            L, alpha = sc.gp_factor(rows, z, hyperparameters.outputscale, hyperparameters.noise_variance,
                                    hyperparameters.lengthscales)
            return cls(space, configs, hyperparameters, L, alpha, mu, sd,
                       log_objective=log_objective, use_transforms=use_transforms)
        sq = sc.pairwise_sq(rows, rows).cpu().numpy()
        inv = 1.0 / np.asarray(hyperparameters.lengthscales, float) ** 2
        W = np.einsum("kab,k->ab", sq, inv)
        d = np.sqrt(np.maximum(W, 0.0))
        K = hyperparameters.outputscale * ((1.0 + SQRT5 * d + (5.0 / 3.0) * d * d) * np.exp(-SQRT5 * d))
        K[np.diag_indices_from(K)] += max(hyperparameters.noise_variance, NOISE_FLOOR) + JITTER
        c, low = cho_factor(K, lower=True)
        alpha = cho_solve((c, low), z)
        return cls(space, configs, hyperparameters, np.tril(c), alpha, mu, sd,
                   log_objective=log_objective, use_transforms=use_transforms)


@dataclass
class Forest:
    """FeasibilityModel flat arrays (feasibility.py:54-71)."""

    n_trees: int
    max_depth: int
    feature: np.ndarray = None
    threshold: np.ndarray = None
    left: np.ndarray = None
    right: np.ndarray = None
    value: np.ndarray = None
    roots: np.ndarray = None
    constant: float | None = None
    space: object = None
    use_transforms: bool = True
