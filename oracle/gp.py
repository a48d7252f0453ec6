"""GP posterior + EI restated (surrogate.py:163-328, acquisition.py:40-79).  Test-only."""
from __future__ import annotations

import math
from itertools import combinations

import numpy as np
from scipy.linalg import solve_triangular
from scipy.special import ndtr

R5 = math.sqrt(5.0)


def coords(p, vals, use_transforms=True) -> np.ndarray:
    """Normalised (optionally log) coordinate of numeric values (surrogate.py:163-170)."""
    if p.kind == "ordinal":
        lo, hi = float(p.values[0]), float(p.values[-1])
    else:
        lo, hi = float(p.lo), float(p.hi)
    x = np.asarray(vals, float)
    if use_transforms and p.transform == "log":
        x, lo, hi = np.log(x), math.log(lo), math.log(hi)
    return np.zeros_like(x) if hi == lo else (x - lo) / (hi - lo)


def _perm_raw(metric, a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Raw permutation semimetric for every pair of rows (surrogate.py:54-72, 201-218)."""
    if metric == "spearman":
        return ((a[:, None, :] - b[None, :, :]) ** 2).sum(-1).astype(float)
    if metric == "hamming":
        return (a[:, None, :] != b[None, :, :]).sum(-1).astype(float)
    if metric == "naive":
        return np.any(a[:, None, :] != b[None, :, :], axis=-1).astype(float)
    m = a.shape[1]
    pairs = list(combinations(range(m), 2))
    oa = np.stack([a[:, i] < a[:, j] for i, j in pairs], 1)
    ob = np.stack([b[:, i] < b[:, j] for i, j in pairs], 1)
    return (oa[:, None, :] != ob[None, :, :]).sum(-1).astype(float)


def _perm_max(metric, m):
    return {"kendall": m * (m - 1) / 2.0, "spearman": m * (m * m - 1) / 3.0,
            "hamming": float(m), "naive": 1.0}[metric]


def pairwise_sq(space, A, B, use_transforms=True) -> np.ndarray:
    """Per-parameter squared distances, shape (D, |A|, |B|) (surrogate.py:173-198)."""
    out = np.empty((len(space.parameters), len(A), len(B)))
    for k, p in enumerate(space.parameters):
        ca = [c[k] for c in A]
        cb = [c[k] for c in B]
        if p.kind in ("real", "integer", "ordinal"):
            d = coords(p, ca, use_transforms)[:, None] - coords(p, cb, use_transforms)[None, :]
            out[k] = d * d
        elif p.kind == "categorical":
            lab = {v: i for i, v in enumerate(p.values)}
            ia = np.array([lab[v] for v in ca])
            ib = np.array([lab[v] for v in cb])
            out[k] = (ia[:, None] != ib[None, :]).astype(float)
        else:
            a = np.asarray(ca, int).reshape(len(A), p.size)
            b = np.asarray(cb, int).reshape(len(B), p.size)
            out[k] = _perm_raw(p.permutation_metric, a, b) / _perm_max(p.permutation_metric, p.size)
    return out


def matern(d):
    return (1.0 + R5 * d + (5.0 / 3.0) * d * d) * np.exp(-R5 * d)


class OracleGP:
    """GP state: either given (L, alpha from the reference) or fitted (GPModel.__init__ restated,
    surrogate.py:286-303)."""

    def __init__(self, space, configs, outputscale, noise, lengthscales, *, y=None, L=None,
                 alpha=None, y_mean=None, y_std=None, log_objective=False, use_transforms=True):
        self.space, self.configs = space, list(configs)
        self.outputscale, self.lengthscales = float(outputscale), np.asarray(lengthscales, float)
        self.noise = max(float(noise), 1e-6)
        self.log_objective, self.use_transforms = bool(log_objective), bool(use_transforms)
        if L is None:
            yy = np.log(np.asarray(y, float)) if log_objective else np.asarray(y, float)
            mu, sd = float(yy.mean()), float(yy.std())
            sd = 1.0 if (not np.isfinite(sd) or sd < 1e-12) else sd
            z = (yy - mu) / sd
            K = self.kernel(self.configs, self.configs)
            K[np.arange(len(K)), np.arange(len(K))] += self.noise + 1e-9
            L = np.linalg.cholesky(K)
            alpha = solve_triangular(L.T, solve_triangular(L, z, lower=True), lower=False)
            y_mean, y_std = mu, sd
        self.L, self.alpha = np.tril(np.asarray(L, float)), np.asarray(alpha, float)
        self.y_mean, self.y_std = float(y_mean), float(y_std)

    def kernel(self, A, B):
        W = np.tensordot(1.0 / self.lengthscales ** 2, pairwise_sq(self.space, A, B, self.use_transforms),
                         axes=(0, 0))
        return self.outputscale * matern(np.sqrt(np.maximum(W, 0.0)))

    def to_model(self, value):
        return math.log(value) if self.log_objective else float(value)


def predict(gp: OracleGP, configs):
    """Noise-free posterior mean / variance, de-standardised (surrogate.py:315-328)."""
    ks = gp.kernel(list(configs), gp.configs)
    mean = ks @ gp.alpha
    v = solve_triangular(gp.L, ks.T, lower=True)
    var = np.maximum(gp.outputscale - (v * v).sum(0), 0.0)
    return gp.y_mean + gp.y_std * mean, gp.y_std ** 2 * var


def expected_improvement(mean, var, f_best):
    """Closed-form EI for minimisation (acquisition.py:40-51)."""
    mean = np.asarray(mean, float)
    s = np.sqrt(np.maximum(np.asarray(var, float), 0.0))
    delta = f_best - mean
    out = np.maximum(delta, 0.0)
    pos = s > 0
    z = delta[pos] / s[pos]
    out[pos] = delta[pos] * ndtr(z) + s[pos] * (np.exp(-0.5 * z * z) / math.sqrt(2 * math.pi))
    return np.maximum(out, 0.0)


def scores(gp: OracleGP, forest, configs, f_best, eps_f=0.0):
    """(values, probs) of a batch (acquisition.py:70-79)."""
    configs = list(configs)
    mean, var = predict(gp, configs)
    ei = expected_improvement(mean, var, gp.to_model(f_best))
    if forest is None:
        return ei, np.ones(len(configs))
    from .forest import predict_proba
    p = predict_proba(forest, configs)
    return np.where(p < eps_f, -np.inf, ei * p), p
