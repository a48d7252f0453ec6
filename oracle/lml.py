"""Batched coarse log marginal likelihood restated (surrogate.py:420-466).  Test-only."""
from __future__ import annotations

import math

import numpy as np

from .gp import matern


def coarse_lml(sq, z, thetas) -> np.ndarray:
    """LML of each hyperparameter row (log sigma, log noise, log l_1..l_D); -inf when the Gram
    is not positive definite."""
    sq, z, thetas = np.asarray(sq, float), np.asarray(z, float), np.asarray(thetas, float)
    n = len(z)
    out = np.full(len(thetas), -np.inf)
    for c, th in enumerate(thetas):
        sigma = math.exp(th[0])
        noise = max(math.exp(th[1]), 1e-6)
        W = np.tensordot(np.exp(-2.0 * th[2:]), sq, axes=(0, 0))
        d = np.sqrt(np.maximum(W, 0.0))
        K = sigma * (1.0 + math.sqrt(5.0) * d + (5.0 / 3.0) * W) * np.exp(-math.sqrt(5.0) * d)
        K[np.arange(n), np.arange(n)] += noise + 1e-9
        try:
            L = np.linalg.cholesky(K)
        except np.linalg.LinAlgError:
            continue
        u = np.linalg.solve(L, z)
        out[c] = -0.5 * float(u @ u) - float(np.log(np.diag(L)).sum()) - 0.5 * n * math.log(2 * math.pi)
    return out


def prior_term(thetas, shape=2.0, rate=2.0) -> np.ndarray:
    """Gamma(shape, rate) log density summed over lengthscales (surrogate.py:459-466)."""
    from scipy.special import gammaln

    ls = np.exp(np.asarray(thetas, float)[:, 2:])
    return (shape * math.log(rate) + (shape - 1.0) * np.log(ls) - rate * ls - float(gammaln(shape))).sum(1)


def lml_core(sq, z, sigma, noise, lengthscales, want_grad=False, prior=(2.0, 2.0)):
    """Log marginal posterior and gradient w.r.t. (log sigma, log noise, log l_i)
    (surrogate.py:356-400); prior = (shape, rate) of the Gamma lengthscale prior or None.
    Raises numpy.linalg.LinAlgError when the Gram matrix is not positive definite."""
    from scipy.special import gammaln

    sq, z = np.asarray(sq, float), np.asarray(z, float)
    ls = np.asarray(lengthscales, float)
    n = len(z)
    noise = max(float(noise), 1e-6)
    W = np.tensordot(1.0 / ls ** 2, sq, axes=(0, 0))
    d = np.sqrt(np.maximum(W, 0.0))
    E = np.exp(-math.sqrt(5.0) * d)
    K = sigma * ((1.0 + math.sqrt(5.0) * d + (5.0 / 3.0) * W) * E)
    L = np.linalg.cholesky(K + (noise + 1e-9) * np.eye(n))
    Linv = np.linalg.inv(L)
    alpha = Linv.T @ (Linv @ z)
    value = -0.5 * float(z @ alpha) - float(np.log(np.diag(L)).sum()) - 0.5 * n * math.log(2 * math.pi)
    if prior is not None:
        k, rate = prior
        value += float(len(ls) * (k * math.log(rate) - gammaln(k)) + (k - 1.0) * np.log(ls).sum()
                       - rate * ls.sum())
    if not want_grad:
        return value
    M = np.outer(alpha, alpha) - Linv.T @ Linv
    grad = np.empty(2 + len(ls))
    grad[0] = 0.5 * float((M * K).sum())
    grad[1] = 0.5 * noise * float(np.trace(M))
    MG = M * ((1.0 + math.sqrt(5.0) * d) * E)
    for i, l in enumerate(ls):
        grad[2 + i] = (5.0 / 6.0) * sigma / (l * l) * float((MG * sq[i]).sum())
        if prior is not None:
            grad[2 + i] += (prior[0] - 1.0) - prior[1] * l
    return value, grad
