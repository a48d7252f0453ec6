"""`gp_fit` (surrogate.py:478-541) with the L-BFGS-B restarts batched on the GPU (SURVEY.md §8f
rank 2).

The reference refines the N_TOP = 8 best coarse hyperparameter settings one after another, each
scipy L-BFGS-B iteration calling `_lml_core` for ONE setting (~200 calls per fit).  Here the
restarts step in lockstep (`lbfgsb.minimize_lockstep`: scipy's own L-BFGS-B routine, one state
machine per restart, no threads): whenever every still-running restart waits for a value, one
`bx_lml_core` call evaluates all of their settings at once (the whole-GPU pipeline with the
settings side by side on grid.y, so a setting's value and gradient are the ones a single call
gives).  A restart's iterates depend only on its own objective values, so the result equals running
the restarts one after another with the GPU `_lml_core` (`install(lml=True)`).

Everything else is the reference's own code, looked up in the caller's package: the coarse stage
(`_search_boxes`, the RNG draw, `_batched_coarse_lml` - the GPU one when installed - and
`_prior_term`), the stable argsort, the L-BFGS-B bounds / options, the best-value selection in
candidate order and the final `GPModel`.  The pairwise distances come from the bit-exact device
kernel (bx_pairwise_sq).  The objective values are FP64 but not bit-identical to LAPACK's, so the
fitted hyperparameters can differ from the reference's in the last bits (the tests bound it).
"""
from __future__ import annotations

import importlib
import math

import numpy as np
import torch

from .device import scorer
from .lbfgsb import minimize_lockstep

_DEFAULT = object()


def _surrogate(space):
    pkg = type(space).__module__.rsplit(".", 1)[0]
    return importlib.import_module(pkg + ".surrogate")


def gp_fit(space, configs, y, rng, prior=_DEFAULT, log_objective="auto", use_transforms: bool = True,
           advanced: bool = True):
    """Drop-in for `gp_fit` (surrogate.py:478-541): same arguments, RNG consumption, errors and
    returned `GPModel` (with `map_value` and `start_values`)."""
    S = _surrogate(space)
    if prior is _DEFAULT:
        prior = S.LengthscalePrior()
    if len(configs) < 2:
        raise S.SurrogateError("need at least 2 feasible records to fit a GP")
    y = np.asarray(y, float)
    if log_objective == "auto":
        log_objective = bool(np.all(y > 0))
    elif log_objective and np.any(y <= 0):
        raise S.SurrogateError("log objective transform requires positive outputs")
    y_model = np.log(y) if log_objective else y
    z, _, _ = S._standardize(y_model)
    sc = scorer()
    dev = f"cuda:{sc.device}"
    lay = sc.set_space(space, use_transforms)
    rows = sc.to_device(lay.encode(list(configs)))
    sq_d = sc.pairwise_sq(rows, rows)                      # bit-exact pairwise_sq_distances
    sq = sq_d.cpu().numpy()

    dim = space.dimension
    lo, hi = S._search_boxes(dim, prior)
    thetas = rng.uniform(lo, hi, size=(S.N_CANDIDATES, 2 + dim))
    scores = S._batched_coarse_lml(sq, z, thetas) + S._prior_term(thetas, prior)
    if not np.any(np.isfinite(scores)):
        raise S.SurrogateError("all hyperparameter candidates failed numerically")
    order = np.argsort(-scores, kind="stable")[:S.N_TOP]

    refined = {}
    if advanced:
        starts = [int(i) for i in order if np.isfinite(scores[i])]
        z_d = torch.as_tensor(np.ascontiguousarray(z, dtype=np.float64), device=dev)

        def evaluate(batch):
            # rows (log sigma, log noise, log l...) -> (sigma, noise, l...) as the reference's
            # objective passes them (surrogate.py:510-516)
            prm = np.array([[math.exp(t[0]), math.exp(t[1]), *np.exp(t[2:])] for t in batch])
            with torch.cuda.device(sc.device):
                value, grad, ok = sc.lml_core_host(sq_d, z_d, prm, prior)
            return [(np.inf, np.zeros(batch.shape[1])) if not k else (-v, -g) for v, g, k in zip(value, grad, ok)]

        results, calls = minimize_lockstep(evaluate, [thetas[i] for i in starts], list(zip(lo, hi)),
                                           S.MAX_OPT_ITERS, S.OPT_TOL)  # surrogate.py:524-526
        refined = dict(zip(starts, results))
        gp_fit.last_batched_calls = calls

    best_theta, best_value = None, -np.inf
    for idx in order:  # surrogate.py:518-531, candidate order
        if not np.isfinite(scores[idx]):
            continue
        theta, value = thetas[idx], scores[idx]
        if advanced:
            x, fun = refined[int(idx)]
            if np.isfinite(fun) and -fun > value:
                theta, value = x, -fun
        if value > best_value:
            best_theta, best_value = theta, value
    if best_theta is None:
        raise S.SurrogateError("all hyperparameter candidates failed numerically")
    h = S.GPHyperparameters(outputscale=float(math.exp(best_theta[0])),
                            noise_variance=float(math.exp(best_theta[1])),
                            lengthscales=tuple(float(v) for v in np.exp(best_theta[2:])))
    model = S.GPModel(space, configs, y, h, log_objective=log_objective, use_transforms=use_transforms)
    model.map_value = float(best_value)
    model.start_values = scores
    return model


gp_fit.last_batched_calls = 0
