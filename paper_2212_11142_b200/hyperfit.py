"""`gp_fit` (surrogate.py:478-541) with the L-BFGS-B restarts batched on the GPU (SURVEY.md §8f
rank 2).

The reference refines the N_TOP = 8 best coarse hyperparameter settings one after another, each
scipy L-BFGS-B iteration calling `_lml_core` for ONE setting (~200 calls per fit).  Here the
restarts run concurrently - one scipy optimizer per thread - and their objective requests are
gathered: whenever every still-running optimizer is waiting for a value, one `bx_lml_core` call
evaluates all of their settings at once (the whole-GPU pipeline with the settings side by side on
grid.y, so a setting's value and gradient are the ones a single call gives).  An optimizer's
iterates depend only on its own objective values, so the result equals running the restarts one
after another with the GPU `_lml_core` (`install(lml=True)`), whatever the thread timing.

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
import threading

import numpy as np
import torch

from .device import scorer

_DEFAULT = object()


def _surrogate(space):
    pkg = type(space).__module__.rsplit(".", 1)[0]
    return importlib.import_module(pkg + ".surrogate")


class _Batcher:
    """Gathers objective requests of concurrent optimizers; evaluates a batch when every active
    optimizer is waiting."""

    def __init__(self, n_active: int, evaluate):
        self.cv = threading.Condition()
        self.pending: dict = {}
        self.results: dict = {}
        self.active = n_active
        self.evaluate = evaluate
        self.calls = 0
        self.error = None

    def _maybe_run(self):
        if self.pending and len(self.pending) == self.active:
            ids = sorted(self.pending)
            try:
                out = self.evaluate(np.stack([self.pending[i] for i in ids]))
                for i, r in zip(ids, out):
                    self.results[i] = r
            except BaseException as exc:  # surface it in every waiting thread
                self.error = exc
                for i in ids:
                    self.results[i] = None
            self.calls += 1
            self.pending.clear()
            self.cv.notify_all()

    def request(self, tid: int, theta: np.ndarray):
        with self.cv:
            self.pending[tid] = np.array(theta, dtype=np.float64)
            self._maybe_run()
            while tid not in self.results:
                self.cv.wait()
            r = self.results.pop(tid)
        if r is None:
            raise RuntimeError("batched objective failed") from self.error
        return r

    def done(self):
        with self.cv:
            self.active -= 1
            self._maybe_run()


def gp_fit(space, configs, y, rng, prior=_DEFAULT, log_objective="auto", use_transforms: bool = True,
           advanced: bool = True):
    """Drop-in for `gp_fit` (surrogate.py:478-541): same arguments, RNG consumption, errors and
    returned `GPModel` (with `map_value` and `start_values`)."""
    from scipy.optimize import minimize

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
                value, grad, ok = sc.lml_core(sq_d, z_d, torch.as_tensor(prm, device=dev), True, prior)
                value, grad, ok = value.cpu().numpy(), grad.cpu().numpy(), ok.cpu().numpy()
            return [(np.inf, np.zeros(batch.shape[1])) if not k else (-v, -g) for v, g, k in zip(value, grad, ok)]

        batcher = _Batcher(len(starts), evaluate)
        bounds = list(zip(lo, hi))

        def run(tid, idx):
            try:
                refined[idx] = minimize(lambda th: batcher.request(tid, th), thetas[idx], jac=True,
                                        method="L-BFGS-B", bounds=bounds,
                                        options={"maxiter": S.MAX_OPT_ITERS, "ftol": S.OPT_TOL})
            except BaseException as exc:
                refined[idx] = exc
            finally:
                batcher.done()

        threads = [threading.Thread(target=run, args=(t, idx), daemon=True) for t, idx in enumerate(starts)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        for r in refined.values():
            if isinstance(r, BaseException):
                raise r
        gp_fit.last_batched_calls = batcher.calls

    best_theta, best_value = None, -np.inf
    for idx in order:  # surrogate.py:518-531, candidate order
        if not np.isfinite(scores[idx]):
            continue
        theta, value = thetas[idx], scores[idx]
        if advanced:
            res = refined[int(idx)]
            if np.isfinite(res.fun) and -res.fun > value:
                theta, value = res.x, -res.fun
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
