"""lbfgsb.minimize_lockstep against scipy.optimize.minimize(method="L-BFGS-B") - the reference's
hyperparameter refinement (surrogate.py:510-530) - on the reference's own objective: the same x and
fun bit for bit for every start (host code, CPU)."""
import math

import numpy as np
import pytest
from scipy.optimize import minimize

from paper_2212_11142_b200 import scenarios
from paper_2212_11142_b200.lbfgsb import minimize_lockstep

pytestmark = pytest.mark.reference


@pytest.mark.parametrize("case,n", [("C5", 12), ("C5", 30), ("C3", 25), ("C2", 8)])
def test_lockstep_restarts_equal_sequential_minimize(case, n):
    from golden_io import ref
    bt = ref()
    S = bt.surrogate
    space = scenarios.build_space(case, bt.space)
    rng = np.random.default_rng(n)
    cfgs = list(dict.fromkeys(bt.space.sample_uniform(space, n + 10, rng)))[:n]
    y = np.array([scenarios.objective(case, c) for c in cfgs])
    z, _, _ = S._standardize(np.log(y) if np.all(y > 0) else y)
    sq = S.pairwise_sq_distances(space, cfgs, cfgs, True)
    prior = S.LengthscalePrior()
    lo, hi = S._search_boxes(space.dimension, prior)
    thetas = rng.uniform(lo, hi, size=(8, 2 + space.dimension))
    thetas[0] = hi + 1.0  # a start outside the box: clipped as minimize clips it

    def objective(theta):
        try:
            value, grad = S._lml_core(sq, z, math.exp(theta[0]), math.exp(theta[1]), np.exp(theta[2:]),
                                      want_grad=True, prior=prior)
        except np.linalg.LinAlgError:
            return np.inf, np.zeros_like(theta)
        return -value, -grad

    bounds = list(zip(lo, hi))
    want = [minimize(objective, th, jac=True, method="L-BFGS-B", bounds=bounds,
                     options={"maxiter": S.MAX_OPT_ITERS, "ftol": S.OPT_TOL}) for th in thetas]
    got, calls = minimize_lockstep(lambda X: [objective(x) for x in X], thetas, bounds, S.MAX_OPT_ITERS, S.OPT_TOL)
    for w, (x, fun) in zip(want, got):
        assert np.array_equal(w.x, x) and w.fun == fun
    assert calls == max(w.nfev for w in want)  # one batched call per lockstep round
