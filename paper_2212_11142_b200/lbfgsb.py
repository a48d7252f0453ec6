"""Several L-BFGS-B minimisations stepped in lockstep with one batched objective call per step.

`scipy.optimize.minimize(fun, x0, jac=True, method="L-BFGS-B", bounds=..., options=...)` is a
Python loop around the compiled reverse-communication routine `_lbfgsb.setulb`: the routine asks
for f and g at its current x (task 3), announces a new iterate (task 1) or stops.  The objective
sits behind `ScalarFunction` (one evaluation at x0 up front, re-evaluation only when x changes).
This module drives k such state machines - each with its own x, workspace and counters, stepped
exactly as `_minimize_lbfgsb` steps it (scipy 1.18: `scipy/optimize/_lbfgsb_py.py`) - until every
one of them waits for an objective value, then evaluates all of those points in ONE call.  A
machine's iterates depend only on its own values, so each result equals the one `minimize` returns
for that start on its own (the tests compare x and fun bit for bit), while the objective runs as
one batched GPU call per step and no Python threads are involved.
"""
from __future__ import annotations

import numpy as np

try:  # scipy's compiled routine and the integer width it was built with (scipy >= 1.15 layout)
    from scipy.optimize import _lbfgsb
    from scipy.optimize._lbfgsb_py import HAS_ILP64
except ImportError:  # another scipy layout: the restarts run through minimize() one by one
    _lbfgsb = None
    HAS_ILP64 = False


class _Machine:
    def __init__(self, x0, lo, hi, maxcor, ftol, gtol, maxiter, maxfun, maxls):
        n = x0.shape[0]
        it = np.int64 if HAS_ILP64 else np.int32
        self.m, self.maxiter, self.maxfun, self.maxls = maxcor, maxiter, maxfun, maxls
        self.factr = ftol / np.finfo(float).eps
        self.pgtol = gtol
        self.low = np.zeros(n, np.float64)
        self.up = np.zeros(n, np.float64)
        self.nbd = np.zeros(n, it)
        bmap = {(-np.inf, np.inf): 0, (1, np.inf): 1, (1, 1): 2, (-np.inf, 1): 3}
        for i in range(n):  # _minimize_lbfgsb's bound coding
            L, U = lo[i], hi[i]
            if not np.isinf(L):
                self.low[i] = L
                L = 1
            if not np.isinf(U):
                self.up[i] = U
                U = 1
            self.nbd[i] = bmap[L, U]
        self.x = np.array(np.clip(x0, lo, hi), dtype=np.float64)
        self.f = np.array(0.0, dtype=np.float64)
        self.g = np.zeros(n, np.float64)
        self.wa = np.zeros(2 * maxcor * n + 5 * n + 11 * maxcor * maxcor + 8 * maxcor, np.float64)
        self.iwa = np.zeros(3 * n, it)
        self.task = np.zeros(2, it)
        self.ln_task = np.zeros(2, it)
        self.lsave = np.zeros(4, it)
        self.isave = np.zeros(44, it)
        self.dsave = np.zeros(29, np.float64)
        self.nit = 0
        self.nfev = 0
        self.last_x = None  # ScalarFunction's memo
        self.last_f = None
        self.last_g = None
        self.done = False

    def take(self, f, g):
        """The objective value at self.want (ScalarFunction's evaluation + memo)."""
        self.nfev += 1
        self.last_x, self.last_f, self.last_g = self.want, f, np.atleast_1d(np.asarray(g, dtype=np.float64))
        self.f, self.g = self.last_f, self.last_g

    def advance(self):
        """Step setulb until it needs f, g at a new point (returns True, self.want set) or stops."""
        while True:
            self.g = self.g.astype(np.float64)
            _lbfgsb.setulb(self.m, self.x, self.low, self.up, self.nbd, self.f, self.g, self.factr, self.pgtol,
                           self.wa, self.iwa, self.task, self.lsave, self.isave, self.dsave, self.maxls,
                           self.ln_task)
            if self.task[0] == 3:
                if self.last_x is not None and np.array_equal(self.x, self.last_x):
                    self.f, self.g = self.last_f, self.last_g
                    continue
                self.want = self.x.copy()
                return True
            if self.task[0] == 1:
                self.nit += 1
                if self.nit >= self.maxiter:
                    self.task[0], self.task[1] = 5, 504
                elif self.nfev > self.maxfun:
                    self.task[0], self.task[1] = 5, 502
                continue
            self.done = True
            return False


def minimize_lockstep(evaluate, x0s, bounds, maxiter: int, ftol: float, gtol: float = 1e-5, maxcor: int = 10,
                      maxfun: int = 15000, maxls: int = 20):
    """Minimise from every start in x0s; evaluate(X (k, n)) -> [(f, g)] for k points at a time.
    Returns [(x, fun)] per start (what `minimize(...).x / .fun` would give) and the number of
    evaluate calls."""
    if _lbfgsb is None:
        from scipy.optimize import minimize
        res = [minimize(lambda th: evaluate(th[None, :])[0], x0, jac=True, method="L-BFGS-B", bounds=bounds,
                        options={"maxiter": maxiter, "ftol": ftol, "gtol": gtol, "maxcor": maxcor, "maxfun": maxfun,
                                 "maxls": maxls}) for x0 in x0s]
        return [(r.x, r.fun) for r in res], sum(r.nfev for r in res)
    lo = np.asarray([b[0] for b in bounds], dtype=np.float64)
    hi = np.asarray([b[1] for b in bounds], dtype=np.float64)
    ms = [_Machine(np.asarray(x, dtype=np.float64).ravel(), lo, hi, maxcor, ftol, gtol, maxiter, maxfun, maxls)
          for x in x0s]
    for mc in ms:  # ScalarFunction evaluates at the (clipped) start before the first setulb call
        mc.want = mc.x.copy()
    calls = 0
    pending = list(ms)
    while pending:
        out = evaluate(np.stack([mc.want for mc in pending]))
        calls += 1
        for mc, (f, g) in zip(pending, out):
            mc.take(f, g)
        pending = [mc for mc in pending if mc.advance()]
    return [(mc.x, mc.f) for mc in ms], calls
