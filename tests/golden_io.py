"""Load tests/golden fixtures into this package's host objects and the oracle's objects."""
from __future__ import annotations

import json
from functools import lru_cache
from pathlib import Path

import numpy as np

from paper_2212_11142_b200 import scenarios
from paper_2212_11142_b200.constraints import build_cot
from paper_2212_11142_b200.models import Forest, GPState, Hyper

GOLDEN = Path(__file__).resolve().parent / "golden"
CASES = ["mixed_fit", "mixed_metrics", "C1", "C2", "C3", "C4"]
TRACES = ["trace_quadratic", "trace_ridge", "trace_perm"]


def to_cfg(space, lst):
    return tuple(tuple(v) if p.kind == "permutation" else v for p, v in zip(space.parameters, lst))


class Case:
    def __init__(self, meta, arrays, prefix=""):
        self.meta, self.arrays, self.prefix = meta, arrays, prefix

    def arr(self, key):
        return self.arrays[self.prefix + key]

    def has(self, key):
        return (self.prefix + key) in self.arrays


@lru_cache(maxsize=None)
def load(case: str):
    meta = json.loads((GOLDEN / f"{case}.json").read_text())
    arrays = dict(np.load(GOLDEN / f"{case}.npz"))
    space = scenarios.build_space(meta["space"])
    return meta, arrays, space


def model(meta, arrays, space, prefix=""):
    """(GPState, Forest | None) for a fixture (or one engine-trace iteration)."""
    h = Hyper(meta["outputscale"], meta["noise_variance"], tuple(meta["lengthscales"]))
    train = [to_cfg(space, c) for c in meta["train"]]
    gp = GPState(space, train, h, arrays[prefix + "L"], arrays[prefix + "alpha"], meta["y_mean"],
                 meta["y_std"], log_objective=meta["log_objective"],
                 use_transforms=meta["use_transforms"])
    feas = None
    if prefix + "rf_constant" in arrays:
        feas = Forest(int(arrays[prefix + "rf_n_trees"][0]), int(arrays[prefix + "rf_max_depth"][0]),
                      constant=float(arrays[prefix + "rf_constant"][0]), space=space)
    elif prefix + "rf_feature" in arrays:
        feas = Forest(int(arrays[prefix + "rf_n_trees"][0]), int(arrays[prefix + "rf_max_depth"][0]),
                      feature=arrays[prefix + "rf_feature"], threshold=arrays[prefix + "rf_threshold"],
                      left=arrays[prefix + "rf_left"], right=arrays[prefix + "rf_right"],
                      value=arrays[prefix + "rf_value"], roots=arrays[prefix + "rf_roots"], space=space,
                      use_transforms=meta["use_transforms"])
    return gp, feas


def oracle_model(meta, arrays, space, prefix=""):
    import oracle

    gp, feas = model(meta, arrays, space, prefix)
    og = oracle.OracleGP(space, gp.configs, meta["outputscale"], meta["noise_variance"],
                         meta["lengthscales"], L=gp._cho[0], alpha=gp.alpha, y_mean=gp.y_mean,
                         y_std=gp.y_std, log_objective=gp.log_objective,
                         use_transforms=gp.use_transforms)
    of = None
    if feas is not None:
        of = oracle.OracleForest(feas.feature, feas.threshold, feas.left, feas.right, feas.value,
                                 feas.roots, feas.max_depth, space, feas.use_transforms, feas.constant)
    return og, of


@lru_cache(maxsize=None)
def cot_for(case: str):
    meta, arrays, space = load(case)
    return build_cot(space) if space.constraints else None


class Ctx:
    """AcquisitionContext look-alike (acquisition.py:54-67)."""

    def __init__(self, gp, feas, best, eps_f=0.0, rng=None, evaluated=None):
        self.gp, self.feas, self.best_feasible_value, self.eps_f = gp, feas, best, eps_f
        self.rng = rng if rng is not None else np.random.default_rng(0)
        self.evaluated = evaluated if evaluated is not None else set()
