"""Load tests/golden fixtures into the REFERENCE's objects (search spaces, chains of trees, and
optionally GPModel / FeasibilityModel), this package's stand-ins and the oracle's objects.

The reference package is imported from oracle/_ref (installed by oracle/ship_ref.sh, which
build() runs; it travels to the GPU box with the snapshot) or, in the build container, from
/root/reference/pkg/src.
"""
from __future__ import annotations

import json
import sys
from functools import lru_cache
from pathlib import Path

import numpy as np

from paper_2212_11142_b200 import scenarios
from paper_2212_11142_b200.models import Forest, GPState, Hyper

GOLDEN = Path(__file__).resolve().parent / "golden"
ROOT = Path(__file__).resolve().parent.parent
REF_PATHS = (ROOT / "oracle" / "_ref", Path("/root/reference/pkg/src"))


def ref():
    """The unmodified reference package (boxtune)."""
    if "boxtune" not in sys.modules:
        for p in REF_PATHS:
            if (p / "boxtune" / "__init__.py").exists():
                sys.path.insert(0, str(p))
                break
        else:
            raise RuntimeError("reference package not found: run oracle/ship_ref.sh (build() does)")
    import boxtune

    return boxtune
CASES = ["mixed_fit", "mixed_metrics", "C1", "C2", "C3", "C4", "M200"]
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
    space = scenarios.build_space(meta["space"], ref().space)
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
    return ref().build_cot(space) if space.constraints else None


class Ctx:
    """AcquisitionContext look-alike (acquisition.py:54-67)."""

    def __init__(self, gp, feas, best, eps_f=0.0, rng=None, evaluated=None):
        self.gp, self.feas, self.best_feasible_value, self.eps_f = gp, feas, best, eps_f
        self.rng = rng if rng is not None else np.random.default_rng(0)
        self.evaluated = evaluated if evaluated is not None else set()


def ref_model(meta, arrays, space, prefix=""):
    """The reference's own GPModel / FeasibilityModel objects for a fixture.  GPModel is rebuilt
    through its constructor (surrogate.py:274-303) from the stored training set and
    hyperparameters - the same numpy/scipy calls that produced the fixture - and its Cholesky
    factor is checked against the stored one; the forest gets the stored arrays."""
    bt = ref()
    h = bt.GPHyperparameters(outputscale=meta["outputscale"], noise_variance=meta["noise_variance"],
                             lengthscales=tuple(meta["lengthscales"]))
    train = [to_cfg(space, c) for c in meta["train"]]
    gp = bt.GPModel(space, train, meta["y"], h, log_objective=meta["log_objective"],
                    use_transforms=meta["use_transforms"])
    np.testing.assert_allclose(np.tril(gp._cho[0]), arrays[prefix + "L"], rtol=1e-12, atol=1e-14)
    feas = None
    _, f = model(meta, arrays, space, prefix)
    if f is not None:
        feas = bt.FeasibilityModel(space=space, n_trees=f.n_trees, max_depth=f.max_depth,
                                   bootstrap_seeds=np.zeros(0, np.int64),
                                   use_transforms=meta["use_transforms"], feature=f.feature,
                                   threshold=f.threshold, left=f.left, right=f.right, value=f.value,
                                   roots=f.roots, constant=f.constant)
    return gp, feas
