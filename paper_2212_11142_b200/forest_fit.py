"""`rf_fit` (feasibility.py:155-197) with the trees built on the GPU.

The reference's own pieces do everything but the tree building: `encode_configs`, the canonical
lexsort of the rows, the per-tree bootstrap seeds drawn from the caller's RNG, the single-class
shortcut and the `FeasibilityModel` returned.  Each tree's generator (`default_rng(seed)`): the
bootstrap rows and, in order, the feature subsets its eligible nodes draw (`tree_rng.choice(F, k,
replace=False)`, feasibility.py:119) are drawn on the host exactly as the reference draws them -
replayed natively for the whole forest (sampling.TreeStreams, bx_pcg64_forest_draws); the device walks
the tree depth first (bx_rf_fit, forest_fit.cu) so its i-th eligible node takes the i-th subset.
A tree that needs more subsets than were drawn is built again after drawing more from the same
generator.  The arrays - node ids, features, thresholds, children, leaf values - equal the
reference's bit for bit.
"""
from __future__ import annotations

import ctypes as C
import importlib
import math

import numpy as np

from . import _native as N
from .device import scorer
from .sampling import TreeStreams

_DEFAULT = object()
DRAWS = 48  # feature subsets drawn per tree up front (M200-sized forests use ~30)


def _feasibility(space):
    pkg = type(space).__module__.rsplit(".", 1)[0]
    return importlib.import_module(pkg + ".feasibility")


def rf_fit(space, configs, labels, rng, n_trees=_DEFAULT, max_depth=_DEFAULT, use_transforms: bool = True):
    """Drop-in for `rf_fit`: same arguments, RNG consumption, errors and `FeasibilityModel`."""
    Fm = _feasibility(space)
    n_trees = Fm.N_TREES if n_trees is _DEFAULT else n_trees
    max_depth = Fm.MAX_DEPTH if max_depth is _DEFAULT else max_depth
    if len(configs) < 1:
        raise Fm.FeasibilityError("need at least one record to fit the feasibility model")
    if len(configs) != len(labels):
        raise Fm.FeasibilityError("configs and labels differ in length")
    X = Fm.encode_configs(space, configs, use_transforms)
    y = np.asarray([1.0 if b else 0.0 for b in labels])
    order = np.lexsort(np.vstack([X.T, y]))   # record-order invariance (feasibility.py:171)
    X, y = X[order], y[order]
    seeds = rng.integers(0, 2 ** 32, size=n_trees, dtype=np.uint64)
    model = Fm.FeasibilityModel(space=space, n_trees=n_trees, max_depth=max_depth, bootstrap_seeds=seeds,
                                use_transforms=use_transforms)
    if y.min() == y.max():
        model.constant = float(y[0])
        return model
    n, F = X.shape
    k = max(1, round(math.sqrt(F)))
    # each tree's generator default_rng(seed): bootstrap rows, then the feature subsets in the order
    # it draws them - replayed natively for the whole forest (bx_pcg64_forest_draws), no per-tree
    # or per-draw Python call
    streams = TreeStreams(seeds, n, F, k, DRAWS)
    boot, draws = streams.boot, streams.draws
    max_nodes = 2 * n + 2
    sc = scorer()
    lib = sc._lib
    Xc = np.ascontiguousarray(X, dtype=np.float64)
    yc = np.ascontiguousarray(y, dtype=np.float64)
    trees = [None] * n_trees
    todo = list(range(n_trees))
    while todo:
        max_draws = max(len(draws[t]) for t in todo)
        T = len(todo)
        feats = np.zeros((T, max_draws, k), dtype=np.int32)
        nd = np.zeros(T, dtype=np.int32)
        for i, t in enumerate(todo):
            feats[i, :len(draws[t])] = draws[t]
            nd[i] = len(draws[t])
        out_f = np.empty((T, max_nodes), np.int32)
        out_t = np.empty((T, max_nodes), np.float64)
        out_l = np.empty((T, max_nodes), np.int32)
        out_r = np.empty((T, max_nodes), np.int32)
        out_v = np.empty((T, max_nodes), np.float64)
        out_n = np.empty(T, np.int32)
        out_s = np.empty(T, np.int32)
        p = lambda a: a.ctypes.data_as(C.c_void_p)
        sc._check(lib.bx_rf_fit(sc.h, p(Xc), p(yc), n, F, T, p(np.ascontiguousarray(boot[todo])), p(feats), p(nd),
                                max_draws, k, max_depth, max_nodes, p(out_f), p(out_t), p(out_l), p(out_r), p(out_v),
                                p(out_n), p(out_s), sc.stream))
        again = []
        for i, t in enumerate(todo):
            if out_s[i] == 1:  # more feature subsets: continue the tree's own generator
                streams.more(t, DRAWS)
                again.append(t)
            elif out_s[i] != 0:
                raise N.NativeError(N.BX_ERR_UNSUPPORTED, f"rf_fit: tree {t} exceeded {max_nodes} nodes")
            else:
                m = int(out_n[i])
                trees[t] = (out_f[i, :m].copy(), out_t[i, :m].copy(), out_l[i, :m].copy(), out_r[i, :m].copy(),
                            out_v[i, :m].copy())
        todo = again
    feature, threshold, left, right, value, roots = [], [], [], [], [], []
    base = 0
    for f, th, lft, rgt, v in trees:  # the reference appends tree after tree to flat arrays
        roots.append(base)
        feature.append(f)
        threshold.append(th)
        left.append(np.where(lft >= 0, lft + base, -1))
        right.append(np.where(rgt >= 0, rgt + base, -1))
        value.append(v)
        base += len(f)
    model.feature = np.concatenate(feature).astype(np.int32)
    model.threshold = np.concatenate(threshold)
    model.left = np.concatenate(left).astype(np.int32)
    model.right = np.concatenate(right).astype(np.int32)
    model.value = np.concatenate(value)
    model.roots = np.asarray(roots, np.int32)
    return model
