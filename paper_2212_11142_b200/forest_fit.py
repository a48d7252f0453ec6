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
    # every tree's node arrays, [tree][node] (a tree finishes in the round whose draws sufficed)
    all_f = np.empty((n_trees, max_nodes), np.int32)
    all_t = np.empty((n_trees, max_nodes), np.float64)
    all_l = np.empty((n_trees, max_nodes), np.int32)
    all_r = np.empty((n_trees, max_nodes), np.int32)
    all_v = np.empty((n_trees, max_nodes), np.float64)
    all_n = np.zeros(n_trees, np.int64)
    todo = np.arange(n_trees)
    while len(todo):
        lens = np.array([len(draws[t]) for t in todo], dtype=np.int32)
        max_draws = int(lens.max())
        T = len(todo)
        if (lens == max_draws).all():
            feats = np.ascontiguousarray(np.stack([draws[t] for t in todo]), dtype=np.int32)
        else:
            feats = np.zeros((T, max_draws, k), dtype=np.int32)
            for i, t in enumerate(todo):
                feats[i, :lens[i]] = draws[t]
        out_f = np.empty((T, max_nodes), np.int32)
        out_t = np.empty((T, max_nodes), np.float64)
        out_l = np.empty((T, max_nodes), np.int32)
        out_r = np.empty((T, max_nodes), np.int32)
        out_v = np.empty((T, max_nodes), np.float64)
        out_n = np.empty(T, np.int32)
        out_s = np.empty(T, np.int32)
        p = lambda a: a.ctypes.data_as(C.c_void_p)
        sc._check(lib.bx_rf_fit(sc.h, p(Xc), p(yc), n, F, T, p(np.ascontiguousarray(boot[todo])), p(feats), p(lens),
                                max_draws, k, max_depth, max_nodes, p(out_f), p(out_t), p(out_l), p(out_r), p(out_v),
                                p(out_n), p(out_s), sc.stream))
        bad = np.flatnonzero((out_s != 0) & (out_s != 1))
        if len(bad):
            raise N.NativeError(N.BX_ERR_UNSUPPORTED, f"rf_fit: tree {int(todo[bad[0]])} exceeded {max_nodes} nodes")
        done = out_s == 0
        for dst, src in ((all_f, out_f), (all_t, out_t), (all_l, out_l), (all_r, out_r), (all_v, out_v)):
            dst[todo[done]] = src[done]
        all_n[todo[done]] = out_n[done]
        for t in todo[~done]:  # more feature subsets: continue the tree's own generator
            streams.more(int(t), DRAWS)
        todo = todo[~done]
    # the reference appends tree after tree to flat arrays: node j of tree t at roots[t] + j, child
    # indices shifted by the tree's base
    roots = np.cumsum(all_n) - all_n
    keep = np.arange(max_nodes)[None, :] < all_n[:, None]
    shift = roots[:, None]
    model.feature = all_f[keep].astype(np.int32)
    model.threshold = all_t[keep]
    model.left = np.where(all_l >= 0, all_l + shift, -1)[keep].astype(np.int32)
    model.right = np.where(all_r >= 0, all_r + shift, -1)[keep].astype(np.int32)
    model.value = all_v[keep]
    model.roots = roots.astype(np.int32)
    return model
