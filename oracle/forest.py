"""Random-forest feasibility restated (feasibility.py:33-89).  Test-only.

Leaves are found by walking each tree per configuration; the mean over trees uses the summation
order numpy applies inside the reference (`value[cur].mean(axis=0)`, feasibility.py:89): running
sum over trees for a batch of q >= 2, numpy's pairwise sum (8 accumulators, blocks of 128) for a
single configuration.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .gp import coords


@dataclass
class OracleForest:
    feature: np.ndarray
    threshold: np.ndarray
    left: np.ndarray
    right: np.ndarray
    value: np.ndarray
    roots: np.ndarray
    max_depth: int
    space: object = None
    use_transforms: bool = True
    constant: float | None = None


def features(space, configs, use_transforms=True) -> np.ndarray:
    """encode_configs (feasibility.py:33-51)."""
    cols = []
    for k, p in enumerate(space.parameters):
        vals = [c[k] for c in configs]
        if p.kind in ("real", "integer", "ordinal"):
            cols.append(coords(p, vals, use_transforms)[:, None])
        elif p.kind == "categorical":
            lab = {v: i for i, v in enumerate(p.values)}
            oh = np.zeros((len(vals), len(p.values)))
            oh[np.arange(len(vals)), [lab[v] for v in vals]] = 1.0
            cols.append(oh)
        else:
            perm = np.asarray(vals, int).reshape(len(vals), p.size)
            pos = np.empty_like(perm)
            rows = np.arange(len(vals))[:, None]
            pos[rows, perm - 1] = np.arange(p.size)[None, :]
            cols.append(pos.astype(float))
    return np.concatenate(cols, axis=1)


def leaves(f: OracleForest, X: np.ndarray) -> np.ndarray:
    """Leaf node of every (tree, row); at most max_depth + 1 descents (feasibility.py:80-88)."""
    feat_of, thr = np.asarray(f.feature), np.asarray(f.threshold)
    lt, rt = np.asarray(f.left), np.asarray(f.right)
    node = np.tile(np.asarray(f.roots, np.int64)[:, None], (1, len(X)))
    col = np.arange(len(X))[None, :]
    for _ in range(f.max_depth + 1):
        fe = feat_of[node]
        live = fe >= 0
        if not live.any():
            break
        go_left = X[col, np.where(live, fe, 0)] <= thr[node]
        node = np.where(live, np.where(go_left, lt[node], rt[node]), node)
    return node


def _pairwise(a) -> float:
    n = len(a)
    if n < 8:
        s = 0.0
        for x in a:
            s += x
        return s
    if n <= 128:
        r = [float(x) for x in a[:8]]
        i = 8
        while i < n - n % 8:
            for j in range(8):
                r[j] += a[i + j]
            i += 8
        s = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
        while i < n:
            s += a[i]
            i += 1
        return s
    h = n // 2
    h -= h % 8
    return _pairwise(a[:h]) + _pairwise(a[h:])


def predict_proba(f: OracleForest, configs, X=None) -> np.ndarray:
    configs = list(configs)
    if f.constant is not None:
        return np.full(len(configs), f.constant)
    if X is None:
        X = features(f.space, configs, f.use_transforms)
    vals = np.asarray(f.value)[leaves(f, X)]  # (T, q)
    T = vals.shape[0]
    if vals.shape[1] == 1:
        return np.array([_pairwise(list(vals[:, 0])) / T])
    acc = vals[0].copy()
    for t in range(1, T):
        acc = acc + vals[t]
    return acc / T
