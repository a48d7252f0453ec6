"""Encoded configuration rows: the HBM layout of candidates, training points and moves.

A configuration tuple (space.py:25) becomes a fixed-width row of uint32 words (format in
include/bx_sm100.h).  Everything the kernels need to reproduce the reference's per-value
arithmetic is tabulated here, on the host, with the reference's own NumPy expressions:

* coordinates of finite numeric domains and of the 64-point real neighbour grid, computed exactly
  as `_numeric_coords` does (surrogate.py:163-170) - so even the host-dependent `np.log` bits
  match the reference running on the same host;
* categorical label ranks under Python's `<` (tuple order used by `_argbest` / `_Tracker`,
  acquisition.py:87-111);
* RF feature columns in `encode_configs` order (feasibility.py:33-51).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _native as N

REAL_NEIGHBOR_GRID = 64
MAX_FINITE_DOMAIN = 1 << 24


def numeric_coords(param, values, use_transforms: bool) -> np.ndarray:
    """`_numeric_coords` (surrogate.py:163-170), same NumPy operations in the same order."""
    lo, hi = param.numeric_bounds() if hasattr(param, "numeric_bounds") else _bounds(param)
    v = np.asarray(values, float)
    if param.transform == "log" and use_transforms:
        v, lo, hi = np.log(v), math.log(lo), math.log(hi)
    if hi == lo:
        return np.zeros_like(v)
    return (v - lo) / (hi - lo)


def _bounds(param):
    if param.kind == "ordinal":
        return float(param.values[0]), float(param.values[-1])
    return float(param.lo), float(param.hi)


def metric_max(metric: str, m: int) -> float:
    """permutation_metric_max (surrogate.py:75-85)."""
    if metric == "kendall":
        return m * (m - 1) / 2.0
    if metric == "spearman":
        return m * (m * m - 1) / 3.0
    if metric == "hamming":
        return float(m)
    if metric == "naive":
        return 1.0
    raise ValueError(f"unknown permutation metric {metric!r}")


def domain_values(param) -> list:
    if param.kind == "integer":
        return list(range(int(param.lo), int(param.hi) + 1))
    return list(param.values)


def pack_perm(perm, m: int) -> int:
    """Element at position i (value 1..m) stored minus one in nibble m-1-i."""
    x = 0
    for v in perm:
        x = (x << 4) | (int(v) - 1)
    return x


def unpack_perm(x: int, m: int) -> tuple:
    return tuple(((x >> (4 * (m - 1 - i))) & 0xF) + 1 for i in range(m))


@dataclass
class _Slot:
    kind: str
    word: int
    index: dict | None  # finite kinds: value -> domain index


class SpaceLayout:
    """Row format + lookup tables of one search space (per `use_transforms` setting)."""

    def __init__(self, space, use_transforms: bool = True):
        self.space = space
        self.use_transforms = bool(use_transforms)
        params = list(space.parameters)
        if not 1 <= len(params) <= N.BX_MAX_PARAMS:
            raise ValueError(f"{len(params)} parameters: supported range is 1..{N.BX_MAX_PARAMS}")
        # 8-byte fields first (real: 4 words, permutation: 2 words), then 1-word fields
        word = 0
        words = [0] * len(params)
        for k, p in enumerate(params):
            if p.kind in ("real", "permutation"):
                words[k] = word
                word += 4 if p.kind == "real" else 2
        for k, p in enumerate(params):
            if p.kind not in ("real", "permutation"):
                words[k] = word
                word += 1
        self.row_words = word + (word & 1)
        if self.row_words > N.BX_MAX_ROW_WORDS:
            raise ValueError(f"row of {self.row_words} words exceeds {N.BX_MAX_ROW_WORDS}")
        descs = (N.ParamDesc * len(params))()
        coord, rank = [], []
        feat = 0
        self.slots: list[_Slot] = []
        self.feature_param: list[int] = []
        for k, p in enumerate(params):
            d = descs[k]
            d.kind = N.KIND_CODES[p.kind]
            d.word = words[k]
            d.is_log = int(p.transform == "log" and self.use_transforms)
            d.feat = feat
            d.rank = 0
            d.coord = 0
            d.raw_mx = 1.0
            index = None
            if p.kind == "permutation":
                if p.size > 16:
                    raise ValueError(f"{p.name}: permutations of more than 16 elements are not supported")
                d.size = p.size
                d.metric = N.METRIC_CODES[p.permutation_metric]
                d.raw_mx = metric_max(p.permutation_metric, p.size)
                feat += p.size
            elif p.kind == "categorical":
                d.size = len(p.values)
                index = {v: i for i, v in enumerate(p.values)}
                d.rank = len(rank)
                try:
                    order = sorted(range(len(p.values)), key=lambda i: p.values[i])
                except TypeError:  # unorderable mixed labels: declaration order
                    order = list(range(len(p.values)))
                r = [0] * len(p.values)
                for pos, i in enumerate(order):
                    r[i] = pos
                rank.extend(r)
                feat += len(p.values)
            elif p.kind == "real":
                d.size = REAL_NEIGHBOR_GRID
                d.lo, d.hi = float(p.lo), float(p.hi)
                step = (p.hi - p.lo) / (REAL_NEIGHBOR_GRID - 1)  # space.py:269
                d.step = float(step)
                grid = [p.lo + j * step for j in range(REAL_NEIGHBOR_GRID)]  # space.py:274
                d.coord = len(coord)
                coord.extend(numeric_coords(p, grid, self.use_transforms).tolist())
                feat += 1
            else:
                dom = domain_values(p)
                if len(dom) > MAX_FINITE_DOMAIN:
                    raise ValueError(f"{p.name}: domain of {len(dom)} values is too large")
                d.size = len(dom)
                d.lo, d.hi = (float(p.lo), float(p.hi)) if p.kind == "integer" else (0.0, 0.0)
                index = {v: i for i, v in enumerate(dom)}
                d.coord = len(coord)
                coord.extend(numeric_coords(p, dom, self.use_transforms).tolist())
                feat += 1
            self.slots.append(_Slot(p.kind, words[k], index))
        self.params = descs
        self.n_params = len(params)
        self.n_features = feat
        self.coord_lut = np.ascontiguousarray(coord if coord else [0.0], dtype=np.float64)
        self.rank_lut = np.ascontiguousarray(rank if rank else [0], dtype=np.int32)
        self._params = params

    # -- rows <-> configurations ------------------------------------------------------------------
    def encode(self, configs) -> np.ndarray:
        """Configuration tuples -> (q, row_words) uint32 rows."""
        configs = list(configs)
        q = len(configs)
        rows = np.zeros((q, self.row_words), dtype=np.uint32)
        if q == 0:
            return rows
        for k in range(self.n_params):
            self.encode_param(rows, k, [cfg[k] for cfg in configs])
        return rows

    def encode_param(self, rows: np.ndarray, k: int, col) -> None:
        """Write parameter k's values `col` (one per row) into its words of `rows`."""
        p, slot = self._params[k], self.slots[k]
        q = rows.shape[0]
        as64 = rows.view(np.uint64)
        if p.kind == "real":
            v = np.asarray(col, dtype=np.float64)
            v = np.where(v == 0.0, 0.0, v)  # -0.0 == 0.0 in tuple equality
            c = numeric_coords(p, v, self.use_transforms)
            as64[:, slot.word // 2] = v.view(np.uint64)
            as64[:, slot.word // 2 + 1] = np.asarray(c, np.float64).view(np.uint64)
        elif p.kind == "permutation":
            m = p.size
            arr = np.asarray(col, dtype=np.int64).reshape(q, m)
            packed = np.zeros(q, dtype=np.uint64)
            for i in range(m):
                packed = (packed << np.uint64(4)) | (arr[:, i] - 1).astype(np.uint64)
            as64[:, slot.word // 2] = packed
        else:
            idx = slot.index
            try:
                rows[:, slot.word] = [idx[v] for v in col]
            except KeyError as exc:
                raise ValueError(f"{p.name}: value {exc.args[0]!r} outside domain") from None

    def param_words(self, k: int) -> slice:
        """The row words parameter k occupies."""
        p, w = self._params[k], self.slots[k].word
        return slice(w, w + (4 if p.kind == "real" else 2 if p.kind == "permutation" else 1))

    def decode(self, rows) -> list:
        """(q, row_words) rows -> configuration tuples with the reference's value types."""
        rows = np.asarray(rows, dtype=np.uint32).reshape(-1, self.row_words)
        cols = []
        as64 = np.ascontiguousarray(rows).view(np.uint64)
        for p, slot in zip(self._params, self.slots):
            if p.kind == "real":
                cols.append([float(x) for x in as64[:, slot.word // 2].view(np.float64)])
            elif p.kind == "permutation":
                cols.append([unpack_perm(int(x), p.size) for x in as64[:, slot.word // 2]])
            else:
                dom = domain_values(p) if p.kind == "integer" else list(p.values)
                cols.append([dom[int(i)] for i in rows[:, slot.word]])
        return [tuple(c[i] for c in cols) for i in range(rows.shape[0])]

    def features(self, rows) -> np.ndarray:
        """encode_configs (feasibility.py:33-51) evaluated from rows (host-side, for tests)."""
        rows = np.asarray(rows, dtype=np.uint32).reshape(-1, self.row_words)
        as64 = np.ascontiguousarray(rows).view(np.uint64)
        out = []
        for k, (p, slot) in enumerate(zip(self._params, self.slots)):
            d = self.params[k]
            if p.kind == "real":
                out.append(as64[:, slot.word // 2 + 1].view(np.float64)[:, None])
            elif p.kind == "permutation":
                m = p.size
                packed = as64[:, slot.word // 2]
                elem = np.stack([((packed >> np.uint64(4 * (m - 1 - i))) & np.uint64(0xF)).astype(np.int64)
                                 for i in range(m)], axis=1)
                out.append(np.argsort(elem, axis=1).astype(float))
            elif p.kind == "categorical":
                oh = np.zeros((rows.shape[0], d.size))
                oh[np.arange(rows.shape[0]), rows[:, slot.word]] = 1.0
                out.append(oh)
            else:
                out.append(self.coord_lut[d.coord + rows[:, slot.word].astype(np.int64)][:, None])
        return np.column_stack(out)
