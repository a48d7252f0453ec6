"""Candidate pools drawn straight into encoded rows.

The reference's uniform sampler (space.py:312-332) builds a Python tuple per candidate: one
vectorised NumPy draw per scalar parameter, n `rng.permutation(m)` calls per permutation
parameter, then a tuple per row - about 45 ms for the 5000-candidate pool of every BO iteration
on a d = 10 mixed space, plus the encoding of those tuples into rows.  Here the same draws land
in the row format directly:

* scalar parameters: the same NumPy calls with the same arguments in the same parameter order,
  so the values are the reference's; the finite kinds keep their domain index, reals their value
  and coordinate (`numeric_coords`, the reference's expression);
* permutations: bx_pcg64_permutations replays numpy's Generator.permutation from the PCG64 state
  (Fisher-Yates from the top with random_interval draws on the buffered 32-bit stream) and leaves
  the generator in the state the n Python calls would;
* the chain-of-trees leaf-uniform sampler (constraints.py:471-518, the default pool when known
  constraints exist): per dependency group the same `rng.integers(leaf_count, size=n)` draw, then a
  gather from the group's encoded leaf rows; real / permutation singletons as above;
* `dict.fromkeys` de-duplication becomes first-occurrence unique rows (a row determines its
  configuration and vice versa).

So the pool, its order and the RNG stream the BO loop continues with are the reference's; the
tests compare rows and generator states with the reference's sampler.  Generators other than
PCG64 take the permutations from `rng.permutation` itself.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .layout import numeric_coords

_M64 = (1 << 64) - 1


def is_reference_sampler(fn) -> bool:
    """True when `fn` is the stock `sample_uniform` of a boxtune-style space module."""
    return getattr(fn, "__name__", "") == "sample_uniform" and getattr(fn, "__module__", "").endswith(".space")


def is_reference_cot(cot) -> bool:
    """True for the stock ChainOfTrees (its leaf-uniform sampler is the one cot_rows replays)."""
    t = type(cot)
    return (t.__name__ == "ChainOfTrees" and t.__module__.endswith(".constraints")
            and getattr(t.sample_leaf_uniform, "__module__", "") == t.__module__
            and hasattr(cot, "groups") and hasattr(cot, "_ensure_leaf_arrays"))


_REPLAY_OK = None


def replay_ok() -> bool:
    """Whether bx_pcg64_* reproduce this NumPy's Generator.permutation / choice (checked once on
    scratch generators; a NumPy whose algorithms differ gets the Python calls instead)."""
    global _REPLAY_OK
    if _REPLAY_OK is None:
        try:
            ok = True
            for seed, m, pop, k in ((11, 5, 21, 5), (12, 9, 64, 8)):
                a, b = np.random.default_rng(seed), np.random.default_rng(seed)
                a.integers(7), b.integers(7)  # a half-used 32-bit buffer
                got = _replay_permutations(a, 64, m)
                want = [sum(int(v) << (4 * (m - 1 - i)) for i, v in enumerate(b.permutation(m))) for _ in range(64)]
                ok &= [int(x) for x in got] == want
                got = _replay_choice(a, 64, pop, k)
                ok &= all(np.array_equal(got[r], b.choice(pop, size=k, replace=False)) for r in range(64))
                ok &= repr(a.bit_generator.state) == repr(b.bit_generator.state)
            seeds = [0, 5, (1 << 32) - 1, 123456789]
            f = TreeStreams(seeds, 9, 13, 3, 4, native=True)
            for t, s in enumerate(seeds):
                g = np.random.default_rng(s)
                ok &= np.array_equal(f.boot[t], g.integers(0, 9, size=9))
                ok &= all(np.array_equal(f.draws[t][r], g.choice(13, size=3, replace=False)) for r in range(4))
                f.more(t, 2)
                ok &= all(np.array_equal(f.draws[t][r], g.choice(13, size=3, replace=False)) for r in (4, 5))
            _REPLAY_OK = bool(ok)
        except Exception:
            _REPLAY_OK = False
    return _REPLAY_OK


def _replay_permutations(rng, n, m):
    out = np.empty(n, dtype=np.uint64)
    _pcg64_call(rng, N.lib().bx_pcg64_permutations, n, m, out.ctypes.data_as(C.c_void_p))
    return out


def _replay_choice(rng, n, pop, k):
    out = np.empty((n, k), dtype=np.int32)
    _pcg64_call(rng, N.lib().bx_pcg64_choice, n, pop, k, out.ctypes.data_as(C.c_void_p))
    return out


def permutation_rows(rng, n: int, m: int) -> np.ndarray:
    """[rng.permutation(m) for _ in range(n)] packed as layout rows (uint64, 0-based elements)."""
    out = np.empty(n, dtype=np.uint64)
    if rng.bit_generator.state.get("bit_generator") == "PCG64" and n > 0 and replay_ok():
        return _replay_permutations(rng, n, m)
    for r in range(n):
        x = 0
        for v in rng.permutation(m):
            x = (x << 4) | int(v)
        out[r] = x
    return out


def _codes(lay, k, p):
    """Row code of each domain index of a finite parameter (the layout's value -> index map)."""
    cache = lay.__dict__.setdefault("_sample_codes", {})
    if k not in cache:
        idx = lay.slots[k].index
        cache[k] = np.asarray([idx[v] for v in p.values], dtype=np.uint32)
    return cache[k]


def uniform_rows(lay, n: int, rng) -> np.ndarray:
    """lay.encode(sample_uniform(space, n, rng)) with the same RNG consumption (space.py:320-331)."""
    rows = np.zeros((n, lay.row_words), dtype=np.uint32)
    as64 = rows.view(np.uint64)
    for k, (p, slot) in enumerate(zip(lay._params, lay.slots)):
        w = slot.word
        if p.kind == "real":
            v = rng.uniform(p.lo, p.hi, size=n)
            v = np.where(v == 0.0, 0.0, v)  # as SpaceLayout.encode: -0.0 == 0.0 in tuple equality
            as64[:, w // 2] = v.view(np.uint64)
            as64[:, w // 2 + 1] = np.asarray(numeric_coords(p, v, lay.use_transforms), np.float64).view(np.uint64)
        elif p.kind == "integer":
            rows[:, w] = rng.integers(int(p.lo), int(p.hi) + 1, size=n) - int(p.lo)
        elif p.kind in ("ordinal", "categorical"):
            rows[:, w] = _codes(lay, k, p)[rng.integers(len(p.values), size=n)]
        else:
            as64[:, w // 2] = permutation_rows(rng, n, p.size)
    return rows


def rejection_rows(lay, n: int, rng, feasible) -> np.ndarray:
    """The rejection front-end of acquisition.py:122-134 over rows: batches of n uniform rows until n
    pass `feasible(rows) -> bool mask` or 50 n were drawn, in draw order."""
    out, count, attempts = [], 0, 0
    while count < n and attempts < 50 * n:
        batch = uniform_rows(lay, n, rng)
        attempts += n
        take = batch[np.asarray(feasible(batch), dtype=bool)][: n - count]
        out.append(take)
        count += len(take)
    return np.concatenate(out) if out else np.zeros((0, lay.row_words), dtype=np.uint32)


def unique_rows(rows: np.ndarray) -> np.ndarray:
    """First occurrences, in order (list(dict.fromkeys(configs))): bx_unique_rows, a hash set over
    the rows in one pass."""
    if len(rows) < 2:
        return rows
    rows = np.ascontiguousarray(rows, dtype=np.uint32)
    first = np.empty(len(rows), dtype=np.int64)
    n = N.lib().bx_unique_rows(rows.ctypes.data_as(C.c_void_p), len(rows), rows.shape[1],
                               first.ctypes.data_as(C.c_void_p))
    if n < 0:
        raise N.NativeError(int(-n), "bx_unique_rows")
    return rows if n == len(rows) else rows[first[:n]]


def _pcg64_call(rng, fn, *args):
    """Run a bx_pcg64_* replay on rng's PCG64 state and store the advanced state back."""
    st = rng.bit_generator.state
    s, inc = int(st["state"]["state"]), int(st["state"]["inc"])
    state = np.array([s >> 64, s & _M64, inc >> 64, inc & _M64], dtype=np.uint64)
    has32 = C.c_int32(int(st["has_uint32"]))
    uint = C.c_uint32(int(st["uinteger"]))
    code = fn(state.ctypes.data_as(C.c_void_p), C.byref(has32), C.byref(uint), *args)
    if code != N.BX_OK:
        raise N.NativeError(code, fn.__name__)
    st["state"]["state"] = (int(state[0]) << 64) | int(state[1])
    st["has_uint32"] = int(has32.value)
    st["uinteger"] = int(uint.value)
    rng.bit_generator.state = st


def choice_rows(rng, n: int, pop: int, k: int) -> np.ndarray:
    """[rng.choice(pop, size=k, replace=False) for _ in range(n)] as an (n, k) int32 array."""
    out = np.empty((n, k), dtype=np.int32)
    if rng.bit_generator.state.get("bit_generator") == "PCG64" and pop <= 10000 and n > 0 and k > 0 and replay_ok():
        return _replay_choice(rng, n, pop, k)
    for r in range(n):
        out[r] = rng.choice(pop, size=k, replace=False)
    return out


def _leaf_table(lay, cot, g):
    """The encoded rows (only the group's words set) of a tree group's leaf paths, cached."""
    cache = lay.__dict__.setdefault("_cot_tables", {})
    key = (id(cot), id(g))
    hit = cache.get(key)
    if hit is not None and hit[0] is g.leaf_values:
        return hit[1]
    paths = g.leaf_values
    table = np.zeros((len(paths), lay.row_words), dtype=np.uint32)
    for j, k in enumerate(g.indices):
        lay.encode_param(table, k, [path[j] for path in paths])
    cache[key] = (paths, table)
    return table


def cot_rows(lay, cot, n: int, rng) -> np.ndarray:
    """lay.encode(cot.sample_leaf_uniform(n, rng)) with the same RNG consumption
    (constraints.py:471-518, the leaf-uniform mode): per group in order - a tree with leaf arrays
    draws `rng.integers(leaf_count, size=n)` and gathers its encoded leaf rows; a real singleton
    draws n scalar uniforms (one vector call consumes the stream identically); a permutation
    singleton n permutations (replayed); a tree too large for leaf arrays runs the reference's own
    per-draw descent and its output is encoded."""
    space = lay.space
    if n < 1 or cot.count() == 0:
        return lay.encode(cot.sample_leaf_uniform(n, rng))  # the reference raises its own error
    rows = np.zeros((n, lay.row_words), dtype=np.uint32)
    as64 = rows.view(np.uint64)
    for g in cot.groups:
        if g.kind != "tree":
            k = g.indices[0]
            p = space.parameters[k]
            if p.kind == "permutation":
                as64[:, lay.slots[k].word // 2] = permutation_rows(rng, n, p.size)
            elif p.kind == "real":
                lay.encode_param(rows, k, rng.uniform(p.lo, p.hi, size=n))
            else:
                lay.encode_param(rows, k, [p.sample(rng) for _ in range(n)])
            continue
        cot._ensure_leaf_arrays(g)
        if g.leaf_values is not None:
            idx = rng.integers(g.root.leaf_count, size=n)
            table = _leaf_table(lay, cot, g)
            for k in g.indices:
                ws = lay.param_words(k)
                rows[:, ws] = table[idx, ws]
        else:
            out = cot._sample_group(g, n, rng, False)
            for j, k in enumerate(g.indices):
                lay.encode_param(rows, k, [v[j] for v in out])
    return rows


class TreeStreams:
    """The random-forest fit's per-tree generators (feasibility.py:119-190): tree t's generator is
    np.random.default_rng(seeds[t]); it draws the bootstrap rows `integers(0, n, size=n)` (`boot[t]`)
    and then the feature subsets `choice(pop, size=k, replace=False)` in order (`draws[t]`, ndraws up
    front, `more(t, count)` continues the same generator).  With PCG64 replay available the whole
    forest's draws are one bx_pcg64_forest_draws call (SeedSequence seeding included) and the
    continuations bx_pcg64_choice calls on the kept states; otherwise numpy's generators draw them."""

    def __init__(self, seeds, n: int, pop: int, k: int, ndraws: int, native: bool | None = None):
        seeds = np.ascontiguousarray(seeds, dtype=np.uint64)
        T = len(seeds)
        self.pop, self.k = pop, k
        if native is None:
            native = pop <= 10000 and replay_ok()
        self.native = native
        if native:
            self.boot = np.empty((T, n), np.int32)
            sub = np.empty((T, ndraws, k), np.int32)
            self._state = np.empty((T, 4), np.uint64)
            self._has32 = np.empty(T, np.int32)
            self._uint = np.empty(T, np.uint32)
            p = lambda a: a.ctypes.data_as(C.c_void_p)
            code = N.lib().bx_pcg64_forest_draws(p(seeds), T, n, pop, k, ndraws, p(self.boot), p(sub), p(self._state),
                                                 p(self._has32), p(self._uint))
            if code != N.BX_OK:
                raise N.NativeError(code, "bx_pcg64_forest_draws")
            self.draws = list(sub)
        else:
            self._gens = [np.random.default_rng(int(s)) for s in seeds]
            self.boot = np.stack([g.integers(0, n, size=n) for g in self._gens]).astype(np.int32).reshape(T, n)
            self.draws = [choice_rows(g, ndraws, pop, k) for g in self._gens]

    def more(self, t: int, count: int) -> None:
        """Append the next `count` feature subsets of tree t's generator to draws[t]."""
        if self.native:
            out = np.empty((count, self.k), np.int32)
            st = self._state[t]  # a view: the advanced state is written back in place
            code = N.lib().bx_pcg64_choice(st.ctypes.data_as(C.c_void_p),
                                           self._has32[t:].ctypes.data_as(C.c_void_p),
                                           self._uint[t:].ctypes.data_as(C.c_void_p), count, self.pop, self.k,
                                           out.ctypes.data_as(C.c_void_p))
            if code != N.BX_OK:
                raise N.NativeError(code, "bx_pcg64_choice")
        else:
            out = choice_rows(self._gens[t], count, self.pop, self.k)
        self.draws[t] = np.concatenate([self.draws[t], out])
