"""Synthetic scenarios of BASELINE.json's configs and encoded pool samplers.

Spaces are given as plain descriptors so the same definition builds the reference's
`boxtune.space` objects (golden-fixture generation, tests/golden/make_golden.py) and this
package's standalone `space` objects (GPU box, bench).

    C1  2-D continuous Branin, GP+EI                          (configs[0])
    C2  TACO SpMM-style: log ordinal tiles + 5-loop permutation + divisibility constraints
    C3  RISE&ELEVATE MM_GPU-style: 10 log ordinals, known + hidden constraints (RF)   (headline)
    C4  HPVM2FPGA-style: 20 categorical/ordinal dims, coarse LML over 64 restarts
    C5  d=10 mixed (BASELINE.md probe space), n=500
    M200  the north-star configuration: the C5 space at n=200 with a hidden rule (RF on)
"""
from __future__ import annotations

import math

import numpy as np

from .layout import SpaceLayout, domain_values, pack_perm

POW2 = [2 ** k for k in range(11)]


def _p(name, kind, **kw):
    d = {"name": name, "kind": kind}
    d.update(kw)
    return d


SCENARIOS = {
    "C1": {
        "params": [_p("x1", "real", lo=-5.0, hi=10.0), _p("x2", "real", lo=0.0, hi=15.0)],
        "constraints": [],
    },
    "C2": {
        "params": [
            _p("i_split", "ordinal", values=POW2, transform="log"),
            _p("k_split", "ordinal", values=POW2, transform="log"),
            _p("unroll", "ordinal", values=POW2[:6], transform="log"),
            _p("omp_chunk", "ordinal", values=POW2[:9], transform="log"),
            _p("threads", "integer", lo=1, hi=32),
            _p("sched", "categorical", values=["static", "dynamic", "guided"]),
            _p("order", "permutation", size=5, metric="spearman"),
        ],
        "constraints": ["i_split % unroll == 0", "k_split >= unroll", "omp_chunk * threads <= 2048",
                        "sched != 'static' || omp_chunk == 1"],
    },
    "C3": {
        "params": [_p(n, "ordinal", values=POW2, transform="log")
                   for n in ("gs0", "gs1", "ls0", "ls1", "tm", "tn", "tk", "vw", "wpt0", "wpt1")],
        "constraints": ["gs0 % ls0 == 0", "gs1 % ls1 == 0", "ls0 * ls1 <= 1024", "tm * tn <= 4096"],
    },
    "C4": {
        "params": ([_p(f"c{i}", "categorical", values=[f"v{j}" for j in range(2 + i % 3)])
                    for i in range(10)]
                   + [_p(f"o{i}", "ordinal", values=POW2[:8], transform="log") for i in range(5)]
                   + [_p(f"n{i}", "integer", lo=1, hi=16) for i in range(5)]),
        "constraints": [],
    },
    "C5": {
        "params": [
            _p("t1", "ordinal", values=POW2, transform="log"),
            _p("t2", "ordinal", values=POW2, transform="log"),
            _p("t3", "ordinal", values=[1, 2, 4, 8, 16, 32], transform="log"),
            _p("u1", "integer", lo=1, hi=16),
            _p("u2", "integer", lo=0, hi=7),
            _p("r1", "real", lo=0.0, hi=1.0),
            _p("c1", "categorical", values=["a", "b", "c", "d"]),
            _p("c2", "categorical", values=["x", "y"]),
            _p("p1", "permutation", size=5, metric="spearman"),
            _p("p2", "permutation", size=4, metric="kendall"),
        ],
        "constraints": [],
    },
}

# GP training size n, pool size q
SIZES = {"C1": (49, 10_000), "C2": (60, 100_000), "C3": (200, 1_000_000), "C4": (200, 0),
         "C5": (500, 1_000_000), "M200": (200, 1_000_000)}


class ParamSpec:
    """A parameter descriptor with the attribute names SpaceLayout reads from the reference's
    `Parameter` (space.py:33-140): kind, name, lo / hi, values, transform, size,
    permutation_metric.  Data only - no validation, sampling or neighbour logic (that is the
    reference's)."""

    def __init__(self, d: dict):
        self.name, self.kind = d["name"], d["kind"]
        self.transform = d.get("transform", "none")
        self.lo, self.hi = d.get("lo"), d.get("hi")
        self.values = tuple(d["values"]) if "values" in d else None
        self.size = d.get("size")
        self.permutation_metric = d.get("metric", "spearman") if self.kind == "permutation" else None

    def numeric_bounds(self):
        if self.kind == "ordinal":
            return float(self.values[0]), float(self.values[-1])
        return float(self.lo), float(self.hi)


class SpaceSpec:
    """A search-space descriptor for workloads built without the reference (bench.py on the GPU
    box): `parameters` and `constraint_texts` as the reference's SearchSpace names them.  Known
    constraints arrive pre-compiled (chain-of-trees tables in the workload fixture)."""

    def __init__(self, desc: dict):
        self.parameters = tuple(ParamSpec(d) for d in desc["params"])
        self.constraint_texts = tuple(desc.get("constraints", ()))
        self.constraints = ()

    @property
    def dimension(self) -> int:
        return len(self.parameters)

    def index_of(self, name: str) -> int:
        return [p.name for p in self.parameters].index(name)


def build_space(name_or_desc, module=None):
    """SearchSpace from a descriptor: the reference's (`module` = boxtune.space) or, without a
    module, a `SpaceSpec`."""
    desc = SCENARIOS[name_or_desc] if isinstance(name_or_desc, str) else name_or_desc
    if module is None:
        return SpaceSpec(desc)
    P = module.Parameter
    params = []
    for d in desc["params"]:
        k = d["kind"]
        if k == "real":
            params.append(P.real(d["name"], d["lo"], d["hi"], d.get("transform", "none")))
        elif k == "integer":
            params.append(P.integer(d["name"], d["lo"], d["hi"], d.get("transform", "none")))
        elif k == "ordinal":
            params.append(P.ordinal(d["name"], d["values"], d.get("transform", "none")))
        elif k == "categorical":
            params.append(P.categorical(d["name"], d["values"]))
        else:
            params.append(P.permutation(d["name"], d["size"], d.get("metric", "spearman")))
    return module.SearchSpace(params, desc.get("constraints", ()))


# -- objectives and hidden rules (deterministic, positive -> log objective on) -----------------
def objective(name: str, cfg) -> float:
    if name == "C1":  # Branin, min 0.397887
        x1, x2 = cfg
        a, b, c, r, s, t = 1.0, 5.1 / (4 * math.pi ** 2), 5 / math.pi, 6.0, 10.0, 1 / (8 * math.pi)
        return a * (x2 - b * x1 ** 2 + c * x1 - r) ** 2 + s * (1 - t) * math.cos(x1) + s
    if name == "C2":
        i, k, u, ch, th, sched, order = cfg
        base = (1.0 + 0.05 * (math.log2(i) - 6) ** 2 + 0.05 * (math.log2(k) - 4) ** 2
                + 0.1 * (math.log2(u) - 2) ** 2 + 0.02 * abs(th - 16)
                + {"static": 0.0, "dynamic": 0.3, "guided": 0.15}[sched])
        return base + 0.05 * sum((a - b) ** 2 for a, b in zip(order, (3, 1, 4, 2, 5)))
    if name == "C3":
        lg = [math.log2(v) for v in cfg]
        return 1.0 + sum(0.03 * (x - (3 + (j % 4))) ** 2 for j, x in enumerate(lg)) \
            + 0.01 * lg[0] * lg[4]
    if name == "C4":
        cats = sum((int(v[1:]) * (0.1 + 0.02 * j)) for j, v in enumerate(cfg[:10]))
        ords = sum(0.05 * (math.log2(v) - 3) ** 2 for v in cfg[10:15])
        ints = sum(0.01 * (v - 9) ** 2 for v in cfg[15:])
        return 1.0 + cats + ords + ints
    if name == "C5":
        t1, t2, t3, u1, u2, r1, c1, c2, p1, p2 = cfg
        return (1.0 + 0.05 * (math.log2(t1) - 5) ** 2 + 0.05 * (math.log2(t2) - 3) ** 2
                + 0.1 * (math.log2(t3) - 2) ** 2 + 0.02 * (u1 - 10) ** 2 + 0.03 * (u2 - 2) ** 2
                + (r1 - 0.3) ** 2 + {"a": 0.0, "b": 0.1, "c": 0.2, "d": 0.05}[c1]
                + (0.07 if c2 == "y" else 0.0)
                + 0.02 * sum((a - b) ** 2 for a, b in zip(p1, (2, 4, 1, 5, 3)))
                + 0.05 * sum(1 for a, b in zip(p2, (4, 3, 2, 1)) if a != b))
    raise KeyError(name)


def hidden_ok(name: str, cfg) -> bool:
    if name == "C3":  # resource budget (~46% of the known-feasible set is hidden-infeasible)
        gs0, gs1, ls0, ls1, tm, tn, tk, vw, wpt0, wpt1 = cfg
        return tm * tn * tk <= 2 ** 18 and vw * wpt0 * wpt1 <= 2 ** 16
    if name == "C4":
        return not (cfg[0] == "v1" and cfg[10] >= 64)
    if name == "M200":  # BASELINE.md probe rule (~70% of the dense space feasible)
        return cfg[0] * cfg[1] <= 4096
    return True


# -- encoded pool samplers (bench pools; statistical, not RNG-stream parity) --------------------
def sample_rows_uniform(layout: SpaceLayout, n: int, rng: np.random.Generator) -> np.ndarray:
    """Uniform draws from the dense space, directly in row form (sample_uniform's distribution,
    space.py:312-332)."""
    rows = np.zeros((n, layout.row_words), dtype=np.uint32)
    as64 = rows.view(np.uint64)
    for k, (p, slot) in enumerate(zip(layout.space.parameters, layout.slots)):
        if p.kind == "real":
            v = rng.uniform(p.lo, p.hi, size=n)
            from .layout import numeric_coords
            c = numeric_coords(p, v, layout.use_transforms)
            as64[:, slot.word // 2] = v.view(np.uint64)
            as64[:, slot.word // 2 + 1] = np.asarray(c, np.float64).view(np.uint64)
        elif p.kind == "permutation":
            m = p.size
            perm = np.argsort(rng.random((n, m)), axis=1)
            packed = np.zeros(n, dtype=np.uint64)
            for i in range(m):
                packed = (packed << np.uint64(4)) | perm[:, i].astype(np.uint64)
            as64[:, slot.word // 2] = packed
        else:
            rows[:, slot.word] = rng.integers(0, layout.params[k].size, size=n, dtype=np.int64)
    return rows


def sample_rows_cot(layout: SpaceLayout, cot, n: int, rng: np.random.Generator) -> np.ndarray:
    """Leaf-uniform draws from a chain of trees (constraints.py:471-523 distribution)."""
    rows = sample_rows_uniform(layout, n, rng)
    for g in cot.groups:
        if g.kind != "tree":
            continue
        paths = _paths(g)
        idx_tab = np.asarray([[layout.slots[i].index[v] for i, v in zip(g.indices, path)]
                              for path in paths], dtype=np.uint32)
        pick = rng.integers(0, len(paths), size=n)
        for col, i in enumerate(g.indices):
            rows[:, layout.slots[i].word] = idx_tab[pick, col]
    return rows


def _paths(g):
    out = []

    def walk(node, acc):
        if not node.children:
            if len(acc) == len(g.indices):
                out.append(tuple(acc))
            return
        for ch in node.children:
            walk(ch, acc + [ch.value])

    walk(g.root, [])
    return out


def all_domain_rows(layout: SpaceLayout) -> int:
    total = 1
    for p in layout.space.parameters:
        total *= len(domain_values(p)) if p.kind != "permutation" else math.factorial(p.size)
    return total


def pack(perm) -> int:
    return pack_perm(perm, len(perm))
