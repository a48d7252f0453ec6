"""Search-space description used when the reference package is not present (GPU box, bench).

Attribute-compatible with the reference's `Parameter` / `SearchSpace` (space.py:32-255): every
function in this package reads only `kind, name, lo, hi, values, size, transform,
permutation_metric` of a parameter and `parameters, constraints, constraint_texts` of a space, so
reference objects and these objects are interchangeable.  Validation mirrors space.py:50-80.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

KINDS = ("real", "integer", "ordinal", "categorical", "permutation")
PERMUTATION_METRICS = ("kendall", "spearman", "hamming", "naive")
REAL_NEIGHBOR_GRID = 64  # space.py:23


class SpaceError(ValueError):
    pass


@dataclass(frozen=True)
class Parameter:
    name: str
    kind: str
    lo: float | None = None
    hi: float | None = None
    values: tuple = ()
    size: int = 0
    transform: str = "none"
    permutation_metric: str = "spearman"

    def __post_init__(self):
        if self.kind not in KINDS:
            raise SpaceError(f"unknown parameter kind {self.kind!r}")
        if self.kind in ("real", "integer") and not (self.lo is not None and self.hi is not None
                                                     and self.lo < self.hi):
            raise SpaceError(f"{self.name}: need lo < hi")
        if self.kind == "ordinal":
            if not self.values or any(b <= a for a, b in zip(self.values, self.values[1:])):
                raise SpaceError(f"{self.name}: ordinal values must be strictly increasing")
        if self.kind == "categorical" and (not self.values or len(set(self.values)) != len(self.values)):
            raise SpaceError(f"{self.name}: categorical labels must be distinct and non-empty")
        if self.kind == "permutation":
            if self.size < 2:
                raise SpaceError(f"{self.name}: permutation needs size >= 2")
            if self.permutation_metric not in PERMUTATION_METRICS:
                raise SpaceError(f"{self.name}: unknown permutation metric")
        if self.transform == "log":
            lo = self.values[0] if self.kind == "ordinal" else self.lo
            if self.kind not in ("real", "integer", "ordinal") or lo <= 0:
                raise SpaceError(f"{self.name}: log transform needs a positive numeric domain")

    @classmethod
    def real(cls, name, lo, hi, transform="none"):
        return cls(name, "real", lo=float(lo), hi=float(hi), transform=transform)

    @classmethod
    def integer(cls, name, lo, hi, transform="none"):
        return cls(name, "integer", lo=int(lo), hi=int(hi), transform=transform)

    @classmethod
    def ordinal(cls, name, values, transform="none"):
        return cls(name, "ordinal", values=tuple(values), transform=transform)

    @classmethod
    def categorical(cls, name, labels):
        return cls(name, "categorical", values=tuple(labels))

    @classmethod
    def permutation(cls, name, size, metric="spearman"):
        return cls(name, "permutation", size=int(size), permutation_metric=metric)

    @property
    def is_numeric(self) -> bool:
        return self.kind in ("real", "integer", "ordinal")

    def numeric_bounds(self):
        if self.kind == "ordinal":
            return float(self.values[0]), float(self.values[-1])
        return float(self.lo), float(self.hi)

    def domain_size(self):
        if self.kind == "real":
            return math.inf
        if self.kind == "integer":
            return int(self.hi) - int(self.lo) + 1
        if self.kind == "permutation":
            return math.factorial(self.size)
        return len(self.values)

    def domain_values(self) -> list:
        if self.kind == "integer":
            return list(range(int(self.lo), int(self.hi) + 1))
        if self.kind in ("ordinal", "categorical"):
            return list(self.values)
        raise SpaceError(f"{self.name}: domain of kind {self.kind} is not enumerable")


class SearchSpace:
    def __init__(self, parameters, constraints=()):
        self.parameters = tuple(parameters)
        names = [p.name for p in self.parameters]
        if len(set(names)) != len(names):
            raise SpaceError("parameter names must be unique")
        self._index = {n: i for i, n in enumerate(names)}
        self.constraint_texts = tuple(constraints)
        if self.constraint_texts:
            from .constraints import parse_constraint
            self.constraints = tuple(parse_constraint(t, self) for t in self.constraint_texts)
        else:
            self.constraints = ()

    @property
    def dimension(self) -> int:
        return len(self.parameters)

    @property
    def names(self) -> tuple:
        return tuple(p.name for p in self.parameters)

    def index_of(self, name: str) -> int:
        try:
            return self._index[name]
        except KeyError:
            raise SpaceError(f"unknown parameter {name!r}") from None

    def as_dict(self, cfg) -> dict:
        return dict(zip(self.names, cfg))

    def __repr__(self):
        return f"SearchSpace({', '.join(f'{p.name}:{p.kind}' for p in self.parameters)})"


def sample_uniform(space, n: int, rng) -> list:
    """Dense uniform draws consuming `rng` exactly like the reference (space.py:312-332), so a
    run seeded identically sees identical pools."""
    if n < 1:
        raise SpaceError("n must be >= 1")
    cols = []
    for p in space.parameters:
        if p.kind == "real":
            cols.append([float(v) for v in rng.uniform(p.lo, p.hi, size=n)])
        elif p.kind == "integer":
            cols.append([int(v) for v in rng.integers(int(p.lo), int(p.hi) + 1, size=n)])
        elif p.kind in ("ordinal", "categorical"):
            cols.append([p.values[int(i)] for i in rng.integers(len(p.values), size=n)])
        else:
            cols.append([tuple(int(v) for v in rng.permutation(p.size) + 1) for _ in range(n)])
    return [tuple(c[i] for c in cols) for i in range(n)]


def param_sample(p, rng):
    """Parameter.sample (space.py:142-149)."""
    if p.kind == "real":
        return float(rng.uniform(p.lo, p.hi))
    if p.kind == "integer":
        return int(rng.integers(int(p.lo), int(p.hi) + 1))
    if p.kind in ("ordinal", "categorical"):
        return p.values[int(rng.integers(len(p.values)))]
    return tuple(int(v) for v in rng.permutation(p.size) + 1)
