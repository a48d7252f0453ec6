"""Known constraints: parsing (standalone), device bytecode, and the chain-of-trees tables.

* `parse_constraint` accepts the reference grammar (constraints.py:3-12) with the same typing
  rules (categoricals only ==/!= against strings, permutations excluded, boolean connectives on
  booleans) and produces an AST whose node classes carry the same attribute names as the
  reference's (Num.value, Str.value, Var.name/index/is_categorical, Unary.op/operand,
  BinOp.op/left/right), so `compile_constraints` takes either AST.
* `compile_constraints` emits the stack bytecode interpreted by feasible.cu (eval_program), which
  reproduces `_eval_node` / `eval_constraint` (constraints.py:309-368) including Python's int/float
  promotion, floor modulo, exact int-float comparison and "any ZeroDivision -> False" with both
  operands of && / || evaluated.
* `build_cot` builds a chain of trees for standalone use (dependency groups by union-find,
  depth-first expansion with pruning, constraints.py:542-643); `flatten_cot` turns either the
  reference's ChainOfTrees or ours into the CSR tables of bx_set_cot.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .layout import domain_values

NOT_YET_DECIDABLE = "not-yet-decidable"


class ConstraintError(ValueError):
    def __init__(self, message: str, position: int | None = None):
        super().__init__(message if position is None else f"{message} (column {position})")
        self.position = position


@dataclass(frozen=True)
class Num:
    value: float


@dataclass(frozen=True)
class Str:
    value: str


@dataclass(frozen=True)
class Var:
    name: str
    index: int
    is_categorical: bool


@dataclass(frozen=True)
class Unary:
    op: str
    operand: object


@dataclass(frozen=True)
class BinOp:
    op: str
    left: object
    right: object


class ConstraintExpr:
    def __init__(self, root, text: str, variables: tuple):
        self.root, self.text, self.variables = root, text, variables

    def __repr__(self):
        return f"ConstraintExpr({self.text!r})"


# ---------------------------------------------------------------------------------------------
# tokenizer + recursive-descent parser
# ---------------------------------------------------------------------------------------------
_CMP = ("<", "<=", ">", ">=", "==", "!=")


def _lex(text: str):
    out, i, n = [], 0, len(text)
    while i < n:
        ch = text[i]
        if ch.isspace():
            i += 1
            continue
        col = i + 1
        if text[i:i + 2] in ("<=", ">=", "==", "!=", "&&", "||"):
            out.append(("op", text[i:i + 2], col))
            i += 2
        elif ch in "<>+-*/%()!":
            out.append(("op", ch, col))
            i += 1
        elif ch.isdigit() or (ch == "." and i + 1 < n and text[i + 1].isdigit()):
            j = i
            while j < n and (text[j].isdigit() or text[j] == "."):
                j += 1
            if j < n and text[j] in "eE":
                k = j + 1 + (1 if j + 1 < n and text[j + 1] in "+-" else 0)
                if k < n and text[k].isdigit():
                    j = k
                    while j < n and text[j].isdigit():
                        j += 1
            try:
                out.append(("num", float(text[i:j]), col))  # every literal is a float
            except ValueError:
                raise ConstraintError(f"bad number literal {text[i:j]!r}", col) from None
            i = j
        elif ch in "\"'":
            j = text.find(ch, i + 1)
            if j < 0:
                raise ConstraintError("unterminated string literal", col)
            out.append(("str", text[i + 1:j], col))
            i = j + 1
        elif ch.isalpha() or ch == "_":
            j = i
            while j < n and (text[j].isalnum() or text[j] == "_"):
                j += 1
            out.append(("ident", text[i:j], col))
            i = j
        else:
            raise ConstraintError(f"unexpected character {ch!r}", col)
    out.append(("eof", None, n + 1))
    return out


class _Parser:
    def __init__(self, text, space):
        self.toks, self.i, self.space, self.text, self.seen = _lex(text), 0, space, text, []

    def _peek(self):
        return self.toks[self.i]

    def _is(self, op):
        k, v, _ = self.toks[self.i]
        return k == "op" and v == op

    def _take(self):
        t = self.toks[self.i]
        self.i += 1
        return t

    def _need(self, typ, want, msg):
        if typ != want:
            raise ConstraintError(msg, self._peek()[2])

    def run(self):
        node, typ = self._or()
        k, v, col = self._peek()
        if k != "eof":
            raise ConstraintError(f"unexpected trailing input {v!r}", col)
        if typ != "bool":
            raise ConstraintError("constraint must be a boolean expression", 1)
        names = sorted(set(self.seen), key=self.space.index_of)
        return ConstraintExpr(node, self.text, tuple(names))

    def _chain(self, sub, ops, want, result):
        node, typ = sub()
        while any(self._is(o) for o in ops):
            op = self._take()[1]
            self._need(typ, want, f"{op!r} needs {want} operands")
            rhs, rtyp = sub()
            self._need(rtyp, want, f"{op!r} needs {want} operands")
            node, typ = BinOp(op, node, rhs), result
        return node, typ

    def _or(self):
        return self._chain(self._and, ("||",), "bool", "bool")

    def _and(self):
        return self._chain(self._unary, ("&&",), "bool", "bool")

    def _unary(self):
        if self._is("!"):
            self._take()
            node, typ = self._unary()
            self._need(typ, "bool", "'!' needs a boolean operand")
            return Unary("!", node), "bool"
        node, typ = self._sum()
        k, v, col = self._peek()
        if k == "op" and v in _CMP:
            self._take()
            rhs, rtyp = self._sum()
            if "bool" in (typ, rtyp):
                raise ConstraintError(f"cannot compare boolean with {v!r}", col)
            if typ != rtyp:
                raise ConstraintError("comparison mixes numeric and categorical operands", col)
            if typ == "str" and v not in ("==", "!="):
                raise ConstraintError(f"categorical values support only == and !=, not {v!r}", col)
            return BinOp(v, node, rhs), "bool"
        return node, typ

    def _sum(self):
        return self._chain(self._term, ("+", "-"), "num", "num")

    def _term(self):
        return self._chain(self._factor, ("*", "/", "%"), "num", "num")

    def _factor(self):
        k, v, col = self._peek()
        if k == "op" and v == "-":
            self._take()
            node, typ = self._factor()
            self._need(typ, "num", "unary '-' needs a numeric operand")
            return Unary("-", node), "num"
        if k == "num":
            self._take()
            return Num(v), "num"
        if k == "str":
            self._take()
            return Str(v), "str"
        if k == "ident":
            self._take()
            try:
                idx = self.space.index_of(v)
            except Exception:
                raise ConstraintError(f"unknown identifier {v!r}", col) from None
            p = self.space.parameters[idx]
            if p.kind == "permutation":
                raise ConstraintError(f"permutation parameter {v!r} may not appear in constraints", col)
            self.seen.append(v)
            cat = p.kind == "categorical"
            return Var(v, idx, cat), ("str" if cat else "num")
        if k == "op" and v == "(":
            self._take()
            node, typ = self._or()
            if not self._is(")"):
                raise ConstraintError("expected ')'", self._peek()[2])
            self._take()
            return node, typ
        raise ConstraintError("expected a value, identifier, or '('", col)


def parse_constraint(text: str, space) -> ConstraintExpr:
    return _Parser(text, space).run()


# ---------------------------------------------------------------------------------------------
# host evaluation (standalone chain-of-trees construction only)
# ---------------------------------------------------------------------------------------------
class _Undecided(Exception):
    pass


def _ev(node, b):
    kind = type(node).__name__
    if kind in ("Num", "Str"):
        return node.value
    if kind == "Var":
        if node.name not in b:
            raise _Undecided
        return b[node.name]
    if kind == "Unary":
        x = _ev(node.operand, b)
        return -x if node.op == "-" else (not x)
    x, y = _ev(node.left, b), _ev(node.right, b)
    return {
        "+": lambda: x + y, "-": lambda: x - y, "*": lambda: x * y, "/": lambda: x / y,
        "%": lambda: x % y, "<": lambda: x < y, "<=": lambda: x <= y, ">": lambda: x > y,
        ">=": lambda: x >= y, "==": lambda: x == y, "!=": lambda: x != y,
        "&&": lambda: x and y, "||": lambda: x or y,
    }[node.op]()


def eval_constraint(expr, mapping):
    try:
        return bool(_ev(expr.root, mapping))
    except _Undecided:
        return NOT_YET_DECIDABLE
    except (ZeroDivisionError, OverflowError):
        return False


# ---------------------------------------------------------------------------------------------
# bytecode
# ---------------------------------------------------------------------------------------------
OPS = {"num": 0, "var": 1, "cat": 2, "str": 3, "neg": 4, "not": 5, "+": 6, "-": 7, "*": 8, "/": 9,
       "%": 10, "<": 11, "<=": 12, ">": 13, ">=": 14, "==": 15, "!=": 16, "&&": 17, "||": 18}
MAX_STACK = 32


class Program:
    """Bytecode of all constraints of a space + the per-value tables (bx_set_constraints)."""

    def __init__(self, space, layout):
        self.strings: dict = {}
        self.consts: list[float] = []
        code, begin = [], [0]
        for expr in getattr(space, "constraints", ()):
            depth = self._emit(expr.root, code, space, 0)
            if depth > MAX_STACK:
                raise ValueError(f"constraint {expr.text!r} needs a stack of {depth} > {MAX_STACK}")
            begin.append(len(code))
        self.n = len(begin) - 1
        self.prog_begin = np.asarray(begin, np.int32)
        self.code = np.asarray(code if code else [0], np.int32)
        self.code_len = len(code)
        tag, ival, fval, sid = [], [], [], []
        for p in space.parameters:
            if p.kind in ("real", "permutation"):
                continue
            for v in domain_values(p):
                if p.kind == "categorical":
                    tag.append(0); ival.append(0); fval.append(0.0); sid.append(self._intern(v))
                elif isinstance(v, (bool, np.bool_)) or isinstance(v, (int, np.integer)):
                    tag.append(0); ival.append(int(v)); fval.append(float(v)); sid.append(0)
                else:
                    tag.append(1); ival.append(0); fval.append(float(v)); sid.append(0)
        self.value_tag = np.asarray(tag or [0], np.int32)
        self.value_int = np.asarray(ival or [0], np.int64)
        self.value_float = np.asarray(fval or [0.0], np.float64)
        self.value_str = np.asarray(sid or [0], np.int32)
        self.n_values = len(tag)
        self.consts_arr = np.asarray(self.consts or [0.0], np.float64)

    def _intern(self, s):
        for k, v in self.strings.items():
            if type(k) is type(s) and k == s:
                return v
        self.strings[s] = len(self.strings)
        return self.strings[s]

    def _emit(self, node, code, space, depth) -> int:
        kind = type(node).__name__
        if kind == "Num":
            code += [OPS["num"], len(self.consts)]
            self.consts.append(float(node.value))
            return depth + 1
        if kind == "Str":
            code += [OPS["str"], self._intern(node.value)]
            return depth + 1
        if kind == "Var":
            idx = space.index_of(node.name)
            code += [OPS["cat" if space.parameters[idx].kind == "categorical" else "var"], idx]
            return depth + 1
        if kind == "Unary":
            d = self._emit(node.operand, code, space, depth)
            code += [OPS["neg" if node.op == "-" else "not"], 0]
            return d
        d1 = self._emit(node.left, code, space, depth)
        d2 = self._emit(node.right, code, space, depth + 1)
        code += [OPS[node.op], 0]
        return max(d1, d2)


# ---------------------------------------------------------------------------------------------
# chain of trees
# ---------------------------------------------------------------------------------------------
class _Node:
    __slots__ = ("value", "children", "leaf_count")

    def __init__(self, value):
        self.value, self.children, self.leaf_count = value, [], 0


@dataclass
class _Group:
    indices: tuple
    root: object
    kind: str = "tree"
    leaf_values: list | None = None


class ChainOfTrees:
    def __init__(self, space, groups):
        self.space, self.groups = space, groups

    def count(self) -> int:
        total = 1
        for g in self.groups:
            if g.kind == "tree":
                total *= g.root.leaf_count
            elif g.kind == "permutation":
                total *= math.factorial(self.space.parameters[g.indices[0]].size)
        return total

    def contains(self, cfg) -> bool:
        for g in self.groups:
            p = self.space.parameters[g.indices[0]]
            if g.kind == "real":
                if not (isinstance(cfg[g.indices[0]], (int, float)) and p.lo <= cfg[g.indices[0]] <= p.hi):
                    return False
                continue
            if g.kind == "permutation":
                v = cfg[g.indices[0]]
                if not (isinstance(v, tuple) and sorted(v) == list(range(1, p.size + 1))):
                    return False
                continue
            node = g.root
            for i in g.indices:
                node = next((ch for ch in node.children if ch.value == cfg[i]), None)
                if node is None:
                    return False
        return True

    def enumerate(self):
        import itertools

        per = []
        for g in self.groups:
            if g.kind == "real":
                raise ValueError("cannot enumerate a space with real parameters")
            if g.kind == "permutation":
                m = self.space.parameters[g.indices[0]].size
                per.append([(q,) for q in itertools.permutations(range(1, m + 1))])
            else:
                per.append(self.leaf_paths(g))
        order = [i for g in self.groups for i in g.indices]
        slot = [order.index(i) for i in range(len(self.space.parameters))]
        for combo in itertools.product(*per):
            flat = [v for path in combo for v in path]
            yield tuple(flat[s] for s in slot)

    def sample_leaf_uniform(self, n: int, rng) -> list:
        """Leaf-uniform draws consuming `rng` like the reference (constraints.py:471-523)."""
        from .space import param_sample

        if n < 1:
            raise ValueError("n must be >= 1")
        if self.count() == 0:
            raise ValueError("feasible set is empty")
        per_group = []
        for g in self.groups:
            if g.kind != "tree":
                p = self.space.parameters[g.indices[0]]
                per_group.append([(param_sample(p, rng),) for _ in range(n)])
                continue
            if g.leaf_values is None and g.root.leaf_count <= 200_000:
                g.leaf_values = self.leaf_paths(g)
            if g.leaf_values is not None:
                idx = rng.integers(g.root.leaf_count, size=n)
                per_group.append([g.leaf_values[int(i)] for i in idx])
                continue
            draws = []
            for _ in range(n):
                node, path = g.root, []
                while node.children:
                    w = np.array([c.leaf_count for c in node.children], float)
                    node = node.children[int(rng.choice(len(node.children), p=w / w.sum()))]
                    path.append(node.value)
                draws.append(tuple(path))
            per_group.append(draws)
        out = []
        dim = len(self.space.parameters)
        for k in range(n):
            cfg = [None] * dim
            for g, samples in zip(self.groups, per_group):
                for i, v in zip(g.indices, samples[k]):
                    cfg[i] = v
            out.append(tuple(cfg))
        return out

    def leaf_paths(self, g) -> list:
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


def _groups(space) -> list:
    parent = list(range(len(space.parameters)))

    def root(a):
        while parent[a] != a:
            parent[a] = parent[parent[a]]
            a = parent[a]
        return a

    for expr in space.constraints:
        ids = [space.index_of(v) for v in expr.variables]
        for other in ids[1:]:
            ra, rb = root(ids[0]), root(other)
            if ra != rb:
                parent[max(ra, rb)] = min(ra, rb)
    comps: dict = {}
    for i in range(len(space.parameters)):
        comps.setdefault(root(i), []).append(i)
    return [tuple(sorted(v)) for _, v in sorted(comps.items())]


def build_cot(space, node_cap: int = 10_000_000) -> ChainOfTrees:
    budget = [node_cap]
    groups = []
    for idx in _groups(space):
        kinds = [space.parameters[i].kind for i in idx]
        if len(idx) == 1 and kinds[0] in ("real", "permutation"):
            groups.append(_Group(idx, None, kinds[0]))
            continue
        if "real" in kinds:
            raise ValueError("real parameters may not appear in constraints")
        names = [space.parameters[i].name for i in idx]
        level = {nm: lv for lv, nm in enumerate(names)}
        checks = [[] for _ in idx]
        for expr in space.constraints:
            if expr.variables and all(v in level for v in expr.variables):
                checks[max(level[v] for v in expr.variables)].append(expr)
        doms = [domain_values(space.parameters[i]) for i in idx]
        root = _Node(None)
        budget[0] -= 1

        def grow(node, lv, bind):
            if lv == len(idx):
                node.leaf_count = 1
                return True
            for v in doms[lv]:
                bind[names[lv]] = v
                if all(eval_constraint(e, bind) is True for e in checks[lv]):
                    child = _Node(v)
                    budget[0] -= 1
                    if budget[0] < 0:
                        raise ValueError("chain-of-trees node cap exceeded")
                    if grow(child, lv + 1, bind):
                        node.children.append(child)
                        node.leaf_count += child.leaf_count
                del bind[names[lv]]
            return bool(node.children)

        grow(root, 0, {})
        groups.append(_Group(idx, root))
    return ChainOfTrees(space, groups)


@dataclass
class CotTables:
    n_groups: int
    group_kind: np.ndarray         # 0 tree, 1 real singleton, 2 permutation singleton
    group_param_begin: np.ndarray  # [n_groups + 1]
    group_params: np.ndarray
    group_root: np.ndarray
    n_nodes: int
    child_begin: np.ndarray        # [n_nodes] first child node id
    child_count: np.ndarray        # [n_nodes]
    node_value: np.ndarray         # [n_nodes] domain index of the node's value (-1 for roots)
    leaf_count: np.ndarray = None  # [n_nodes] leaves below each node (leaf-uniform generation)


def flatten_cot(cot, layout) -> CotTables:
    """Breadth-first node tables of a ChainOfTrees (the reference's or ours).  Children of a node
    get consecutive ids, in creation order = ascending domain index (constraints.py:621)."""
    kinds, pbeg, plist, roots = [], [0], [], []
    begin, count, value, leaves = [], [], [], []
    for g in cot.groups:
        plist.extend(int(i) for i in g.indices)
        pbeg.append(len(plist))
        if g.kind != "tree":
            kinds.append(1 if g.kind == "real" else 2)
            roots.append(0)
            continue
        kinds.append(0)
        base = len(value)
        roots.append(base)
        order = [(g.root, -1)]
        qi = 0
        while qi < len(order):
            node, depth = order[qi]
            qi += 1
            order.extend((ch, depth + 1) for ch in node.children)
        nxt = base + 1
        for node, depth in order:
            begin.append(nxt)
            count.append(len(node.children))
            leaves.append(int(node.leaf_count))
            nxt += len(node.children)
            value.append(-1 if depth < 0 else layout.slots[g.indices[depth]].index[node.value])
    return CotTables(len(kinds), np.asarray(kinds, np.int32), np.asarray(pbeg, np.int32),
                     np.asarray(plist or [0], np.int32), np.asarray(roots or [0], np.int32),
                     len(value), np.asarray(begin or [0], np.int32), np.asarray(count or [0], np.int32),
                     np.asarray(value or [0], np.int32), np.asarray(leaves or [0], np.int64))
