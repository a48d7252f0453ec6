"""Neighbour sets, chain-of-trees membership and constraint evaluation restated.  Test-only.

space.py:258-309 (neighbors), constraints.py:413-430 (ChainOfTrees.contains),
constraints.py:309-368 (_eval_node / eval_constraint).
"""
from __future__ import annotations


def _moves(p, v) -> list:
    if p.kind in ("integer",):
        return [v + d for d in (-1, 1) if p.lo <= v + d <= p.hi]
    if p.kind == "ordinal":
        i = list(p.values).index(v)
        return [p.values[j] for j in (i - 1, i + 1) if 0 <= j < len(p.values)]
    if p.kind == "categorical":
        return [w for w in p.values if w != v]
    if p.kind == "real":
        step = (p.hi - p.lo) / 63
        i = round((v - p.lo) / step)
        return [p.lo + j * step for j in (i - 1, i + 1) if 0 <= j < 64 and p.lo + j * step != v]
    out = []
    for a in range(p.size):
        for b in range(a + 1, p.size):
            w = list(v)
            w[a], w[b] = w[b], w[a]
            out.append(tuple(w))
    return out


def neighbors(space, cfg, cot=None) -> list:
    out, seen = [], set()
    for k, p in enumerate(space.parameters):
        for v in _moves(p, cfg[k]):
            c = cfg[:k] + (v,) + cfg[k + 1:]
            if c in seen:
                continue
            seen.add(c)
            if cot is None or cot_contains(cot, c):
                out.append(c)
    return out


def cot_contains(cot, cfg) -> bool:
    for g in cot.groups:
        i0 = g.indices[0]
        p = cot.space.parameters[i0]
        if g.kind == "real":
            if not (isinstance(cfg[i0], (int, float)) and p.lo <= cfg[i0] <= p.hi):
                return False
        elif g.kind == "permutation":
            v = cfg[i0]
            if not (isinstance(v, tuple) and sorted(v) == list(range(1, p.size + 1))):
                return False
        else:
            node = g.root
            for i in g.indices:
                node = next((c for c in node.children if c.value == cfg[i]), None)
                if node is None:
                    return False
    return True


class _Open(Exception):
    pass


def _value(node, env):
    name = type(node).__name__
    if name in ("Num", "Str"):
        return node.value
    if name == "Var":
        if node.name not in env:
            raise _Open
        return env[node.name]
    if name == "Unary":
        x = _value(node.operand, env)
        return (not x) if node.op == "!" else -x
    a, b = _value(node.left, env), _value(node.right, env)
    op = node.op
    if op in ("&&", "||"):
        return (a and b) if op == "&&" else (a or b)
    if op == "+":
        return a + b
    if op == "-":
        return a - b
    if op == "*":
        return a * b
    if op == "/":
        return a / b
    if op == "%":
        return a % b
    return {"<": a < b, "<=": a <= b, ">": a > b, ">=": a >= b, "==": a == b, "!=": a != b}[op]


def eval_constraint(expr, env):
    try:
        return bool(_value(expr.root, env))
    except _Open:
        return "not-yet-decidable"
    except (ZeroDivisionError, OverflowError):
        return False
