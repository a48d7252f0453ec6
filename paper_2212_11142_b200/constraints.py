"""Known constraints on the device: the bytecode compiler and the chain-of-trees tables.

The reference owns parsing (`parse_constraint`, constraints.py:153-299) and the chain of trees
(`build_cot`, constraints.py:567-643); this module consumes the objects it produces:

* `Program` walks the reference's constraint AST (node classes Num / Str / Var / Unary / BinOp,
  constraints.py:51-79) and emits the stack bytecode interpreted by feasible.cu (eval_program),
  which reproduces `_eval_node` / `eval_constraint` (constraints.py:309-368) including Python's
  int/float promotion, floor modulo, exact int-float comparison and "any ZeroDivision -> False"
  with both operands of && / || evaluated.
* `flatten_cot` turns the reference's `ChainOfTrees` (constraints.py:375-410: groups of
  `_Node` trees) into the breadth-first CSR tables of bx_set_cot.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .layout import domain_values


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
    """Breadth-first node tables of the reference's ChainOfTrees.  Children of a node
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
