"""Host-side logic on CPU: row encoding, constraint bytecode, chain-of-trees tables, sharding."""
import itertools
import math

import numpy as np
import pytest

import oracle
from golden_io import CASES, TRACES, cot_for, load, ref, to_cfg
from paper_2212_11142_b200 import scenarios
from paper_2212_11142_b200.constraints import OPS, Program, flatten_cot
from paper_2212_11142_b200.layout import SpaceLayout, pack_perm

_bt = ref()
Parameter, SearchSpace, sample_uniform, build_cot = (_bt.Parameter, _bt.SearchSpace, _bt.sample_uniform,
                                                     _bt.build_cot)


@pytest.mark.parametrize("case", CASES + TRACES)
def test_encode_decode_round_trip(case):
    meta, arr, space = load(case)
    lay = SpaceLayout(space, meta.get("use_transforms", True))
    rng = np.random.default_rng(0)
    cfgs = sample_uniform(space, 300, rng)
    assert lay.decode(lay.encode(cfgs)) == cfgs
    X = lay.features(lay.encode(cfgs))
    assert np.array_equal(X, oracle.features(space, cfgs, lay.use_transforms))


def test_permutation_packing_preserves_tuple_order():
    perms = list(itertools.permutations(range(1, 6)))
    packed = [pack_perm(p, 5) for p in perms]
    assert sorted(range(len(perms)), key=lambda i: packed[i]) == sorted(range(len(perms)),
                                                                         key=lambda i: perms[i])


def test_categorical_rank_is_python_order():
    sp = SearchSpace([Parameter.categorical("c", ["zeta", "alpha", "Mid", "beta"])])
    lay = SpaceLayout(sp)
    ranks = list(lay.rank_lut[:4])
    labels = list(sp.parameters[0].values)
    assert [labels[i] for i in sorted(range(4), key=lambda i: ranks[i])] == sorted(labels)


def test_real_grid_coordinates_follow_numeric_coords():
    p = Parameter.real("x", 0.5, 9.5, transform="log")
    lay = SpaceLayout(SearchSpace([p]))
    step = (9.5 - 0.5) / 63
    grid = [0.5 + j * step for j in range(64)]
    assert np.array_equal(lay.coord_lut[:64], oracle.gp.coords(p, grid))


# ---- bytecode: a host emulation of feasible.cu eval_program ----------------------------------
def run_program(prog: Program, space, lay: SpaceLayout, cfg):
    row = lay.encode([cfg])[0]
    inv = {v: k for k, v in OPS.items()}
    offs, o = [], 0
    for p in space.parameters:
        offs.append(o)
        o += 0 if p.kind in ("real", "permutation") else len(p.values if p.kind != "integer"
                                                             else range(p.lo, p.hi + 1))
    results = []
    for c in range(prog.n):
        code = prog.code[prog.prog_begin[c]:prog.prog_begin[c + 1]]
        st = []
        try:
            for pc in range(0, len(code), 2):
                op, arg = inv[int(code[pc])], int(code[pc + 1])
                if op == "num":
                    st.append(("f", prog.consts[arg]))
                elif op == "str":
                    st.append(("s", arg))
                elif op in ("var", "cat"):
                    p = space.parameters[arg]
                    d = lay.params[arg]
                    if p.kind == "real":
                        st.append(("f", float(row[d.word:d.word + 2].view(np.float64)[0])))
                    else:
                        i = offs[arg] + int(row[d.word])
                        if op == "cat":
                            st.append(("s", int(prog.value_str[i])))
                        elif prog.value_tag[i]:
                            st.append(("f", float(prog.value_float[i])))
                        else:
                            st.append(("i", int(prog.value_int[i])))
                elif op == "neg":
                    t, v = st.pop()
                    st.append((t, -v))
                elif op == "not":
                    st.append(("b", not st.pop()[1]))
                elif op in ("&&", "||"):
                    b, a = st.pop()[1], st.pop()[1]
                    st.append(("b", (a and b) if op == "&&" else (a or b)))
                elif op in ("+", "-", "*", "/", "%"):
                    (tb, b), (ta, a) = st.pop(), st.pop()
                    if op == "/":
                        if float(b) == 0.0:
                            raise ZeroDivisionError
                        st.append(("f", float(a) / float(b)))
                    elif ta == tb == "i":
                        st.append(("i", {"+": a + b, "-": a - b, "*": a * b}[op] if op != "%" else a % b))
                    else:
                        x, y = float(a), float(b)
                        if op == "%":
                            if y == 0.0:
                                raise ZeroDivisionError
                            r = math.fmod(x, y)
                            r = (r + y if r and (y < 0) != (r < 0) else r) if r else math.copysign(0.0, y)
                            st.append(("f", r))
                        else:
                            st.append(("f", {"+": x + y, "-": x - y, "*": x * y}[op]))
                else:
                    (tb, b), (ta, a) = st.pop(), st.pop()
                    if "s" in (ta, tb):
                        eq = ta == tb and a == b
                        st.append(("b", eq if op == "==" else not eq))
                    else:
                        st.append(("b", {"<": a < b, "<=": a <= b, ">": a > b, ">=": a >= b,
                                         "==": a == b, "!=": a != b}[op]))
            results.append(bool(st[-1][1]))
        except ZeroDivisionError:
            results.append(False)
    return results


TRICKY = [
    "a % b == 1", "a / b >= 1", "-a + b * 2 <= 3.5", "(a - 3) % 4 != 0 || c == 'x'",
    "!(a > 2) && b != 0", "c != 'z' && (a * a + b * b) % 3.0 == 1", "r * 2 < a || r / (b - 2) > 0.1",
    "o % 2.5 == 0.5 || o / a > 1", "c == 'y' || c == 'nope'", "a % -3 == -1", "-(a % 3) == 0 && o >= 0.5",
]


def tricky_space():
    return SearchSpace([Parameter.integer("a", -4, 6), Parameter.integer("b", -3, 3),
                        Parameter.categorical("c", ["x", "y", "z"]), Parameter.real("r", -1.0, 1.0),
                        Parameter.ordinal("o", [0.5, 1, 2.5, 4])], TRICKY)


def test_bytecode_matches_python_semantics():
    sp = tricky_space()
    lay = SpaceLayout(sp)
    prog = Program(sp, lay)
    rng = np.random.default_rng(3)
    for cfg in sample_uniform(sp, 3000, rng):
        want = [oracle.eval_constraint(e, sp.as_dict(cfg)) is True for e in sp.constraints]
        assert run_program(prog, sp, lay, cfg) == want, cfg


def _walk_tables(t, lay, space, cfg):
    row = lay.encode([cfg])[0]
    for g in range(t.n_groups):
        params = t.group_params[t.group_param_begin[g]:t.group_param_begin[g + 1]]
        if t.group_kind[g] != 0:
            continue
        node = t.group_root[g]
        for k in params:
            x = int(row[lay.params[int(k)].word])
            kids = range(t.child_begin[node], t.child_begin[node] + t.child_count[node])
            hit = [c for c in kids if t.node_value[c] == x]
            if not hit:
                return False
            node = hit[0]
    return True


@pytest.mark.parametrize("case", ["C2", "C3"])
def test_flattened_cot_tables_walk_like_contains(case):
    meta, arr, space = load(case)
    lay = SpaceLayout(space)
    t = flatten_cot(cot_for(case), lay)
    probe = [to_cfg(space, c) for c in meta["cot_probe"][:600]]
    got = np.array([_walk_tables(t, lay, space, c) for c in probe])
    assert np.array_equal(got, arr["cot_mask"][:600])
    for u in range(t.n_nodes):  # siblings sorted ascending (binary search on the device)
        vals = t.node_value[t.child_begin[u]:t.child_begin[u] + t.child_count[u]]
        assert np.all(np.diff(vals) > 0)


def test_shard_ranges_cover_pool():
    from paper_2212_11142_b200.distributed import shard_range
    for q in (1, 7, 1000, 1 << 20):
        for world in (1, 2, 3, 8):
            spans = [shard_range(q, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == q
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))


def test_scenario_spaces_build_and_sample():
    for name in scenarios.SCENARIOS:
        sp = scenarios.build_space(name, _bt.space)
        lay = SpaceLayout(sp)
        spec = SpaceLayout(scenarios.build_space(name))  # the reference-free descriptor
        assert np.array_equal(spec.coord_lut, lay.coord_lut) and spec.row_words == lay.row_words
        rows = scenarios.sample_rows_uniform(lay, 500, np.random.default_rng(0))
        cfgs = lay.decode(rows)
        assert lay.decode(lay.encode(cfgs)) == cfgs
        if sp.constraints:
            cot = build_cot(sp)
            rows = scenarios.sample_rows_cot(lay, cot, 500, np.random.default_rng(1))
            assert all(cot.contains(c) for c in lay.decode(rows))
