"""Device-side candidate generation (§8f rank 1): membership exact, distribution statistical
(the reference's own sampler tests use chi-square: test_constraints.py:238-251, test_space.py:182-195)."""
import itertools

import numpy as np
import pytest
import torch
from scipy.stats import chi2

from golden_io import cot_for, load, model, ref
from paper_2212_11142_b200.device import Scorer

_bt = ref()
Parameter, SearchSpace, build_cot = _bt.Parameter, _bt.SearchSpace, _bt.build_cot

pytestmark = pytest.mark.gpu


def rows_np(t):
    return t.cpu().numpy().view(np.uint32)


def chi2_ok(counts, expected):
    stat = float(((counts - expected) ** 2 / expected).sum())
    return stat < chi2.ppf(0.9999, df=len(counts) - 1)


def test_uniform_marginals_and_permutations():
    sp = SearchSpace([Parameter.ordinal("o", [1, 2, 4, 8, 16]), Parameter.categorical("c", ["x", "y", "z"]),
                      Parameter.integer("i", -3, 3), Parameter.permutation("p", 3, "kendall"),
                      Parameter.real("r", 0.5, 4.0, transform="log")])
    sc = Scorer()
    lay = sc.set_space(sp)
    q = 600_000
    cfgs = lay.decode(rows_np(sc.generate(q, seed=11)))
    for k, p in enumerate(sp.parameters[:3]):
        dom = list(p.values) if p.kind != "integer" else list(range(p.lo, p.hi + 1))
        counts = np.array([sum(1 for c in cfgs if c[k] == v) for v in dom], float)
        assert chi2_ok(counts, np.full(len(dom), q / len(dom))), p.name
    perms = list(itertools.permutations((1, 2, 3)))
    counts = np.array([sum(1 for c in cfgs if c[3] == pm) for pm in perms], float)
    assert chi2_ok(counts, np.full(6, q / 6))
    r = np.array([c[4] for c in cfgs])
    assert r.min() >= 0.5 and r.max() <= 4.0
    assert abs(np.mean(r < 2.25) - (2.25 - 0.5) / 3.5) < 0.005
    sc.close()


def test_leaf_uniform_over_chain_of_trees():
    sp = SearchSpace([Parameter.ordinal("a", [1, 2, 4, 8]), Parameter.ordinal("b", [1, 2, 4, 8]),
                      Parameter.categorical("c", ["u", "v"])], ["a >= b", "c == 'u' || a > 2"])
    cot = build_cot(sp)
    leaves = list(cot.enumerate())
    sc = Scorer()
    lay = sc.set_space(sp)
    sc.set_cot(cot)
    q = 400_000
    rows = sc.generate(q, seed=5, mode=1)
    assert bool(sc.cot_contains(rows).all())
    cfgs = lay.decode(rows_np(rows))
    counts = np.array([sum(1 for c in cfgs if c == leaf) for leaf in leaves], float)
    assert counts.sum() == q
    assert chi2_ok(counts, np.full(len(leaves), q / len(leaves)))
    sc.close()


def test_path_biased_over_chain_of_trees():
    """mode 2 = sample_path_biased (constraints.py:478-501): a uniform child at every level, so a
    leaf's probability is the product of 1 / (children) along its path; the reference's own
    sampler (same tree) gives the same distribution."""
    sp = SearchSpace([Parameter.ordinal("a", [1, 2, 4, 8]), Parameter.ordinal("b", [1, 2, 4, 8]),
                      Parameter.categorical("c", ["u", "v"])], ["a >= b", "c == 'u' || a > 2"])
    cot = build_cot(sp)
    (g,) = [g for g in cot.groups if g.kind == "tree"]
    probs = {}

    def walk(node, acc, pr):
        if not node.children:
            probs[tuple(acc)] = pr
            return
        for ch in node.children:
            walk(ch, acc + [ch.value], pr / len(node.children))
    walk(g.root, [], 1.0)
    leaves = sorted(probs)
    sc = Scorer()
    lay = sc.set_space(sp)
    sc.set_cot(cot)
    q = 400_000
    rows = sc.generate(q, seed=9, mode=2)
    assert bool(sc.cot_contains(rows).all())
    cfgs = lay.decode(rows_np(rows))
    pos = {leaf: i for i, leaf in enumerate(leaves)}
    counts = np.zeros(len(leaves))
    for c in cfgs:
        counts[pos[tuple(c[i] for i in g.indices)]] += 1
    expected = np.array([probs[leaf] for leaf in leaves]) * q
    assert chi2_ok(counts, expected)
    ref_draw = cot.sample_path_biased(20_000, np.random.default_rng(3))
    rc = np.zeros(len(leaves))
    for c in ref_draw:
        rc[pos[tuple(c[i] for i in g.indices)]] += 1
    assert chi2_ok(rc, np.array([probs[leaf] for leaf in leaves]) * 20_000)
    sc.close()


def test_generation_is_counter_based():
    meta, arr, space = load("C3")
    sc = Scorer()
    sc.set_space(space)
    sc.set_cot(cot_for("C3"))
    whole = rows_np(sc.generate(50_000, seed=3, mode=1))
    part = rows_np(sc.generate(1_000, seed=3, mode=1, index_base=31_000))
    assert np.array_equal(whole[31_000:32_000], part)
    assert not np.array_equal(whole, rows_np(sc.generate(50_000, seed=4, mode=1)))
    sc.close()


def test_score_generated_matches_materialised_pool():
    meta, arr, space = load("C3")
    gp, feas = model(meta, arr, space)
    sc = Scorer()
    sc.set_gp(gp)
    sc.set_forest(feas)
    sc.set_cot(cot_for("C3"))
    f = gp.objective_to_model(meta["f_best"])
    q = (1 << 22) + 1_003  # crosses the 2^22 generation chunk
    a = sc.score_generated(q, seed=9, f_model=f, eps_f=meta["eps_f"], k=10, mode=1)
    rows = sc.generate(q, seed=9, mode=1)
    b, _, _ = sc.score(rows, f, meta["eps_f"], k=10)
    assert (a.n_scored, a.n_finite) == (b.n_scored, b.n_finite) == (q, b.n_finite)
    assert [c.index for c in a.top] == [c.index for c in b.top]
    assert [c.value for c in a.top] == [c.value for c in b.top]
    assert all(np.array_equal(x.row, y.row) for x, y in zip(a.top, b.top))
    assert a.best.index == b.best.index
    sc.close()
