"""Live cross-checks against the reference package (build container only: /root/reference).

These pin the standalone host pieces (parser, chain of trees, RNG-consuming samplers, coordinate
tables) and the oracle on fresh inputs beyond the committed golden vectors.
"""
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.reference

REF = "/root/reference/pkg/src"


@pytest.fixture(scope="module")
def ref():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import boxtune
    return boxtune


CORPUS = ["p1 >= p2", "p5 >= 2*p4", "p1 >= ", "p1 >= zz", "p1 + (p2 > 1)", "(p1 + 2) * 3 == 9",
          "-p1 + 1 <= 0", "p1 >= p2 &&", "p1 % 0 == 1 || p3 != 4", "1e3 > p1", "p1 @ 2", "'a' == p1",
          "!(p1 > 2)", "p1 > 2 > 3", "((p1)", "p1 >= 2.5e-1 && !(p4 < p5) || p3 == 1"]


def test_parser_agrees(ref):
    from paper_2212_11142_b200 import constraints as mine
    from paper_2212_11142_b200.space import Parameter, SearchSpace
    params = [("p1", [2, 4]), ("p2", [2, 4]), ("p3", [1, 4]), ("p4", [1, 2, 4]), ("p5", [2, 4, 8])]
    rs = ref.SearchSpace([ref.Parameter.ordinal(n, v) for n, v in params])
    ms = SearchSpace([Parameter.ordinal(n, v) for n, v in params])
    for text in CORPUS:
        try:
            r = ref.parse_constraint(text, rs)
            r_err = None
        except ref.ConstraintError as e:
            r, r_err = None, e.position
        try:
            m = mine.parse_constraint(text, ms)
            m_err = None
        except mine.ConstraintError as e:
            m, m_err = None, e.position
        assert (r is None) == (m is None), text
        assert r_err == m_err, text
        if r is not None:
            assert r.variables == m.variables


@pytest.mark.parametrize("name", ["C2", "C3"])
def test_cot_and_samplers_agree(ref, name):
    from paper_2212_11142_b200 import scenarios
    from paper_2212_11142_b200.constraints import build_cot
    from paper_2212_11142_b200.space import sample_uniform
    rs = scenarios.build_space(name, ref.space)
    ms = scenarios.build_space(name)
    rc, mc = ref.build_cot(rs), build_cot(ms)
    assert rc.count() == mc.count()
    a = rc.sample_leaf_uniform(3000, np.random.default_rng(5))
    b = mc.sample_leaf_uniform(3000, np.random.default_rng(5))
    assert a == b
    u1 = ref.sample_uniform(rs, 2000, np.random.default_rng(6))
    u2 = sample_uniform(ms, 2000, np.random.default_rng(6))
    assert u1 == u2
    assert [rc.contains(c) for c in u1] == [mc.contains(c) for c in u2]


def test_layout_coordinates_are_the_reference_ones(ref):
    from boxtune.surrogate import _numeric_coords
    from paper_2212_11142_b200 import scenarios
    from paper_2212_11142_b200.layout import SpaceLayout, domain_values
    for name in ("C2", "C3", "C5"):
        rs = scenarios.build_space(name, ref.space)
        lay = SpaceLayout(scenarios.build_space(name))
        for k, p in enumerate(rs.parameters):
            d = lay.params[k]
            if p.kind in ("integer", "ordinal"):
                want = _numeric_coords(p, domain_values(p), True)
                assert np.array_equal(lay.coord_lut[d.coord:d.coord + d.size], want)


def test_oracle_matches_live_reference_on_fresh_inputs(ref):
    import oracle
    from boxtune import acquisition as A
    from boxtune import feasibility as F
    from boxtune import surrogate as S
    from paper_2212_11142_b200 import scenarios
    rng = np.random.default_rng(123)
    rs = scenarios.build_space("C5", ref.space)
    ms = scenarios.build_space("C5")
    train = list(dict.fromkeys(ref.sample_uniform(rs, 25, rng)))
    y = [scenarios.objective("C5", c) for c in train]
    gp = S.gp_fit(rs, train, y, rng)
    labels = [c[3] < 9 for c in train]
    feas = F.rf_fit(rs, train, labels, rng)
    cands = ref.sample_uniform(rs, 800, rng)
    ctx = A.AcquisitionContext(gp=gp, feas=feas, best_feasible_value=min(y), eps_f=0.2, rng=rng)
    v, p = A._scores(ctx, cands)
    og = oracle.OracleGP(ms, train, gp.hyperparameters.outputscale, gp.hyperparameters.noise_variance,
                         gp.hyperparameters.lengthscales, L=gp._cho[0], alpha=gp.alpha, y_mean=gp.y_mean,
                         y_std=gp.y_std, log_objective=gp.log_objective)
    of = oracle.OracleForest(feas.feature, feas.threshold, feas.left, feas.right, feas.value,
                             feas.roots, feas.max_depth, ms)
    ov, op = oracle.scores(og, of, cands, min(y), 0.2)
    assert np.array_equal(op, p)
    fin = np.isfinite(v)
    np.testing.assert_allclose(ov[fin], v[fin], rtol=1e-7, atol=1e-12)
    for c in cands[:20]:
        assert oracle.neighbors(ms, c) == ref.neighbors(rs, c)
