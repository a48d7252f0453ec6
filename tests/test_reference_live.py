"""Live cross-checks against the reference package (build container only: /root/reference).

These pin the host pieces (coordinate tables, encoded-row samplers) and the oracle on fresh
inputs beyond the committed golden vectors.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.reference

@pytest.fixture(scope="module")
def ref():
    from golden_io import ref as load_ref
    return load_ref()


@pytest.mark.parametrize("name", ["C2", "C3"])
def test_encoded_row_samplers_stay_inside_the_reference_chain_of_trees(ref, name):
    """scenarios.sample_rows_cot draws leaf-uniform rows from the reference's chain of trees."""
    from paper_2212_11142_b200 import scenarios
    from paper_2212_11142_b200.layout import SpaceLayout
    rs = scenarios.build_space(name, ref.space)
    cot = ref.build_cot(rs)
    lay = SpaceLayout(rs)
    cfgs = lay.decode(scenarios.sample_rows_cot(lay, cot, 3000, np.random.default_rng(5)))
    assert all(cot.contains(c) for c in cfgs)


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
    ms = rs
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
