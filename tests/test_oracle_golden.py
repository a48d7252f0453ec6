"""Pin the oracle against the reference's own outputs (tests/golden, made by make_golden.py)."""
import numpy as np
import pytest

import oracle
from golden_io import CASES, TRACES, cot_for, load, oracle_model, to_cfg


@pytest.mark.parametrize("case", CASES)
def test_posterior_matches_reference(case):
    meta, arr, space = load(case)
    og, _ = oracle_model(meta, arr, space)
    cands = [to_cfg(space, c) for c in meta["cands"]]
    mean, var = oracle.predict(og, cands)
    np.testing.assert_allclose(mean, arr["mean"], rtol=1e-9, atol=1e-9)
    np.testing.assert_allclose(var, arr["var"], rtol=1e-6, atol=1e-9 * float(np.max(arr["var"])))


@pytest.mark.parametrize("case", CASES)
def test_scores_match_reference(case):
    meta, arr, space = load(case)
    og, of = oracle_model(meta, arr, space)
    cands = [to_cfg(space, c) for c in meta["cands"]]
    values, probs = oracle.scores(og, of, cands, meta["f_best"], meta["eps_f"])
    assert np.array_equal(probs, arr["probs"])  # forest probabilities: bit-exact
    assert np.array_equal(np.isinf(values), np.isinf(arr["values"]))
    fin = np.isfinite(values)
    np.testing.assert_allclose(values[fin], arr["values"][fin], rtol=1e-6,
                               atol=1e-9 * float(np.max(np.abs(arr["values"][fin]), initial=1.0)))


@pytest.mark.parametrize("case", [c for c in CASES if c not in ("C1", "C2")])
def test_forest_single_config_order(case):
    meta, arr, space = load(case)
    _, of = oracle_model(meta, arr, space)
    cands = [to_cfg(space, c) for c in meta["cands"]]
    X = oracle.features(space, cands[:256], of.use_transforms)
    assert np.array_equal(X, arr["rf_X"])
    single = np.array([oracle.predict_proba(of, [c])[0] for c in cands[:64]])
    assert np.array_equal(single, arr["probs_q1"])


@pytest.mark.parametrize("case", CASES)
def test_neighbors_match_reference(case):
    meta, arr, space = load(case)
    cot = cot_for(case)
    for start, plain in zip(meta["nbr_starts"], meta["nbr_plain"]):
        got = oracle.neighbors(space, to_cfg(space, start))
        assert got == [to_cfg(space, c) for c in plain]
    if cot is not None:
        for start, filt in zip(meta["nbr_starts"], meta["nbr_cot"]):
            got = oracle.neighbors(space, to_cfg(space, start), cot)
            assert got == [to_cfg(space, c) for c in filt]


@pytest.mark.parametrize("case", ["C2", "C3"])
def test_feasible_set_masks(case):
    meta, arr, space = load(case)
    cot = cot_for(case)
    probe = [to_cfg(space, c) for c in meta["cot_probe"]]
    assert cot.count() == meta["cot_count"]
    mask = np.array([oracle.cot_contains(cot, c) for c in probe])
    assert np.array_equal(mask, arr["cot_mask"])
    cons = np.array([[oracle.eval_constraint(e, space.as_dict(c)) is True for e in space.constraints]
                     for c in probe])
    assert np.array_equal(cons, arr["cons_mask"])


@pytest.mark.parametrize("case", CASES)
def test_pairwise_and_lml(case):
    meta, arr, space = load(case)
    og, _ = oracle_model(meta, arr, space)
    sq = oracle.pairwise_sq(space, og.configs, og.configs, og.use_transforms)
    assert np.array_equal(sq[:, :16, :16], arr["sq_train_head"])
    lml = oracle.coarse_lml(sq, arr["lml_z"], arr["lml_thetas"])
    assert np.array_equal(np.isfinite(lml), np.isfinite(arr["lml"]))
    fin = np.isfinite(lml)
    np.testing.assert_allclose(lml[fin], arr["lml"][fin], rtol=1e-9, atol=1e-7)
    np.testing.assert_allclose(oracle.prior_term(arr["lml_thetas"]), arr["lml_prior"], rtol=1e-13)


@pytest.mark.parametrize("case", CASES)
def test_lml_core_value_and_gradient(case):
    meta, arr, space = load(case)
    og, _ = oracle_model(meta, arr, space)
    sq = oracle.pairwise_sq(space, og.configs, og.configs, og.use_transforms)
    for t, v, g, ok in zip(arr["lml_thetas"][:8], arr["core_value"], arr["core_grad"], arr["core_ok"]):
        if not ok:
            with pytest.raises(np.linalg.LinAlgError):
                oracle.lml_core(sq, arr["lml_z"], np.exp(t[0]), np.exp(t[1]), np.exp(t[2:]), True)
            continue
        val, grad = oracle.lml_core(sq, arr["lml_z"], np.exp(t[0]), np.exp(t[1]), np.exp(t[2:]), True)
        assert val == pytest.approx(v, rel=1e-9, abs=1e-7)
        np.testing.assert_allclose(grad, g, rtol=1e-6, atol=1e-6 * max(1.0, np.abs(g).max()))


@pytest.mark.parametrize("case", ["C1", "C2", "C3"])
def test_selection_matches_reference(case):
    meta, arr, space = load(case)
    og, of = oracle_model(meta, arr, space)
    pool = [to_cfg(space, c) for c in meta["sel_pool"]]
    evaluated = {to_cfg(space, c) for c in meta["evaluated"]}
    got = oracle.optimize(og, of, space, pool, meta["f_best"], meta["eps_f"], evaluated, cot_for(case))
    assert got == to_cfg(space, meta["sel_chosen"])


@pytest.mark.parametrize("trace", TRACES)
def test_engine_trace_selections(trace):
    meta, arr, space = load(trace)
    cot = cot_for(trace)
    from golden_io import Case  # noqa: F401
    for i, it in enumerate(meta["iters"]):
        og, of = oracle_model(it, arr, space, prefix=f"it{i}_")
        pool = [to_cfg(space, c) for c in it["pool"]]
        ev = {to_cfg(space, c) for c in it["evaluated"]}
        got = oracle.optimize(og, of, space, pool, it["f_best"], it["eps_f"], ev, cot)
        assert got == to_cfg(space, it["chosen"]), f"iteration {i}"
