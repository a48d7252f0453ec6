"""The drop-in through the REAL reference on the GPU.

The unmodified reference package (oracle/_ref, shipped by oracle/ship_ref.sh) runs complete tuning
runs - `run_bo_loop` (engine.py:294-331) with its own gp_fit, rf_fit, chain of trees, samplers and
threshold draws - once as shipped and once with `patch.install(boxtune)` routing the hot path to
the GPU.  The histories (every configuration, objective, feasibility flag, phase and timestamp) and
the CSV artifact must be identical: the reference's own determinism criteria
(test_engine.py:130-134, test_acceptance.py:318-329) applied across the two implementations.

Modes: whole_path=False keeps the reference's optimize_acquisition and patches _scores /
neighbors / predict_batch / predict_proba_batch (the per-call parity mode); whole_path=True also
replaces optimize_acquisition (fused top-k, trackers, lockstep climb); lml=True additionally moves
the hyperparameter-fit objectives to the GPU.
"""
import functools
import math

import numpy as np
import pytest

from golden_io import ref

pytestmark = pytest.mark.gpu

RUNS = [("quadratic-mixed", 3, None), ("hidden-ridge", 5, None), ("perm-assignment", 7, 30)]


def _scenario(bt, bench, budget, seed, **opts):
    return bt.Scenario(name=bench.name, space=bench.space, budget=budget, seed=seed,
                       options=bt.EngineOptions(**opts))


def _run(bt, bench, budget, seed, **opts):
    return bt.run_bo_loop(_scenario(bt, bench, budget, seed, **opts), bench,
                          np.random.default_rng(seed))


def _patched(bt, fn, **kw):
    from paper_2212_11142_b200.patch import install
    undo = install(bt, **kw)
    try:
        return fn()
    finally:
        undo()


def _first_divergence(a, b):
    for i, (x, y) in enumerate(zip(a, b)):
        if x != y:
            return i, x, y
    return (min(len(a), len(b)), None, None) if len(a) != len(b) else None


@pytest.mark.parametrize("whole_path", [False, True])
@pytest.mark.parametrize("name,seed,budget", RUNS)
def test_patched_bo_loop_history_is_the_reference_history(name, seed, budget, whole_path):
    bt = ref()
    bench = bt.builtin(name)
    budget = budget or bench.default_budget
    want = _run(bt, bench, budget, seed)
    got = _patched(bt, lambda: _run(bt, bench, budget, seed), whole_path=whole_path)
    assert _first_divergence(got.history, want.history) is None, _first_divergence(got.history,
                                                                                   want.history)
    assert sum(r.phase == "bo" for r in got.history) > 0


def test_patched_run_with_gpu_lml_objectives():
    """lml=True: the coarse LML and the L-BFGS-B objective run on the GPU too.  Their values are
    FP64 but not bit-identical to LAPACK's, so the fitted hyperparameters may differ in the last
    bits; the history must still match the reference's on this run (the argsort of 64 coarse
    values and the L-BFGS-B iterates are insensitive at 1e-12 relative)."""
    bt = ref()
    bench = bt.builtin("quadratic-mixed")
    want = _run(bt, bench, 30, 3)
    got = _patched(bt, lambda: _run(bt, bench, 30, 3), whole_path=True, lml=True)
    assert _first_divergence(got.history, want.history) is None, _first_divergence(got.history,
                                                                                   want.history)


def test_csv_artifact_byte_identical(tmp_path):
    """test_acceptance.py:318-329 (criterion 10) across implementations."""
    bt = ref()
    b = bt.builtin("quadratic-mixed")
    blobs = []
    for patched in (False, True):
        sc = bt.Scenario(name="det", space=b.space, budget=20, seed=11)
        path = tmp_path / f"run{int(patched)}.csv"

        def go():
            with bt.ResultsWriter(path, b.space) as w:
                bt.run_bo_loop(sc, b, np.random.default_rng(sc.seed), on_record=w.write)
        if patched:
            _patched(bt, go)
        else:
            go()
        blobs.append(path.read_bytes())
    assert blobs[0] == blobs[1]


def _branin(bt):
    P = bt.Parameter
    space = bt.SearchSpace([P.real("x1", -5.0, 10.0), P.real("x2", 0.0, 15.0)])

    def f(cfg):
        x1, x2 = cfg
        a, b, c, r, s, t = 1.0, 5.1 / (4 * math.pi ** 2), 5 / math.pi, 6.0, 10.0, 1 / (8 * math.pi)
        return a * (x2 - b * x1 ** 2 + c * x1 - r) ** 2 + s * (1 - t) * math.cos(x1) + s
    return bt.Benchmark("branin", space, f, default_budget=50)


def test_branin_c1_end_to_end():
    """BASELINE.json configs[0] (C1): Branin, 10 DoE + 40 BO iterations, 10k-candidate pool,
    log objective on (min 0.397887 > 0).  The engine binds n_candidates at definition time
    (acquisition.py:155), so both runs wrap their optimize_acquisition with n_candidates=10_000."""
    bt = ref()
    bench = _branin(bt)
    eng = bt.engine

    def run():
        inner = eng.optimize_acquisition
        eng.optimize_acquisition = functools.partial(inner, n_candidates=10_000)
        try:
            sc = bt.Scenario(name="branin", space=bench.space, budget=50, seed=21, doe_size=10)
            return bt.run_bo_loop(sc, bench, np.random.default_rng(21))
        finally:
            eng.optimize_acquisition = inner
    want = run()
    got = _patched(bt, run)
    assert _first_divergence(got.history, want.history) is None, _first_divergence(got.history,
                                                                                   want.history)
    assert sum(r.phase == "bo" for r in got.history) == 40


def _one_neighbour_space(bt):
    """A chain of trees in which (1, 1) has exactly one valid neighbour: a + b == 5 || a == 1
    admits (1, 2) from (1, 1) but not (2, 1); (4, 1) has none, (1, 3) three."""
    P = bt.Parameter
    return bt.SearchSpace([P.integer("a", 1, 4), P.integer("b", 1, 4)], ["a + b == 5 || a == 1"])


def test_single_neighbour_lists_use_the_q1_forest_order():
    """bx_climb scores a start whose CoT-filtered neighbour list has length one with the forest's
    q == 1 (pairwise) summation order, as the reference's per-start _scores call does
    (feasibility.py:89); longer lists keep the sequential order.  The proposal equals the
    reference's optimize_acquisition for every evaluated set / RNG seed tried."""
    from golden_io import Ctx
    from paper_2212_11142_b200 import acquisition as A
    from paper_2212_11142_b200.device import scorer
    bt = ref()
    sp = _one_neighbour_space(bt)
    cot = bt.build_cot(sp)
    rng = np.random.default_rng(0)
    cfgs = list(cot.enumerate())
    y = [1.0 + 0.3 * a + 0.1 * b for a, b in cfgs]
    gp = bt.gp_fit(sp, cfgs, y, rng)
    feas = bt.rf_fit(sp, cfgs + [(2, 2), (3, 3)], [True] * len(cfgs) + [False, False], rng)
    sc = scorer()
    A._prepare(Ctx(gp, feas, min(y), 0.0), sc, evaluated=False)
    sc.set_cot(cot)
    nb, valid = sc.neighbors(sc.to_device(sc.layout.encode([(1, 1), (1, 3), (4, 1)])), use_cot=True)
    counts = valid.bool().view(3, sc.n_slots).sum(1).cpu().numpy()
    assert list(counts) == [1, 3, 0]
    for n_ev, seed in ((0, 4), (1, 5), (2, 4), (3, 6), (5, 7)):
        evaluated = set(cfgs[:n_ev])
        want = bt.optimize_acquisition(
            bt.AcquisitionContext(gp=gp, feas=feas, best_feasible_value=min(y), eps_f=0.0,
                                  rng=np.random.default_rng(seed), evaluated=evaluated), sp, cot)
        got = A.optimize_acquisition(Ctx(gp, feas, min(y), 0.0, np.random.default_rng(seed), evaluated), sp, cot)
        assert got == want, (n_ev, seed)


def test_device_climb_matches_reference_climb_with_many_starts():
    """n_starts above the fused top-k (BX_MAX_K = 32): the starts come from a host stable argsort
    of the pool values and climb in chunks of 32 on the device; the proposal equals the
    reference's."""
    from golden_io import Ctx, load, ref_model, to_cfg
    from paper_2212_11142_b200 import acquisition as A
    bt = ref()
    meta, arr, space = load("mixed_fit")
    gp, feas = ref_model(meta, arr, space)
    cands = [to_cfg(space, c) for c in meta["cands"][:800]]
    evaluated = {to_cfg(space, c) for c in meta["evaluated"]}
    for n_starts in (1, 10, 40):
        want = bt.optimize_acquisition(
            bt.AcquisitionContext(gp=gp, feas=feas, best_feasible_value=meta["f_best"], eps_f=meta["eps_f"],
                                  rng=np.random.default_rng(0), evaluated=evaluated), space, None,
            sample_fn=lambda n, r: cands, n_starts=n_starts)
        got = A.optimize_acquisition(Ctx(gp, feas, meta["f_best"], meta["eps_f"], np.random.default_rng(0), evaluated),
                                     space, None, sample_fn=lambda n, r: cands, n_starts=n_starts)
        assert got == want, n_starts


@pytest.mark.parametrize("cap", [1, 2, 3, 5, 7, 50])
def test_device_climb_step_cap_matches_reference(cap, monkeypatch):
    """The climb's steps go out four per device -> host read; a cap that is not a multiple of four
    still stops every start after exactly `cap` steps (MAX_CLIMB_STEPS patched on both sides), and
    the reported step count is the reference loop's (the longest start's iterations, <= cap)."""
    from golden_io import Ctx, load, ref_model, to_cfg
    from paper_2212_11142_b200 import acquisition as A
    from paper_2212_11142_b200 import device as D
    bt = ref()
    meta, arr, space = load("mixed_fit")
    gp, feas = ref_model(meta, arr, space)
    cands = [to_cfg(space, c) for c in meta["cands"][:800]]
    evaluated = {to_cfg(space, c) for c in meta["evaluated"]}
    monkeypatch.setattr(bt.acquisition, "MAX_CLIMB_STEPS", cap)
    monkeypatch.setattr(A, "MAX_CLIMB_STEPS", cap)
    steps = []
    orig = D.Scorer.climb

    def climb(self, *a, **k):
        out = orig(self, *a, **k)
        steps.append(out[1])
        return out
    monkeypatch.setattr(D.Scorer, "climb", climb)
    want = bt.optimize_acquisition(
        bt.AcquisitionContext(gp=gp, feas=feas, best_feasible_value=meta["f_best"], eps_f=meta["eps_f"],
                              rng=np.random.default_rng(0), evaluated=evaluated), space, None,
        sample_fn=lambda n, r: cands)
    got = A.optimize_acquisition(Ctx(gp, feas, meta["f_best"], meta["eps_f"], np.random.default_rng(0), evaluated),
                                 space, None, sample_fn=lambda n, r: cands)
    assert got == want
    assert steps and all(1 <= s <= cap for s in steps)


def test_reference_model_objects_reach_the_gpu():
    """The reference's own GPModel / FeasibilityModel / ChainOfTrees / SearchSpace objects are
    consumed as they are (the fixtures' models rebuilt through the reference constructors)."""
    import oracle
    from golden_io import Ctx, load, oracle_model, ref_model, to_cfg
    from paper_2212_11142_b200 import acquisition as A
    bt = ref()
    for case in ("C3", "M200", "mixed_fit"):
        meta, arr, space = load(case)
        gp, feas = ref_model(meta, arr, space)
        assert isinstance(gp, bt.GPModel) and isinstance(feas, bt.FeasibilityModel)
        cands = [to_cfg(space, c) for c in meta["cands"][:512]]
        values, probs = A.scores(Ctx(gp, feas, meta["f_best"], meta["eps_f"]), cands)
        rv, rp = bt.acquisition._scores(
            bt.AcquisitionContext(gp=gp, feas=feas, best_feasible_value=meta["f_best"],
                                  eps_f=meta["eps_f"], rng=np.random.default_rng(0)), cands)
        assert np.array_equal(probs, rp), case
        fin = np.isfinite(rv)
        assert np.array_equal(fin, np.isfinite(values)), case
        np.testing.assert_allclose(values[fin], rv[fin], rtol=1e-5, atol=1e-9 * np.abs(rv[fin]).max())
        og, of = oracle_model(meta, arr, space)
        ov, _ = oracle.scores(og, of, cands, meta["f_best"], meta["eps_f"])
        np.testing.assert_allclose(ov[fin], rv[fin], rtol=1e-7, atol=1e-12 * np.abs(rv[fin]).max())


@pytest.mark.parametrize("case", ["mixed_fit", "C2", "M200"])
def test_batched_gp_fit_matches_reference_fit(case):
    """hyperfit.gp_fit (the 8 L-BFGS-B restarts concurrent, their objective calls batched on the
    GPU) against the reference's gp_fit on the same training set and RNG state: the coarse stage
    is the reference's own (identical RNG draw and candidate order), the refined optimum agrees to
    1e-6 relative (the objective is FP64 but not LAPACK's bits), and the fit takes a fraction of
    the objective launches."""
    import time

    from golden_io import load, to_cfg
    from paper_2212_11142_b200 import hyperfit
    bt = ref()
    meta, arr, space = load(case)
    train = [to_cfg(space, c) for c in meta["train"]]
    y = meta["y"]
    t0 = time.perf_counter()
    want = bt.gp_fit(space, train, y, np.random.default_rng(9))
    t1 = time.perf_counter()
    got = hyperfit.gp_fit(space, train, y, np.random.default_rng(9))
    t2 = time.perf_counter()
    print(f"{case} n={len(train)}: reference gp_fit {t1 - t0:.2f} s, batched {t2 - t1:.3f} s, "
          f"{hyperfit.gp_fit.last_batched_calls} batched objective calls")
    assert np.array_equal(got.start_values, want.start_values)
    hw, hg = want.hyperparameters, got.hyperparameters
    np.testing.assert_allclose([hg.outputscale, hg.noise_variance, *hg.lengthscales],
                               [hw.outputscale, hw.noise_variance, *hw.lengthscales], rtol=1e-6)
    assert abs(got.map_value - want.map_value) <= 1e-9 * max(1.0, abs(want.map_value))
    # batching changes nothing: the reference's sequential fit with the GPU objective installed
    # (lml=True) reaches bit-identical hyperparameters
    seq = _patched(bt, lambda: bt.gp_fit(space, train, y, np.random.default_rng(9)), lml=True)
    got2 = _patched(bt, lambda: hyperfit.gp_fit(space, train, y, np.random.default_rng(9)), lml=True)
    hs, h2 = seq.hyperparameters, got2.hyperparameters
    assert (hs.outputscale, hs.noise_variance, hs.lengthscales) == (h2.outputscale, h2.noise_variance, h2.lengthscales)
    assert seq.map_value == got2.map_value


def test_patched_run_with_batched_gp_fit():
    """install(fit=True, lml=True): the whole BO loop with the GPU hyperparameter fit; the history
    equals the reference's on this run."""
    bt = ref()
    for name, seed, budget in (("quadratic-mixed", 3, 30), ("hidden-ridge", 5, 24)):
        bench = bt.builtin(name)
        want = _run(bt, bench, budget, seed)
        got = _patched(bt, lambda: _run(bt, bench, budget, seed), whole_path=True, lml=True, fit=True)
        assert _first_divergence(got.history, want.history) is None, (name, _first_divergence(got.history,
                                                                                              want.history))


@pytest.mark.parametrize("case", ["C3", "C4", "M200", "mixed_fit", "mixed_metrics"])
@pytest.mark.parametrize("draws", [48, 3])
def test_device_rf_fit_equals_reference(case, draws, monkeypatch):
    """forest_fit.rf_fit (trees built on the GPU, feature subsets drawn from numpy in the
    reference's order) returns the reference's FeasibilityModel arrays bit for bit; draws=3 forces
    the "draw more and build again" path for every tree."""
    import time

    from golden_io import load, to_cfg
    from paper_2212_11142_b200 import forest_fit
    monkeypatch.setattr(forest_fit, "DRAWS", draws)
    bt = ref()
    meta, arr, space = load(case)
    ev = [to_cfg(space, c) for c in meta["evaluated"]]
    labels = meta["labels"]
    t0 = time.perf_counter()
    want = bt.rf_fit(space, ev, labels, np.random.default_rng(31), use_transforms=meta["use_transforms"])
    t1 = time.perf_counter()
    got = forest_fit.rf_fit(space, ev, labels, np.random.default_rng(31), use_transforms=meta["use_transforms"])
    t2 = time.perf_counter()
    print(f"{case}: {len(ev)} records, {len(want.feature)} nodes; reference rf_fit {t1 - t0:.3f} s, device {t2 - t1:.3f} s")
    assert np.array_equal(got.bootstrap_seeds, want.bootstrap_seeds)
    assert got.constant == want.constant
    for name in ("feature", "threshold", "left", "right", "value", "roots"):
        a, b = getattr(got, name), getattr(want, name)
        assert a.dtype == b.dtype and np.array_equal(a, b), name


def test_patched_loop_on_chain_of_trees_pool_is_the_reference_history():
    """C3 (known constraints, 10 parameters, chain of trees larger than the 5000-candidate pool,
    hidden resource rule): the leaf-uniform pool is drawn straight into rows (sampling.cot_rows)
    and the whole run still equals the reference's."""
    bt = ref()
    from paper_2212_11142_b200 import scenarios
    space = scenarios.build_space("C3", bt.space)
    assert bt.build_cot(space).count() > 5000
    bench = bt.Benchmark("c3-cot", space, lambda c: scenarios.objective("C3", c),
                         hidden_rule=lambda c: scenarios.hidden_ok("C3", c), default_budget=24)
    want = _run(bt, bench, 24, 4)
    got = _patched(bt, lambda: _run(bt, bench, 24, 4), whole_path=True)
    assert _first_divergence(got.history, want.history) is None, _first_divergence(got.history,
                                                                                   want.history)
    assert sum(r.phase == "bo" for r in got.history) > 0
