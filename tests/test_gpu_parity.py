"""GPU parity: libbx_sm100 through the package API vs the reference's golden outputs and the oracle.

Bars (BASELINE.json north_star): bit-exact for forest probabilities, neighbour sets, chain-of-trees
and constraint masks and pairwise distances; mean / variance / EI within 1e-5 relative (with an
absolute floor of 1e-9 x the largest magnitude, because standardised quantities cross zero);
identical selected configuration.
"""
import numpy as np
import pytest
import torch

import oracle
from golden_io import CASES, TRACES, Ctx, cot_for, load, model, oracle_model, to_cfg

pytestmark = pytest.mark.gpu

RTOL = 1e-5


def close(got, want, rtol=RTOL, floor=1e-9):
    got, want = np.asarray(got), np.asarray(want)
    atol = floor * max(float(np.max(np.abs(want))), 1e-300)
    np.testing.assert_allclose(got, want, rtol=rtol, atol=atol)


@pytest.fixture(scope="module")
def sc():
    from paper_2212_11142_b200.device import scorer
    return scorer()


@pytest.mark.parametrize("case", CASES)
def test_predict(case, sc):
    from paper_2212_11142_b200 import acquisition as A
    meta, arr, space = load(case)
    gp, _ = model(meta, arr, space)
    cands = [to_cfg(space, c) for c in meta["cands"]]
    mean, var = A.predict_batch(gp, cands)
    close(mean, arr["mean"])
    close(var, arr["var"])


@pytest.mark.parametrize("case", CASES)
def test_scores(case, sc):
    from paper_2212_11142_b200 import acquisition as A
    meta, arr, space = load(case)
    gp, feas = model(meta, arr, space)
    ctx = Ctx(gp, feas, meta["f_best"], meta["eps_f"])
    cands = [to_cfg(space, c) for c in meta["cands"]]
    values, probs = A.scores(ctx, cands)
    assert np.array_equal(probs, arr["probs"])
    assert np.array_equal(np.isneginf(values), np.isneginf(arr["values"]))
    fin = np.isfinite(arr["values"])
    close(values[fin], arr["values"][fin])


@pytest.mark.parametrize("case", ["mixed_fit", "mixed_metrics", "C3", "C4"])
def test_forest_bit_exact(case, sc):
    from paper_2212_11142_b200 import acquisition as A
    meta, arr, space = load(case)
    _, feas = model(meta, arr, space)
    cands = [to_cfg(space, c) for c in meta["cands"]]
    assert np.array_equal(A.predict_proba_batch(feas, cands), arr["probs"])
    single = np.array([A.predict_proba_batch(feas, [c])[0] for c in cands[:64]])
    assert np.array_equal(single, arr["probs_q1"])
    lay = sc.layout
    assert np.array_equal(lay.features(lay.encode(cands[:256])), arr["rf_X"])


@pytest.mark.parametrize("case", ["mixed_fit", "mixed_metrics", "C3", "C4"])
def test_forest_generic_kernel_matches_coded(case, monkeypatch):
    """The integer-coded fast path and the generic f64 traversal give identical bits."""
    from paper_2212_11142_b200.device import Scorer
    meta, arr, space = load(case)
    _, feas = model(meta, arr, space)
    cands = [to_cfg(space, c) for c in meta["cands"]]
    monkeypatch.setenv("BX_FOREST_GENERIC", "1")
    generic = Scorer()
    monkeypatch.delenv("BX_FOREST_GENERIC")
    coded = Scorer()
    out = []
    for s in (generic, coded):
        s.set_space(space, feas.use_transforms)
        s.set_forest(feas)
        rows = s.to_device(s.layout.encode(cands))
        out.append(s.rf_predict(rows, pairwise=False).cpu().numpy())
        out.append(np.array([s.rf_predict(rows[i:i + 1]).item() for i in range(32)]))
    generic.close()
    coded.close()
    assert np.array_equal(out[0], arr["probs"]) and np.array_equal(out[2], arr["probs"])
    assert np.array_equal(out[1], arr["probs_q1"][:32]) and np.array_equal(out[3], arr["probs_q1"][:32])


@pytest.mark.parametrize("case", CASES)
def test_neighbors(case, sc):
    from paper_2212_11142_b200 import acquisition as A
    meta, arr, space = load(case)
    cot = cot_for(case)
    for start, plain in zip(meta["nbr_starts"], meta["nbr_plain"]):
        assert A.neighbors(space, to_cfg(space, start)) == [to_cfg(space, c) for c in plain]
    if cot is not None:
        for start, filt in zip(meta["nbr_starts"], meta["nbr_cot"]):
            assert A.neighbors(space, to_cfg(space, start), cot) == [to_cfg(space, c) for c in filt]


@pytest.mark.parametrize("case", ["C2", "C3"])
def test_masks(case, sc):
    from paper_2212_11142_b200 import acquisition as A
    meta, arr, space = load(case)
    cot = cot_for(case)
    probe = [to_cfg(space, c) for c in meta["cot_probe"]]
    assert np.array_equal(A.contains_batch(cot, probe), arr["cot_mask"])
    assert np.array_equal(A.constraints_batch(space, probe), arr["cons_mask"].all(1))


@pytest.mark.parametrize("case", CASES)
def test_pairwise_and_lml(case, sc):
    from paper_2212_11142_b200 import acquisition as A
    meta, arr, space = load(case)
    og, _ = oracle_model(meta, arr, space)
    lay = sc.set_space(space, meta["use_transforms"])
    rows = sc.to_device(lay.encode(og.configs))
    sq = sc.pairwise_sq(rows, rows).cpu().numpy()
    assert np.array_equal(sq, oracle.pairwise_sq(space, og.configs, og.configs, og.use_transforms))
    assert np.array_equal(sq[:, :16, :16], arr["sq_train_head"])
    lml = A.batched_coarse_lml(sq, arr["lml_z"], arr["lml_thetas"])
    want = arr["lml"]
    assert np.array_equal(np.isfinite(lml), np.isfinite(want))
    fin = np.isfinite(want)
    np.testing.assert_allclose(lml[fin], want[fin], rtol=1e-9, atol=1e-7)


@pytest.mark.parametrize("case", CASES)
def test_lml_core_gradient(case, sc):
    """_lml_core value and gradient (surrogate.py:356-400) vs the reference's own numbers."""
    from paper_2212_11142_b200 import acquisition as A

    class Prior:
        shape, rate = 2.0, 2.0

    meta, arr, space = load(case)
    og, _ = oracle_model(meta, arr, space)
    sq = oracle.pairwise_sq(space, og.configs, og.configs, og.use_transforms)
    for t, v, g, ok in zip(arr["lml_thetas"][:8], arr["core_value"], arr["core_grad"], arr["core_ok"]):
        args = (sq, arr["lml_z"], np.exp(t[0]), np.exp(t[1]), np.exp(t[2:]))
        if not ok:
            with pytest.raises(np.linalg.LinAlgError):
                A.lml_core(*args, want_grad=True, prior=Prior())
            continue
        val, grad = A.lml_core(*args, want_grad=True, prior=Prior())
        assert val == pytest.approx(v, rel=1e-9, abs=1e-7)
        np.testing.assert_allclose(grad, g, rtol=1e-6, atol=1e-6 * max(1.0, np.abs(g).max()))
        assert A.lml_core(*args, want_grad=False, prior=None) == pytest.approx(
            oracle.lml_core(*args, want_grad=False, prior=None), rel=1e-9, abs=1e-7)


@pytest.mark.parametrize("case", CASES)
def test_summary_consistent_with_values(case, sc):
    """Fused top-k / tracker reductions equal the host reductions over the same values."""
    meta, arr, space = load(case)
    gp, feas = model(meta, arr, space)
    sc.set_gp(gp)
    sc.set_forest(feas)
    ev = {to_cfg(space, c) for c in meta["evaluated"]}
    sc.set_evaluated(list(ev))
    cands = [to_cfg(space, c) for c in meta["cands"]]
    rows = sc.to_device(sc.layout.encode(cands))
    f_model = gp.objective_to_model(meta["f_best"])
    summ, values, probs = sc.score(rows, f_model, meta["eps_f"], k=10, want_values=True)
    v = values.cpu().numpy()
    order = [i for i in np.argsort(-v, kind="stable")[:10] if v[i] != -np.inf]
    assert [c.index for c in summ.top] == order
    assert summ.n_finite == int(np.sum(v != -np.inf))
    best = None
    for i, c in enumerate(cands):
        if v[i] == -np.inf or c in ev:
            continue
        if best is None or v[i] > v[best] or (v[i] == v[best] and c < cands[best]):
            best = i
    assert (summ.best.index if summ.best else None) == best


@pytest.mark.parametrize("case", ["C1", "C2", "C3"])
def test_selection(case, sc):
    from paper_2212_11142_b200 import acquisition as A
    meta, arr, space = load(case)
    gp, feas = model(meta, arr, space)
    pool = [to_cfg(space, c) for c in meta["sel_pool"]]
    ev = {to_cfg(space, c) for c in meta["evaluated"]}
    ctx = Ctx(gp, feas, meta["f_best"], meta["eps_f"], np.random.default_rng(0), ev)
    got = A.optimize_acquisition(ctx, space, cot_for(case), sample_fn=lambda n, r: pool)
    assert got == to_cfg(space, meta["sel_chosen"])


@pytest.mark.parametrize("trace", TRACES)
def test_engine_trace(trace, sc):
    from paper_2212_11142_b200 import acquisition as A
    meta, arr, space = load(trace)
    cot = cot_for(trace)
    for i, it in enumerate(meta["iters"]):
        gp, feas = model(it, arr, space, prefix=f"it{i}_")
        pool = [to_cfg(space, c) for c in it["pool"]]
        ev = {to_cfg(space, c) for c in it["evaluated"]}
        ctx = Ctx(gp, feas, it["f_best"], it["eps_f"], np.random.default_rng(0), ev)
        got = A.optimize_acquisition(ctx, space, cot, sample_fn=lambda n, r, pool=pool: pool)
        assert got == to_cfg(space, it["chosen"]), f"iteration {i}"


@pytest.mark.parametrize("case", CASES)
def test_posterior_kernels_agree(case, monkeypatch):
    """The tensor-core split product (gp_tc.cu) against the FP64 DMMA kernel (gp_fused.cu) on a
    generated pool much larger than the golden one; both must also meet the golden bar above."""
    from paper_2212_11142_b200.device import Scorer
    meta, arr, space = load(case)
    gp, _ = model(meta, arr, space)
    monkeypatch.setenv("BX_GP_DMMA", "1")
    ref = Scorer()
    ref.set_space(space)
    ref.set_gp(gp)
    monkeypatch.delenv("BX_GP_DMMA")
    tc = Scorer()
    tc.set_space(space)
    tc.set_gp(gp)
    assert ref.gp_kernel() == "dmma"
    assert tc.gp_kernel() == ("tensor" if len(gp.configs) <= 255 else "dmma")
    rows = tc.generate(300_001, seed=7)
    m1, v1 = (x.cpu().numpy() for x in tc.predict(rows))
    m0, v0 = (x.cpu().numpy() for x in ref.predict(rows))
    close(m1, m0, rtol=1e-7)
    close(v1, v0, rtol=1e-6)
    # and at the golden candidates, against the reference's numbers
    lay = tc.layout
    gold = tc.to_device(lay.encode([to_cfg(space, c) for c in meta["cands"]]))
    m2, v2 = (x.cpu().numpy() for x in tc.predict(gold))
    close(m2, arr["mean"])
    close(v2, arr["var"])
    ref.close()
    tc.close()


@pytest.mark.parametrize("case", ["C3", "C4", "mixed_fit", "mixed_metrics", "M200"])
def test_forest_paths_bit_exact(case, monkeypatch):
    """QuickScorer tables (with indirect slots for real parameters with many thresholds: M200,
    mixed_fit), the integer-coded node walk and the generic f64 walk give bit-identical
    probabilities and scores, in both summation orders."""
    from paper_2212_11142_b200.device import Scorer
    meta, arr, space = load(case)
    gp, feas = model(meta, arr, space)
    f = gp.objective_to_model(meta["f_best"])
    out = {}
    for name, env in [("generic", {"BX_FOREST_GENERIC": "1"}), ("walk", {"BX_FOREST_WALK": "1"}), ("qs", {})]:
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        sc = Scorer()
        sc.set_gp(gp)
        sc.set_forest(feas)
        rows = sc.generate(200_003, seed=3)
        _, values, probs = sc.score(rows, f, meta["eps_f"], k=10, want_values=True)
        out[name] = (values.cpu().numpy(), probs.cpu().numpy(), sc.rf_predict(rows, pairwise=False).cpu().numpy(),
                     sc.rf_predict(rows[:4099], pairwise=True).cpu().numpy())
        sc.close()
        for k in env:
            monkeypatch.delenv(k)
    for name in ("qs", "walk"):
        for a, b in zip(out[name], out["generic"]):
            assert np.array_equal(a, b), name


@pytest.mark.parametrize("case", CASES)
def test_embedding_distances_match_fma_distances(case, monkeypatch):
    """The tensor-core distance producers (W = |x'|^2 + |y'|^2 - 2 x'.y' over the Euclidean
    embedding of every metric, on DMMA) against the FMA producers (BX_TC_NO_DMMA=1): they differ
    only in the rounding of W, far inside the 1e-5 parity bar.  Every golden space embeds except
    mixed_metrics (naive permutation indicator), which falls back to the FMA producers."""
    from paper_2212_11142_b200 import scenarios
    from paper_2212_11142_b200.device import Scorer
    meta, arr, space = load(case)
    gp, _ = model(meta, arr, space)
    res, ks = [], []
    for no_dmma in (True, False):
        if no_dmma:
            monkeypatch.setenv("BX_TC_NO_DMMA", "1")
        else:
            monkeypatch.delenv("BX_TC_NO_DMMA")
        sc = Scorer()
        sc.set_gp(gp)
        ks.append(sc.distance_ksteps())
        rows = sc.to_device(scenarios.sample_rows_uniform(sc.layout, 200_000, np.random.default_rng(2)))
        res.append([x.cpu().numpy() for x in sc.predict(rows)])
        sc.close()
    assert ks[0] == 0 and (ks[1] == 0) == (case == "mixed_metrics"), ks
    (m0, v0), (m1, v1) = res
    close(m1, m0, rtol=1e-8)
    close(v1, v0, rtol=1e-7)


@pytest.mark.parametrize("n", [7, 40, 64, 200, 300, 500])
def test_lml_wide_paths_large_n(n, monkeypatch):
    """_lml_core with its gradient - the shared-memory kernel (n <= 40) or the whole-GPU pipeline
    (one setting over every SM) - and the coarse LML (one CTA per setting up to n = 96, else the
    batched blocked pipeline) at n up to 500 (BASELINE config 5) against the oracle, and against
    the one-CTA-per-setting global-memory kernels (BX_LML_NARROW=1)."""
    from paper_2212_11142_b200 import acquisition as A
    from paper_2212_11142_b200.device import Scorer

    rng = np.random.default_rng(n)
    D = 10
    X = rng.uniform(0, 1, (n, D))
    sq = np.stack([(X[:, k, None] - X[None, :, k]) ** 2 for k in range(D)])
    z = rng.standard_normal(n)
    ls = rng.uniform(0.3, 2.0, D)
    args = (sq, z, 1.3, 1e-3, ls)
    v, g = A.lml_core(*args, want_grad=True)
    v0, g0 = oracle.lml_core(*args, want_grad=True, prior=None)
    assert v == pytest.approx(v0, rel=1e-9, abs=1e-7)
    np.testing.assert_allclose(g, g0, rtol=1e-7, atol=1e-7 * np.abs(g0).max())
    th = np.concatenate([np.log([[1.3, 1e-3]]).repeat(16, 0), np.log(rng.uniform(0.3, 2.0, (16, D)))], 1)
    th[3, 2:] = np.log(50.0)  # long lengthscales: near-singular Gram, may fail like LAPACK
    out = A.batched_coarse_lml(sq, z, th)
    ref = oracle.lml.coarse_lml(sq, z, th)
    fin = np.isfinite(ref)
    assert np.array_equal(np.isfinite(out), fin)
    np.testing.assert_allclose(out[fin], ref[fin], rtol=1e-9, atol=1e-7)
    monkeypatch.setenv("BX_LML_NARROW", "1")
    sc = Scorer()
    monkeypatch.setattr(A, "scorer", lambda: sc)
    v1, g1 = A.lml_core(*args, want_grad=True)
    out1 = A.batched_coarse_lml(sq, z, th)
    sc.close()
    assert v1 == pytest.approx(v, rel=1e-10, abs=1e-8)
    np.testing.assert_allclose(g1, g, rtol=1e-8, atol=1e-8 * np.abs(g).max())
    np.testing.assert_allclose(out1[fin], out[fin], rtol=1e-10, atol=1e-8)


def test_lml_core_batched_equals_single_calls():
    """bx_lml_core over c settings (side by side on grid.y) gives, bit for bit, the value, gradient
    and ok flag of c single-setting calls: what the batched L-BFGS-B restarts rely on."""
    import torch

    from paper_2212_11142_b200.device import scorer
    meta, arr, space = load("M200")
    og, _ = oracle_model(meta, arr, space)
    sq = oracle.pairwise_sq(space, og.configs, og.configs, og.use_transforms)
    sc = scorer()
    dev = f"cuda:{sc.device}"
    sq_d = torch.as_tensor(sq, device=dev)
    z = torch.as_tensor(arr["lml_z"], device=dev)
    th = arr["lml_thetas"][:9]
    prm = torch.as_tensor(np.exp(th), device=dev)
    v, g, ok = sc.lml_core(sq_d, z, prm, True, None)
    for i in range(len(th)):
        v1, g1, ok1 = sc.lml_core(sq_d, z, prm[i:i + 1], True, None)
        assert int(ok1.item()) == int(ok[i].item())
        if int(ok1.item()):
            assert v1.item() == v[i].item() and torch.equal(g1[0], g[i])


@pytest.mark.parametrize("n", [100, 232])
def test_lml_small_kernel_up_to_its_shared_memory_limit(n, monkeypatch):
    """The one-CTA shared-memory _lml_core (packed triangle factored and inverted in place) at sizes
    beyond its default range (BX_LML_SMALL_MAX), up to the largest triangle that fits: value and
    gradient against the oracle and equal to the whole-GPU pipeline's to FP64 rounding."""
    from paper_2212_11142_b200 import acquisition as A
    from paper_2212_11142_b200.device import Scorer

    rng = np.random.default_rng(n + 1)
    D = 10
    X = rng.uniform(0, 1, (n, D))
    sq = np.stack([(X[:, k, None] - X[None, :, k]) ** 2 for k in range(D)])
    z = rng.standard_normal(n)
    args = (sq, z, 0.9, 1e-4, rng.uniform(0.3, 2.0, D))
    v, g = A.lml_core(*args, want_grad=True)  # default: the whole-GPU pipeline at this n
    monkeypatch.setenv("BX_LML_SMALL_MAX", "232")
    sc = Scorer()
    monkeypatch.setattr(A, "scorer", lambda: sc)
    v1, g1 = A.lml_core(*args, want_grad=True)
    sc.close()
    v0, g0 = oracle.lml_core(*args, want_grad=True, prior=None)
    assert v1 == pytest.approx(v0, rel=1e-9, abs=1e-7)
    np.testing.assert_allclose(g1, g0, rtol=1e-7, atol=1e-7 * np.abs(g0).max())
    assert v1 == pytest.approx(v, rel=1e-10, abs=1e-8)
    np.testing.assert_allclose(g1, g, rtol=1e-8, atol=1e-8 * np.abs(g).max())
