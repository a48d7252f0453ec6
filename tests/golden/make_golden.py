"""Generate the golden fixtures by running the REFERENCE (boxtune, /root/reference/pkg/src).

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

Each case writes <case>.json (space descriptor, configurations, scalars) and <case>.npz (arrays:
Cholesky factor, alpha, forest, and the reference's outputs).  The GPU tests and the oracle tests
read only these files.  Everything is seeded; rerunning reproduces the files on the same host.
"""
from __future__ import annotations

import json
import math
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

import boxtune  # noqa: E402  (the reference)
from boxtune import acquisition as ref_acq  # noqa: E402
from boxtune import constraints as ref_con  # noqa: E402
from boxtune import engine as ref_engine  # noqa: E402
from boxtune import feasibility as ref_feas  # noqa: E402
from boxtune import space as ref_space  # noqa: E402
from boxtune import surrogate as ref_sur  # noqa: E402

from paper_2212_11142_b200 import scenarios as S  # noqa: E402
from paper_2212_11142_b200.constraints import flatten_cot  # noqa: E402
from paper_2212_11142_b200.layout import SpaceLayout  # noqa: E402


def jcfg(cfg):
    return [list(v) if isinstance(v, tuple) else v for v in cfg]


def model_arrays(gp, feas):
    arr = {"L": np.tril(gp._cho[0]), "alpha": np.asarray(gp.alpha)}
    if feas is not None:
        if feas.constant is not None:
            arr["rf_constant"] = np.array([feas.constant])
        else:
            arr.update(rf_feature=feas.feature, rf_threshold=feas.threshold, rf_left=feas.left,
                       rf_right=feas.right, rf_value=feas.value, rf_roots=feas.roots)
        arr["rf_max_depth"] = np.array([feas.max_depth])
        arr["rf_n_trees"] = np.array([feas.n_trees])
    return arr


def model_meta(gp, y):
    h = gp.hyperparameters
    return {"outputscale": h.outputscale, "noise_variance": h.noise_variance,
            "lengthscales": list(h.lengthscales), "log_objective": bool(gp.log_objective),
            "use_transforms": bool(gp.use_transforms), "y_mean": gp.y_mean, "y_std": gp.y_std,
            "train": [jcfg(c) for c in gp.configs], "y": [float(v) for v in y]}


def save(case, meta, arrays):
    (HERE / f"{case}.json").write_text(json.dumps(meta, indent=None, separators=(",", ":")))
    np.savez_compressed(HERE / f"{case}.npz", **arrays)
    print(f"{case}: {len(json.dumps(meta)) // 1024} KB json, arrays {sorted(arrays)}")


def score_case(case, desc, n_train, q, seed, *, rf_rule=None, eps=0.0, hyper="fit",
               sampler="uniform", probe_neighbors=8, extra=None):
    rng = np.random.default_rng(seed)
    space = S.build_space(desc, ref_space)
    cot = ref_con.build_cot(space) if space.constraints else None
    draw = (lambda k: cot.sample_leaf_uniform(k, rng)) if cot is not None else \
        (lambda k: ref_space.sample_uniform(space, k, rng))
    name = desc.get("name", case)
    evals, feas_flags, ys = [], [], []
    seen = set()
    while sum(feas_flags) < n_train:
        for cfg in draw(64):
            if cfg in seen:
                continue
            seen.add(cfg)
            ok = rf_rule(cfg) if rf_rule else True
            evals.append(cfg)
            feas_flags.append(ok)
            ys.append(S.objective(name, cfg) if ok else None)
            if sum(feas_flags) >= n_train:
                break
    train = [c for c, f in zip(evals, feas_flags) if f]
    y = [v for v in ys if v is not None]
    if hyper == "fit":
        gp = ref_sur.gp_fit(space, train, y, rng)
    else:
        h = ref_sur.GPHyperparameters(outputscale=float(rng.uniform(0.5, 2.0)),
                                      noise_variance=float(rng.uniform(1e-4, 0.1)),
                                      lengthscales=tuple(rng.uniform(0.4, 1.5, space.dimension)))
        gp = ref_sur.GPModel(space, train, y, h, log_objective=True)
    feas = None
    if rf_rule is not None and not all(feas_flags):
        feas = ref_feas.rf_fit(space, evals, feas_flags, rng)
    f_best = min(y)
    cands = list(dict.fromkeys(draw(q)))
    ctx = ref_acq.AcquisitionContext(gp=gp, feas=feas, best_feasible_value=f_best, eps_f=eps,
                                     rng=rng, evaluated=set(evals))
    mean, var = gp.predict_batch(cands)
    values, probs = ref_acq._scores(ctx, cands)
    arrays = model_arrays(gp, feas)
    arrays.update(mean=mean, var=var, values=values, probs=probs)
    meta = {"case": case, "space": desc, **model_meta(gp, y), "f_best": f_best,
            "f_model": gp.objective_to_model(f_best), "eps_f": eps,
            "cands": [jcfg(c) for c in cands], "evaluated": [jcfg(c) for c in evals],
            "labels": [bool(f) for f in feas_flags]}
    if feas is not None:
        # q == 1 summation order: the reference's per-config probabilities
        single = cands[:64]
        arrays["probs_q1"] = np.array([feas.predict_proba(c) for c in single])
        arrays["rf_X"] = ref_feas.encode_configs(space, cands[:256])
    # neighbours of a few candidates, with and without the chain of trees
    starts = cands[:probe_neighbors]
    meta["nbr_starts"] = [jcfg(c) for c in starts]
    meta["nbr_plain"] = [[jcfg(c) for c in ref_space.neighbors(space, s)] for s in starts]
    if cot is not None:
        meta["nbr_cot"] = [[jcfg(c) for c in ref_space.neighbors(space, s, cot)] for s in starts]
        probe = ref_space.sample_uniform(space, 4000, rng)
        meta["cot_probe"] = [jcfg(c) for c in probe]
        arrays["cot_mask"] = np.array([cot.contains(c) for c in probe])
        arrays["cons_mask"] = np.array([[ref_con.eval_constraint(e, space.as_dict(c)) is True
                                         for e in space.constraints] for c in probe])
        meta["cot_count"] = cot.count()
        # the chain of trees as the device tables (bench.py loads workloads without the reference)
        t = flatten_cot(cot, SpaceLayout(space))
        for k in ("group_kind", "group_param_begin", "group_params", "group_root", "child_begin",
                  "child_count", "node_value", "leaf_count"):
            arrays["cot_" + k] = getattr(t, k)
    # pairwise squared distances of the training set (bit-exact target) and the coarse LML
    sq = ref_sur.pairwise_sq_distances(space, train, train)
    arrays["sq_train_sum"] = np.array([sq.sum()])
    arrays["sq_train_head"] = sq[:, :16, :16]
    lo, hi = ref_sur._search_boxes(space.dimension, ref_sur.LengthscalePrior())
    th = np.random.default_rng(seed + 1).uniform(lo, hi, size=(64, 2 + space.dimension))
    z, _, _ = ref_sur._standardize(np.log(np.asarray(y)) if gp.log_objective else np.asarray(y))
    arrays["lml_thetas"] = th
    arrays["lml_z"] = z
    arrays["lml"] = ref_sur._batched_coarse_lml(sq, z, th)
    arrays["lml_prior"] = ref_sur._prior_term(th, ref_sur.LengthscalePrior())
    # _lml_core value + gradient (the L-BFGS-B objective) at the first 8 coarse settings
    core_v, core_g, core_ok = [], [], []
    for t in th[:8]:
        try:
            v, g = ref_sur._lml_core(sq, z, math.exp(t[0]), math.exp(t[1]), np.exp(t[2:]),
                                     want_grad=True, prior=ref_sur.LengthscalePrior())
            core_v.append(v), core_g.append(g), core_ok.append(True)
        except np.linalg.LinAlgError:
            core_v.append(-np.inf), core_g.append(np.zeros(2 + space.dimension)), core_ok.append(False)
    arrays["core_value"] = np.array(core_v)
    arrays["core_grad"] = np.array(core_g)
    arrays["core_ok"] = np.array(core_ok)
    if extra:
        extra(space, cot, gp, feas, ctx, cands, meta, arrays, rng)
    save(case, meta, arrays)


def selection_extra(n_pool, seed):
    def run(space, cot, gp, feas, ctx, cands, meta, arrays, rng):
        prng = np.random.default_rng(seed)
        pool = (cot.sample_leaf_uniform(n_pool, prng) if cot is not None
                else ref_space.sample_uniform(space, n_pool, prng))
        ctx.rng = np.random.default_rng(seed + 7)
        chosen = ref_acq.optimize_acquisition(ctx, space, cot, sample_fn=lambda n, r: pool)
        meta["sel_pool"] = [jcfg(c) for c in pool]
        meta["sel_chosen"] = jcfg(chosen)
        vals, _ = ref_acq._scores(ctx, list(dict.fromkeys(pool)))
        srt = np.sort(vals[np.isfinite(vals)])[::-1]
        meta["sel_margin"] = float((srt[0] - srt[1]) / abs(srt[0])) if len(srt) > 1 and srt[0] else None
    return run


def engine_trace(case, bench_name, seed, budget=None):
    """Record every BO iteration of a reference run: model state, pool, chosen configuration."""
    bench = boxtune.builtin(bench_name)
    iters = []
    orig = ref_engine.optimize_acquisition

    def spy(ctx, space, cot=None, sample_fn=None, local_search=True, **kw):
        holder = {}

        def sfn(n, rng):
            raw = sample_fn(n, rng) if sample_fn is not None else \
                ref_acq._default_sampler(space, cot)(n, rng)
            holder["pool"] = list(raw)
            return raw

        out = orig(ctx, space, cot, sample_fn=sfn, local_search=local_search, **kw)
        gp, feas = ctx.gp, ctx.feas
        rec = {"meta": {**model_meta(gp, [bench.objective(c) for c in gp.configs]), "f_best": ctx.best_feasible_value, "eps_f": ctx.eps_f,
                        "f_model": gp.objective_to_model(ctx.best_feasible_value),
                        "evaluated": [jcfg(c) for c in sorted(ctx.evaluated, key=repr)],
                        "pool": [jcfg(c) for c in holder["pool"]], "chosen": jcfg(out)},
               "arrays": model_arrays(gp, feas)}
        iters.append(rec)
        return out

    class Scn:
        pass

    scn = Scn()
    scn.space, scn.budget, scn.method = bench.space, budget or bench.default_budget, "bo"
    scn.options, scn.doe_size, scn.name, scn.seed = ref_engine.EngineOptions(), None, bench_name, seed
    ref_engine.optimize_acquisition = spy
    try:
        run = ref_engine.run_bo_loop(scn, bench, np.random.default_rng(seed))
    finally:
        ref_engine.optimize_acquisition = orig
    desc = {"params": [], "constraints": list(bench.space.constraint_texts)}
    for p in bench.space.parameters:
        d = {"name": p.name, "kind": p.kind, "transform": p.transform}
        if p.kind in ("real", "integer"):
            d.update(lo=p.lo, hi=p.hi)
        elif p.kind in ("ordinal", "categorical"):
            d["values"] = list(p.values)
        else:
            d.update(size=p.size, metric=p.permutation_metric)
        desc["params"].append(d)
    meta = {"case": case, "space": desc, "iters": [r["meta"] for r in iters],
            "history": [jcfg(r.configuration) for r in run.history]}
    arrays = {}
    for i, r in enumerate(iters):
        for k, v in r["arrays"].items():
            arrays[f"it{i}_{k}"] = v
    save(case, meta, arrays)


def main():
    which = set(sys.argv[1:])

    def want(c):
        return not which or c in which

    mixed = {**S.SCENARIOS["C5"], "name": "C5"}
    if want("mixed_fit"):
        score_case("mixed_fit", mixed, 40, 2000, 11, rf_rule=lambda c: c[3] <= 12, eps=0.0)
    if want("mixed_metrics"):
        alt = {"params": [dict(p) for p in mixed["params"]], "constraints": [], "name": "C5"}
        alt["params"][8]["metric"] = "hamming"
        alt["params"][9]["metric"] = "naive"
        alt["params"][5]["transform"] = "log"
        alt["params"][5]["lo"] = 0.5
        alt["params"][5]["hi"] = 4.0
        score_case("mixed_metrics", alt, 30, 1500, 12, hyper="random",
                   rf_rule=lambda c: c[6] != "d", eps=0.25)
    if want("C1"):
        score_case("C1", {**S.SCENARIOS["C1"], "name": "C1"}, 30, 2000, 13,
                   extra=selection_extra(2000, 101))
    if want("C2"):
        score_case("C2", {**S.SCENARIOS["C2"], "name": "C2"}, 60, 3000, 14,
                   extra=selection_extra(5000, 102))
    if want("C3"):
        score_case("C3", {**S.SCENARIOS["C3"], "name": "C3"}, 200, 2000, 15,
                   rf_rule=lambda c: S.hidden_ok("C3", c), eps=0.3,
                   extra=selection_extra(5000, 103))
    if want("M200"):  # the north-star configuration: d=10 mixed, n=200, RF on
        score_case("M200", {**S.SCENARIOS["C5"], "name": "C5"}, 200, 2000, 17,
                   rf_rule=lambda c: S.hidden_ok("M200", c), eps=0.3,
                   extra=selection_extra(5000, 104))
    if want("C4"):
        score_case("C4", {**S.SCENARIOS["C4"], "name": "C4"}, 60, 1000, 16,
                   rf_rule=lambda c: S.hidden_ok("C4", c))
    if want("trace_quadratic"):
        engine_trace("trace_quadratic", "quadratic-mixed", 3)
    if want("trace_ridge"):
        engine_trace("trace_ridge", "hidden-ridge", 5)
    if want("trace_perm"):
        engine_trace("trace_perm", "perm-assignment", 7, budget=30)


if __name__ == "__main__":
    main()
