"""The acquisition hot path behind the reference's own Python API.

Signatures, argument meaning, return values and exceptions follow the reference functions they
replace; each docstring names its counterpart.  Every number is produced on the GPU by
libbx_sm100; the host only samples the pool (so the caller's RNG stream is consumed exactly as the
reference consumes it), encodes/decodes configurations and runs the O(n_starts x steps) control
logic of the hill climb.
"""
from __future__ import annotations


import numpy as np
import torch

from . import _native as N
from . import sampling
from .device import Scorer, scorer

N_CANDIDATES = 5000   # acquisition.py:23
N_STARTS = 10         # acquisition.py:24
MAX_CLIMB_STEPS = 50  # acquisition.py:25
FAST_SAMPLER = True   # default samplers drawn straight into rows (sampling.py); False: the caller's


class SpaceExhausted(Exception):
    """Every feasible configuration has already been evaluated (acquisition.py:30-31)."""


def _exhausted_type(space):
    # raise the reference's own exception class when the caller uses the reference package
    mod = type(space).__module__.rsplit(".", 1)[0]
    try:
        import importlib

        return importlib.import_module(mod + ".acquisition").SpaceExhausted
    except Exception:
        return SpaceExhausted


class _State:
    """Tracks which model objects are resident on the device (identity-keyed)."""

    def __init__(self):
        self.gen = -1
        self.gp = None
        self.feas = None
        self.feas_set = False
        self.evaluated_len = -1
        self.evaluated_id = None


_STATE: dict = {}


def _state(sc: Scorer) -> _State:
    st = _STATE.setdefault(id(sc), _State())
    if st.gen != sc.space_gen:  # a space change dropped every model upload
        st.__init__()
        st.gen = sc.space_gen
    return st


def _prepare(ctx, sc: Scorer, evaluated: bool):
    st = _state(sc)
    gp = ctx.gp
    if st.gp is not gp:
        sc.set_gp(gp)
        st = _state(sc)
        st.gp = gp
        st.evaluated_len = -1
    if not st.feas_set or st.feas is not ctx.feas:
        sc.set_forest(ctx.feas)
        st.feas, st.feas_set = ctx.feas, True
    if evaluated:
        ev = ctx.evaluated if ctx.evaluated is not None else ()
        if st.evaluated_id != id(ev) or st.evaluated_len != len(ev):
            sc.set_evaluated(list(ev))
            st.evaluated_id, st.evaluated_len = id(ev), len(ev)
    return sc.layout


def scores(ctx, configs):
    """`_scores(ctx, configs) -> (values, probs)` (acquisition.py:70-79) on the GPU."""
    configs = list(configs)
    sc = scorer()
    lay = _prepare(ctx, sc, evaluated=False)
    f_model = ctx.gp.objective_to_model(ctx.best_feasible_value)
    rows = sc.to_device(lay.encode(configs))
    _, values, probs = sc.score(rows, f_model, ctx.eps_f, k=0, want_values=True, summary=False)
    return values.cpu().numpy(), probs.cpu().numpy()


def acquisition_value(ctx, cfg) -> float:
    """acquisition.py:82-84."""
    return float(scores(ctx, [cfg])[0][0])


def predict_batch(gp, configs, include_noise: bool = False):
    """`GPModel.predict_batch` (surrogate.py:315-328) on the GPU."""
    sc = scorer()
    st = _state(sc)
    if st.gp is not gp:
        sc.set_gp(gp)
        st = _state(sc)
        st.gp = gp
    rows = sc.to_device(sc.layout.encode(list(configs)))
    mean, var = sc.predict(rows)
    mean, var = mean.cpu().numpy(), var.cpu().numpy()
    if include_noise:
        var = var + gp.noise * gp.y_std ** 2
    return mean, var


def predict_proba_batch(feas, configs):
    """`FeasibilityModel.predict_proba_batch` (feasibility.py:72-89) on the GPU, bit-exact."""
    configs = list(configs)
    if feas.constant is not None:
        return np.full(len(configs), feas.constant)
    if feas.roots is None or len(feas.roots) == 0:
        raise N.NativeError(N.BX_ERR_NO_TREES, "feasibility model has no trees")
    sc = scorer()
    if sc.layout is None or sc.layout.space is not feas.space or \
            sc.layout.use_transforms != bool(feas.use_transforms):
        sc.set_space(feas.space, feas.use_transforms)
    st = _state(sc)
    if st.feas is not feas or not st.feas_set:
        sc.set_forest(feas)
        st.feas, st.feas_set = feas, True
    rows = sc.to_device(sc.layout.encode(configs))
    return sc.rf_predict(rows).cpu().numpy()


def neighbors(space, cfg, cot=None) -> list:
    """`neighbors(space, cfg, cot)` (space.py:289-309) on the GPU: same set, same order."""
    sc = scorer()
    lay = sc.layout_for(space)
    if cot is not None:
        sc.set_cot(cot)
    out, valid = sc.neighbors(sc.to_device(lay.encode([cfg])), use_cot=cot is not None)
    keep = out[valid.bool()]
    return lay.decode(keep.cpu().numpy().view(np.uint32))


def contains_batch(cot, configs) -> np.ndarray:
    """`ChainOfTrees.contains` (constraints.py:413-430) over a batch, bit-exact."""
    sc = scorer()
    lay = sc.layout_for(cot.space)
    sc.set_cot(cot)
    return sc.cot_contains(sc.to_device(lay.encode(list(configs)))).cpu().numpy().astype(bool)


def constraints_batch(space, configs) -> np.ndarray:
    """all(eval_constraint(c, cfg) is True for c in space.constraints) over a batch."""
    sc = scorer()
    lay = sc.layout_for(space)
    sc.set_constraints(space)
    return sc.constraints_eval(sc.to_device(lay.encode(list(configs)))).cpu().numpy().astype(bool)


# ---------------------------------------------------------------------------------------------
# whole-path replacement
# ---------------------------------------------------------------------------------------------
def _default_sampler(space, cot):
    """acquisition.py:114-134, consuming the RNG identically."""
    if cot is not None:
        return lambda n, rng: cot.sample_leaf_uniform(n, rng)
    sample_uniform = _sample_uniform_for(space)
    if not space.constraints:
        return lambda n, rng: sample_uniform(space, n, rng)

    def rejection(n, rng):
        out, attempts = [], 0
        while len(out) < n and attempts < 50 * n:
            batch = sample_uniform(space, n, rng)
            attempts += n
            ok = constraints_batch(space, batch)
            for cfg, good in zip(batch, ok):
                if good:
                    out.append(cfg)
                    if len(out) == n:
                        break
        return out

    return rejection


def _sample_uniform_for(space):
    """The caller's own `sample_uniform` (space.py:312-332): the module that defines the space."""
    import importlib

    return importlib.import_module(type(space).__module__).sample_uniform


def _better(a_val, a_cfg, b_val, b_cfg) -> bool:
    """(value desc, configuration asc) - the order of _argbest / _Tracker (acquisition.py:87-111)."""
    return a_val > b_val or (a_val == b_val and a_cfg < b_cfg)


def optimize_acquisition(ctx, space, cot=None, sample_fn=None, local_search: bool = True,
                         n_candidates: int = N_CANDIDATES, n_starts: int = N_STARTS):
    """`optimize_acquisition` (acquisition.py:152-206) with every score, top-k, tracker reduction and
    neighbour set computed on the GPU."""
    Exhausted = _exhausted_type(space)
    sc = scorer()
    lay = _prepare(ctx, sc, evaluated=True)
    rows_h = None
    if sample_fn is None and cot is not None and FAST_SAMPLER and n_candidates >= 1 \
            and sampling.is_reference_cot(cot):
        # leaf-uniform chain-of-trees pool (acquisition.py:115-116) straight into rows
        rows_h = sampling.unique_rows(sampling.cot_rows(lay, cot, n_candidates, ctx.rng))
    elif sample_fn is None and cot is None and FAST_SAMPLER and n_candidates >= 1 \
            and sampling.is_reference_sampler(_sample_uniform_for(space)):
        # the default samplers (acquisition.py:114-134) straight into rows, same RNG stream
        if not space.constraints:
            rows_h = sampling.uniform_rows(lay, n_candidates, ctx.rng)
        else:
            sc.set_constraints(space)
            rows_h = sampling.rejection_rows(
                lay, n_candidates, ctx.rng,
                lambda b: sc.constraints_eval(sc.to_device(b)).cpu().numpy().astype(bool))
        rows_h = sampling.unique_rows(rows_h)  # dict.fromkeys: first draws, in order
    else:
        if sample_fn is None:
            sample_fn = _default_sampler(space, cot)
        raw = sample_fn(n_candidates, ctx.rng)
        hit = _POOL_CACHE.get("k")
        if hit is not None and hit[0] is raw and hit[1] is lay and hit[2] == len(raw):
            rows_h = hit[3]  # the engine's enumerated small feasible set: the same list every iteration
        else:
            candidates = list(dict.fromkeys(raw))
            if candidates:
                rows_h = lay.encode(candidates)
                if isinstance(raw, list):
                    _POOL_CACHE["k"] = (raw, lay, len(raw), rows_h)
    if rows_h is None or len(rows_h) == 0:
        raise Exhausted("candidate sampler produced nothing")
    if cot is not None:
        sc.set_cot(cot)
    f_model = ctx.gp.objective_to_model(ctx.best_feasible_value)
    rows = sc.to_device(rows_h)
    many = local_search and n_starts > N.BX_MAX_K  # the fused top-k holds BX_MAX_K records
    summ, pool_vals, _ = sc.score(rows, f_model, ctx.eps_f, k=min(n_starts, N.BX_MAX_K),
                                  want_values=many, rf_pairwise=len(rows_h) == 1)
    if summ.n_finite == 0:  # acquisition.py:179-184
        if summ.best_prob is None:
            return _exhaustion_fallback(ctx, space, cot, sc, f_model, Exhausted)
        return lay.decode(rows_h[summ.best_prob.index])[0]

    best = summ.best
    if local_search:
        # the climb of every start runs on the device (bx_climb): per step one neighbour launch, the
        # scoring launches and one bookkeeping launch; one 4-byte read of the active count per four
        # steps.
        # Each start's trajectory depends only on its own state and the tracker is a maximum under a
        # total order (value desc, configuration asc), so the lockstep result equals the reference's
        # start-after-start loop (acquisition.py:186-205).
        if many:  # np.argsort(-values, kind="stable")[:n_starts] on the host (acquisition.py:188)
            v = pool_vals.cpu().numpy()
            order = [int(i) for i in np.argsort(-v, kind="stable")[:n_starts] if v[i] != -np.inf]
            starts = [(i, float(v[i])) for i in order]
        else:
            starts = [(st.index, st.value) for st in summ.top[:n_starts]]
        for c0 in range(0, len(starts), N.BX_MAX_K):
            chunk = starts[c0:c0 + N.BX_MAX_K]
            best, _ = sc.climb(rows, [i for i, _ in chunk], [v for _, v in chunk], cot is not None, f_model,
                               ctx.eps_f, best, MAX_CLIMB_STEPS)
    best_cfg = lay.decode(best.row)[0] if best is not None else None
    if best_cfg is None:
        return _exhaustion_fallback(ctx, space, cot, sc, f_model, Exhausted)
    return best_cfg


def _enumerate_feasible(space, cot, Exhausted):
    """acquisition.py:137-149."""
    import itertools

    if cot is not None:
        yield from cot.enumerate()
        return
    if any(p.kind == "real" for p in space.parameters):
        raise Exhausted("cannot enumerate a space with real parameters")
    doms = [list(range(int(p.lo), int(p.hi) + 1)) if p.kind == "integer"
            else list(p.values) if p.kind != "permutation"
            else [tuple(q) for q in itertools.permutations(range(1, p.size + 1))]
            for p in space.parameters]
    for batch in _chunks(itertools.product(*doms), 65536):
        ok = constraints_batch(space, batch) if space.constraints else [True] * len(batch)
        for cfg, good in zip(batch, ok):
            if good:
                yield cfg


def _chunks(it, n):
    buf = []
    for x in it:
        buf.append(x)
        if len(buf) == n:
            yield buf
            buf = []
    if buf:
        yield buf


_POOL_CACHE: dict = {}


def _exhaustion_fallback(ctx, space, cot, sc, f_model, Exhausted):
    """acquisition.py:209-222."""
    remaining = []
    for cfg in _enumerate_feasible(space, cot, Exhausted):
        if cfg not in ctx.evaluated:
            remaining.append(cfg)
            if len(remaining) >= 20_000:
                break
    if not remaining:
        raise Exhausted("every feasible configuration has been evaluated")
    rows = sc.to_device(sc.layout.encode(remaining))
    _, vals, probs = sc.score(rows, f_model, ctx.eps_f, k=0, want_values=True, summary=False,
                              rf_pairwise=len(remaining) == 1)
    v = vals.cpu().numpy()
    key = probs.cpu().numpy() if np.all(v == -np.inf) else v
    best = None
    for i, x in enumerate(key):
        if best is None or _better(x, remaining[i], key[best], remaining[best]):
            best = i
    return remaining[best]


_SQ_CACHE: dict = {}


def _device_sq(sc, sq_dists):
    """The (D, n, n) distance tensor on the device, cached across the ~200 objective calls of one
    gp_fit (the reference passes the same array object every time, surrogate.py:512)."""
    arr = np.ascontiguousarray(sq_dists, dtype=np.float64)
    key = (id(sq_dists), arr.shape, arr.ctypes.data)
    hit = _SQ_CACHE.get("k")
    if hit is not None and hit[0] == key and hit[2] is sq_dists:
        return hit[1]
    t = torch.as_tensor(arr, device=f"cuda:{sc.device}")
    _SQ_CACHE["k"] = (key, t, sq_dists)
    return t


def lml_core(sq_dists, z, sigma, noise, lengthscales, want_grad=False, prior=None):
    """`_lml_core` (surrogate.py:356-400) on the GPU: value, or (value, grad) with the gradient
    with respect to (log sigma, log noise, log l_1..l_D).  Raises numpy.linalg.LinAlgError when
    the Gram matrix is not positive definite, as the reference's np.linalg.cholesky does."""
    sc = scorer()
    dev = f"cuda:{sc.device}"
    sq = _device_sq(sc, sq_dists)
    zz = torch.as_tensor(np.ascontiguousarray(z, dtype=np.float64), device=dev)
    prm = np.concatenate([[float(sigma), float(noise)], np.asarray(lengthscales, dtype=np.float64)])
    params = torch.as_tensor(prm[None, :], device=dev)
    value, grad, ok = sc.lml_core(sq, zz, params, want_grad, prior)
    if int(ok.item()) == 0:
        raise np.linalg.LinAlgError("Matrix is not positive definite")
    if not want_grad:
        return float(value.item())
    return float(value.item()), grad[0].cpu().numpy()


def batched_coarse_lml(sq_dists, z, thetas):
    """`_batched_coarse_lml` (surrogate.py:420-456) on the GPU: one CTA per hyperparameter
    candidate, -inf where the Cholesky factorisation fails."""
    sc = scorer()
    dev = f"cuda:{sc.device}"
    sq = torch.as_tensor(np.ascontiguousarray(sq_dists, dtype=np.float64), device=dev)
    zz = torch.as_tensor(np.ascontiguousarray(z, dtype=np.float64), device=dev)
    th = torch.as_tensor(np.ascontiguousarray(thetas, dtype=np.float64), device=dev)
    return sc.lml_batched(sq, zz, th).cpu().numpy()
