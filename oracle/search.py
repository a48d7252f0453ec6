"""optimize_acquisition restated (acquisition.py:87-206) over the oracle scorer.  Test-only."""
from __future__ import annotations

import math

import numpy as np

from .gp import scores
from .moves import neighbors


def _pick(configs, values):
    best = None
    for i, v in enumerate(values):
        if best is None or v > values[best] or (v == values[best] and configs[i] < configs[best]):
            best = i
    return best


def optimize(gp, forest, space, pool, f_best, eps_f, evaluated, cot=None, local_search=True,
             n_starts=10, max_steps=50):
    cands = list(dict.fromkeys(pool))
    vals, probs = scores(gp, forest, cands, f_best, eps_f)
    state = {"cfg": None, "v": -math.inf}

    def track(cfgs, vs):
        for c, v in zip(cfgs, vs):
            if v == -math.inf or c in evaluated:
                continue
            if v > state["v"] or (v == state["v"] and (state["cfg"] is None or c < state["cfg"])):
                state["cfg"], state["v"] = c, v

    if np.all(vals == -np.inf):
        track(cands, probs)
        return state["cfg"]
    track(cands, vals)
    if local_search:
        for i in np.argsort(-vals, kind="stable")[:n_starts]:
            if vals[i] == -np.inf:
                continue
            cur, cur_v = cands[i], vals[i]
            for _ in range(max_steps):
                nb = neighbors(space, cur, cot)
                if not nb:
                    break
                nv, _ = scores(gp, forest, nb, f_best, eps_f)
                track(nb, nv)
                j = _pick(nb, nv)
                if nv[j] <= cur_v:
                    break
                cur, cur_v = nb[j], nv[j]
    return state["cfg"]
