"""Whole-path timing of the drop-in optimize_acquisition (row a9) on a golden model: pool scoring
plus the local search (development aid).  python tools/acq_bench.py [case] [pool]"""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))

from golden_io import Ctx, cot_for, load, model, to_cfg  # noqa: E402
from paper_2212_11142_b200 import acquisition as A  # noqa: E402
from paper_2212_11142_b200 import scenarios  # noqa: E402
from paper_2212_11142_b200.device import scorer  # noqa: E402


def main(case="C3", q=5000):
    meta, arr, space = load(case)
    gp, feas = model(meta, arr, space)
    cot = cot_for(case)
    ev = {to_cfg(space, c) for c in meta["evaluated"]}
    sc = scorer()
    lay = sc.set_space(space, meta["use_transforms"])
    rng = np.random.default_rng(1)
    rows = scenarios.sample_rows_cot(lay, cot, q, rng) if cot else scenarios.sample_rows_uniform(lay, q, rng)
    pool = lay.decode(rows)
    calls = {"neighbors": 0, "score": 0, "climb_ms": 0.0, "steps": 0}
    orig_nb, orig_score, orig_climb = sc.neighbors, sc.score, sc.climb

    def climb(*a, **k):
        torch.cuda.synchronize()
        t = time.perf_counter()
        out = orig_climb(*a, **k)
        calls["climb_ms"] += (time.perf_counter() - t) * 1e3
        calls["steps"] += out[1]
        return out

    def nb(*a, **k):
        calls["neighbors"] += 1
        return orig_nb(*a, **k)

    def score(*a, **k):
        calls["score"] += 1
        return orig_score(*a, **k)

    sc.neighbors, sc.score, sc.climb = nb, score, climb
    for rep in range(3):
        ctx = Ctx(gp, feas, meta["f_best"], meta["eps_f"], np.random.default_rng(0), ev)
        calls.update(neighbors=0, score=0, climb_ms=0.0, steps=0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        got = A.optimize_acquisition(ctx, space, cot, sample_fn=lambda n, r: pool)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(f"{case} pool {q}: optimize_acquisition {dt * 1e3:8.1f} ms  ({calls['score']} score calls, "
              f"{calls['neighbors']} neighbour calls; device climb {calls['climb_ms']:.2f} ms, "
              f"{calls['steps']} steps)")
    t0 = time.perf_counter()
    enc = lay.encode(pool)
    print(f"host encode of the pool: {(time.perf_counter() - t0) * 1e3:.1f} ms")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "C3", int(sys.argv[2]) if len(sys.argv) > 2 else 5000)
