"""Wall time per BO iteration of the patched loop split by the replaced entry points (gp_fit,
rf_fit, optimize_acquisition) and the rest, without a profiler.  python tools/engine_breakdown.py"""
import sys
import time
from collections import defaultdict
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from golden_io import ref  # noqa: E402
from paper_2212_11142_b200 import scenarios  # noqa: E402
from paper_2212_11142_b200.patch import install  # noqa: E402


def main(budget=40, seed=1, fit=True, lml=True):
    bt = ref()
    space = scenarios.build_space("C5", bt.space)
    bench = bt.Benchmark("m200-mixed", space, lambda c: scenarios.objective("C5", c),
                         hidden_rule=lambda c: scenarios.hidden_ok("M200", c), default_budget=budget)
    spent = defaultdict(float)

    def timed(mod, attr):
        fn = getattr(mod, attr)

        def wrapper(*a, **k):
            t = time.perf_counter()
            try:
                return fn(*a, **k)
            finally:
                spent[attr] += time.perf_counter() - t
        setattr(mod, attr, wrapper)
        return lambda: setattr(mod, attr, fn)

    for label, patched in (("reference", False), ("b200", True)):
        undo = install(bt, whole_path=True, lml=lml, fit=fit) if patched else (lambda: None)
        undos = [timed(bt.engine, a) for a in ("gp_fit", "rf_fit", "optimize_acquisition")]
        try:
            for rep in range(2 if patched else 1):  # patched: a warm-up run first
                spent.clear()
                sc = bt.Scenario(name=bench.name, space=space, budget=budget, seed=seed)
                t0 = time.perf_counter()
                r = bt.run_bo_loop(sc, bench, np.random.default_rng(seed))
                total = time.perf_counter() - t0
        finally:
            for u in undos:
                u()
            undo()
        n_bo = sum(rec.phase == "bo" for rec in r.history)
        parts = {k: 1e3 * v / n_bo for k, v in spent.items()}
        rest = 1e3 * total / n_bo - sum(parts.values())
        print(f"{label:10s} per BO iteration (ms): " + ", ".join(f"{k} {v:.1f}" for k, v in parts.items())
              + f", rest {rest:.1f}; total {1e3 * total / n_bo:.1f} over {n_bo} iterations")


if __name__ == "__main__":
    main()
