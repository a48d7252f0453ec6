"""Whole BO loop of the shipped reference (run_bo_loop, engine.py:294-331) on the north-star space
(d = 10 mixed, hidden rule t1 * t2 <= 4096), as shipped and with the B200 path installed
(patch.install(boxtune, lml=True, fit=True)): wall time per BO iteration and history equality.

    python tools/engine_bench.py [budget] [seed] > profiles/r02_engine.txt
"""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from golden_io import ref  # noqa: E402
from paper_2212_11142_b200 import scenarios  # noqa: E402
from paper_2212_11142_b200.patch import install  # noqa: E402


def main(budget=40, seed=1):
    bt = ref()
    space = scenarios.build_space("C5", bt.space)
    bench = bt.Benchmark("m200-mixed", space, lambda c: scenarios.objective("C5", c),
                         hidden_rule=lambda c: scenarios.hidden_ok("M200", c), default_budget=budget)
    times = {}

    def run(label):
        stamps = []
        sc = bt.Scenario(name=bench.name, space=space, budget=budget, seed=seed)
        t0 = time.perf_counter()
        r = bt.run_bo_loop(sc, bench, np.random.default_rng(seed), on_record=lambda rec: stamps.append(time.perf_counter()))
        times[label] = (time.perf_counter() - t0, stamps, r)
        return r

    want = run("reference")
    undo = install(bt, whole_path=True, lml=True, fit=True)
    try:
        run("b200 (warm-up)")
        got = run("b200")
    finally:
        undo()
    for label in ("reference", "b200"):
        total, stamps, r = times[label]
        bo = [i for i, rec in enumerate(r.history) if rec.phase == "bo"]
        per = np.diff([stamps[i - 1] for i in bo] + [stamps[bo[-1]]]) if bo else []
        print(f"{label:10s}: {len(r.history)} evaluations ({len(bo)} BO), total {total:.2f} s, "
              f"BO iteration mean {np.mean(per) * 1e3:.1f} ms, last {per[-1] * 1e3:.1f} ms; "
              f"best {r.best_feasible()[1]:.6f}")
    same = got.history == want.history
    first = next((i for i, (a, b) in enumerate(zip(got.history, want.history)) if a != b), None)
    print(f"histories identical: {same}" + ("" if same else f" (first divergence at evaluation {first})"))


if __name__ == "__main__":
    main(*(int(x) for x in sys.argv[1:3]))
