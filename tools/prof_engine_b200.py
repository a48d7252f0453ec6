"""cProfile of the patched BO loop alone (C5 space, 40 evaluations, after a warm-up run):
where the host time of a BO iteration goes.  python tools/prof_engine_b200.py [out.prof]"""
import cProfile
import pstats
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from golden_io import ref  # noqa: E402
from paper_2212_11142_b200 import scenarios  # noqa: E402
from paper_2212_11142_b200.patch import install  # noqa: E402


def main(out="gpurun_out/engine_b200.prof", budget=40, seed=1):
    bt = ref()
    space = scenarios.build_space("C5", bt.space)
    bench = bt.Benchmark("m200-mixed", space, lambda c: scenarios.objective("C5", c),
                         hidden_rule=lambda c: scenarios.hidden_ok("M200", c), default_budget=budget)
    install(bt, whole_path=True, lml=True, fit=True)

    def run():
        sc = bt.Scenario(name=bench.name, space=space, budget=budget, seed=seed)
        return bt.run_bo_loop(sc, bench, np.random.default_rng(seed))

    run()
    prof = cProfile.Profile()
    prof.enable()
    run()
    prof.disable()
    prof.dump_stats(out)
    st = pstats.Stats(out)
    st.sort_stats("tottime").print_stats(40)
    st.sort_stats("cumulative").print_stats(40)


if __name__ == "__main__":
    main(*sys.argv[1:2])
