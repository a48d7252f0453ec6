"""Where optimize_acquisition's time goes inside the patched BO loop (M200 space, n <= 40):
cProfile of the B200 run only, sorted by own time.  python tools/prof_acq.py"""
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

bt = ref()
space = scenarios.build_space("C5", bt.space)
bench = bt.Benchmark("m200-mixed", space, lambda c: scenarios.objective("C5", c),
                     hidden_rule=lambda c: scenarios.hidden_ok("M200", c), default_budget=40)
install(bt, whole_path=True, lml=True, fit=True)
run = lambda: bt.run_bo_loop(bt.Scenario(name=bench.name, space=space, budget=40, seed=1), bench,
                             np.random.default_rng(1))
run()
cProfile.run("run()", "/tmp/acq.prof")
pstats.Stats("/tmp/acq.prof").sort_stats("tottime").print_stats(25)
