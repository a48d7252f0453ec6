"""gp_fit: the reference's vs hyperfit.gp_fit wall time, batched objective calls and the time spent
inside them.  python tools/fit_small_n.py [case] [--lml]  (--lml: the GPU coarse LML stage too,
as install(lml=True) routes it; BASELINE configs[3] is case C4)"""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from golden_io import ref  # noqa: E402
from paper_2212_11142_b200 import hyperfit, scenarios  # noqa: E402


def main(case="C5", lml=False):
    bt = ref()
    space = scenarios.build_space(case, bt.space)
    if lml:
        from paper_2212_11142_b200.patch import install
        install(bt, whole_path=False, lml=True, fit=False, rf=False)
    for n in (10, 20, 40, 100, 200):
        rng = np.random.default_rng(n)
        cfgs = list(dict.fromkeys(bt.space.sample_uniform(space, n + 20, rng)))[:n]
        y = np.array([scenarios.objective(case, c) for c in cfgs])
        t = time.perf_counter()
        bt.surrogate.gp_fit(space, cfgs, y, np.random.default_rng(1))
        t_ref = time.perf_counter() - t
        hyperfit.gp_fit(space, cfgs, y, np.random.default_rng(1))  # warm-up
        spent = [0.0]
        orig = hyperfit.scorer

        class Timed:
            def __init__(self, sc):
                self.sc = sc

            def __getattr__(self, a):
                f = getattr(self.sc, a)
                if a not in ("lml_core", "lml_core_host"):
                    return f

                def g(*args, **kw):
                    t0 = time.perf_counter()
                    try:
                        return f(*args, **kw)
                    finally:
                        spent[0] += time.perf_counter() - t0
                return g
        hyperfit.scorer = lambda: Timed(orig())
        try:
            t = time.perf_counter()
            hyperfit.gp_fit(space, cfgs, y, np.random.default_rng(1))
            t_gpu = time.perf_counter() - t
        finally:
            hyperfit.scorer = orig
        print(f"{case} n {n:4d}: reference {t_ref * 1e3:7.1f} ms, hyperfit {t_gpu * 1e3:7.1f} ms "
              f"({hyperfit.gp_fit.last_batched_calls} batched calls, {spent[0] * 1e3:.1f} ms in lml_core incl. copies)")


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    main(args[0] if args else "C5", "--lml" in sys.argv)
