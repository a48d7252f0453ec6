"""Hill-climb statistics inside the patched BO loop (C5 space, 40 evaluations): per bx_climb call
the number of starts, steps and wall time, and the kernels one step launches (with
CUDA_LAUNCH_BLOCKING unset).  python tools/climb_stats.py"""
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from golden_io import ref  # noqa: E402
from paper_2212_11142_b200 import device, scenarios  # noqa: E402
from paper_2212_11142_b200.patch import install  # noqa: E402

bt = ref()
space = scenarios.build_space("C5", bt.space)
bench = bt.Benchmark("m200-mixed", space, lambda c: scenarios.objective("C5", c),
                     hidden_rule=lambda c: scenarios.hidden_ok("M200", c), default_budget=40)
install(bt, whole_path=True, lml=True, fit=True)
log = []
orig = device.Scorer.climb


def climb(self, pool_rows, start_index, *a, **k):
    torch.cuda.synchronize()
    t = time.perf_counter()
    out = orig(self, pool_rows, start_index, *a, **k)
    log.append((len(start_index), out[1], time.perf_counter() - t, self.n_slots))
    return out


device.Scorer.climb = climb
run = lambda: bt.run_bo_loop(bt.Scenario(name=bench.name, space=space, budget=40, seed=1), bench,
                             np.random.default_rng(1))
run()
log.clear()
run()
starts, steps, secs, slots = (np.array(v) for v in zip(*log))
print(f"{len(log)} climbs: starts {starts.mean():.1f}, slots {slots.mean():.0f}, steps mean {steps.mean():.1f} "
      f"max {steps.max()}, {1e3 * secs.mean():.2f} ms per climb, {1e6 * secs.sum() / steps.sum():.0f} us per step")
