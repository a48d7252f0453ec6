"""Per-call cost of the L-BFGS-B objective call (bx_lml_core_host, 8 settings) at small n: wall
time per call against the kernel's own duration (run under ncu for the latter).
python tools/lml_call_probe.py"""
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from golden_io import ref  # noqa: E402
from paper_2212_11142_b200 import scenarios  # noqa: E402
from paper_2212_11142_b200.device import scorer  # noqa: E402

bt = ref()
space = scenarios.build_space("C5", bt.space)
sc = scorer()
lay = sc.set_space(space)
S = bt.surrogate
for n in (10, 40):
    rng = np.random.default_rng(n)
    rows = sc.to_device(scenarios.sample_rows_uniform(lay, n, rng))
    sq = sc.pairwise_sq(rows, rows)
    z = torch.as_tensor(rng.standard_normal(n), device="cuda")
    prm = np.exp(rng.uniform(-1, 1, size=(8, 2 + space.dimension)))
    prior = S.LengthscalePrior()
    for _ in range(20):
        sc.lml_core_host(sq, z, prm, prior)
    reps = 300
    t = time.perf_counter()
    for _ in range(reps):
        sc.lml_core_host(sq, z, prm, prior)
    print(f"n {n}: {1e6 * (time.perf_counter() - t) / reps:.1f} us per call (wall)")
