"""bx_lml_core (value + gradient, c settings) and bx_lml_batched (coarse values, 64 settings) at
several n, per call (wall, including the result read): python tools/lml_bench2.py"""
import os
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
from paper_2212_11142_b200.device import Scorer  # noqa: E402


def timeit(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    return (time.perf_counter() - t) / reps * 1e3


def main():
    bt = ref()
    S = bt.surrogate
    space = scenarios.build_space("C4", bt.space)
    sc = Scorer()
    lay = sc.set_space(space)
    prior = S.LengthscalePrior()
    label = os.environ.get("BX_LML_NARROW", "0") == "1" and "narrow" or "wide"
    for n in tuple(int(x) for x in os.environ.get("LML_NS", "20,40,100,200,300").split(",")):
        rng = np.random.default_rng(n)
        cfgs = list(dict.fromkeys(bt.space.sample_uniform(space, n + 20, rng)))[:n]
        y = np.array([scenarios.objective("C4", c) for c in cfgs])
        z, _, _ = S._standardize(np.log(y))
        rows = sc.to_device(lay.encode(cfgs))
        sq = sc.pairwise_sq(rows, rows)
        zd = torch.as_tensor(z, device="cuda")
        prm = torch.as_tensor(np.exp(rng.uniform(-1, 1, size=(8, 2 + space.dimension))), device="cuda")
        th = torch.as_tensor(rng.uniform(-1, 1, size=(64, 2 + space.dimension)), device="cuda")
        t_core = timeit(lambda: sc.lml_core(sq, zd, prm, True, prior)[0].cpu())
        t_coarse = timeit(lambda: sc.lml_batched(sq, zd, th).cpu())
        print(f"{label:6s} n {n:4d}: lml_core x8 {t_core:7.3f} ms, coarse x64 {t_coarse:7.3f} ms")


if __name__ == "__main__":
    main()
