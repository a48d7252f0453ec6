"""Device time of the hyperparameter-fit kernels (rows a14 / a15) against the CPU restatement
(development aid).  python tools/lml_bench.py [n ...]"""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import oracle  # noqa: E402  (checker / CPU baseline only)
from paper_2212_11142_b200 import acquisition as A  # noqa: E402
from paper_2212_11142_b200 import scenarios  # noqa: E402
from paper_2212_11142_b200.device import scorer  # noqa: E402


def main(ns=(200, 500), D=10, c=64):
    rng = np.random.default_rng(0)
    for n in ns:
        X = rng.uniform(0, 1, (n, D))
        sq = np.stack([(X[:, k, None] - X[None, :, k]) ** 2 for k in range(D)])
        z = rng.standard_normal(n)
        ls = rng.uniform(0.3, 2.0, D)
        args = (sq, z, 1.3, 1e-3, ls)
        A.lml_core(*args, want_grad=True)  # warm-up (uploads, allocations)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(5):
            v, g = A.lml_core(*args, want_grad=True)
        dt = (time.perf_counter() - t0) / 5
        t0 = time.perf_counter()
        v0, g0 = oracle.lml_core(*args, want_grad=True, prior=None)
        dc = time.perf_counter() - t0
        print(f"n={n} _lml_core+grad: device {dt * 1e3:8.2f} ms/call  cpu {dc * 1e3:8.2f} ms  "
              f"|dv| {abs(v - v0):.2e} max|dg| {np.max(np.abs(g - g0)):.2e}")
        th = np.concatenate([np.log([[1.3, 1e-3]]).repeat(c, 0), np.log(rng.uniform(0.3, 2.0, (c, D)))], 1)
        A.batched_coarse_lml(sq, z, th)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            out = A.batched_coarse_lml(sq, z, th)
        dt = (time.perf_counter() - t0) / 3
        t0 = time.perf_counter()
        ref = oracle.lml.coarse_lml(sq, z, th)
        dc = time.perf_counter() - t0
        ok = np.isfinite(ref)
        print(f"n={n} coarse LML x{c}: device {dt * 1e3:8.2f} ms/call  cpu {dc * 1e3:8.2f} ms  "
              f"max|d| {np.max(np.abs(out[ok] - ref[ok])):.2e}")


if __name__ == "__main__":
    main(tuple(int(a) for a in sys.argv[1:]) or (200, 500))
