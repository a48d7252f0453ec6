"""Device scoring throughput of every golden case on a 2^20 pool (development aid)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))

from golden_io import CASES, load, model  # noqa: E402
from paper_2212_11142_b200 import scenarios  # noqa: E402
from paper_2212_11142_b200.device import Scorer  # noqa: E402


def main(q=1 << 20):
    for case in CASES:
        meta, arr, space = load(case)
        gp, feas = model(meta, arr, space)
        sc = Scorer()
        sc.set_gp(gp)
        if feas is not None:
            sc.set_forest(feas)
        rows = sc.to_device(scenarios.sample_rows_uniform(sc.layout, q, np.random.default_rng(1)))
        f = gp.objective_to_model(meta["f_best"])
        sc.score(rows, f, meta["eps_f"], k=10)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(3):
            sc.score(rows, f, meta["eps_f"], k=10)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 3
        kinds = {}
        for p in space.parameters:
            kinds[p.kind] = kinds.get(p.kind, 0) + 1
        print(f"{case:14s} n={len(gp.configs):4d} d={len(space.parameters):2d} {kinds} forest={feas is not None} "
              f"kernel={sc.gp_kernel():7s} ks={sc.distance_ksteps()} {ms:7.3f} ms  {q / ms * 1e3:,.0f} cand/s")
        sc.close()


if __name__ == "__main__":
    main()
