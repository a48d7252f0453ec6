"""Short fixed workload for ncu captures: score a bench config's 1M device-generated pool `reps`
times through bx_score (posterior, forest + summary, merge).

    python tools/profile_run.py [M200|C3|C5] [reps]
"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))

import bench  # noqa: E402
from paper_2212_11142_b200.device import Scorer  # noqa: E402


def main(case="M200", reps=3, q=1 << 20):
    sc = Scorer()
    meta, space, gp, feas, cot = bench.load_workload(case, scorer=sc)
    sc.set_gp(gp)
    sc.set_forest(feas)
    if cot is not None:
        sc.set_cot(cot)
    rows = sc.generate(q, seed=1000, mode=bench.CONFIGS[case]["mode"])
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=rows.device)
    f_model = gp.objective_to_model(meta["f_best"])
    for _ in range(reps):
        flush.zero_()  # L2 flushed before every step, as in bench.py
        summ, _, _ = sc.score(rows, f_model, meta["eps_f"], k=10)
    torch.cuda.synchronize()
    print("ok", summ.n_finite, summ.top[0].value)


if __name__ == "__main__":
    main(*(sys.argv[1:2] or ["M200"]), reps=int(sys.argv[2]) if len(sys.argv) > 2 else 3)
