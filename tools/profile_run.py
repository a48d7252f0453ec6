"""Short fixed workload for ncu captures: score the C3 1M pool `reps` times (default 3)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))

from golden_io import cot_for, load, model  # noqa: E402
from paper_2212_11142_b200 import scenarios  # noqa: E402
from paper_2212_11142_b200.device import scorer  # noqa: E402


def main(case="C3", reps=3, q=1 << 20):
    meta, arr, space = load(case)
    gp, feas = model(meta, arr, space)
    sc = scorer()
    sc.set_gp(gp)
    sc.set_forest(feas)
    cot = cot_for(case)
    rng = np.random.default_rng(0)
    rows_h = (scenarios.sample_rows_cot(sc.layout, cot, q, rng) if cot
              else scenarios.sample_rows_uniform(sc.layout, q, rng))
    rows = sc.to_device(rows_h)
    f_model = gp.objective_to_model(meta["f_best"])
    for _ in range(reps):
        summ, _, _ = sc.score(rows, f_model, meta["eps_f"], k=10)
    torch.cuda.synchronize()
    print("ok", summ.n_finite, summ.top[0].value)


if __name__ == "__main__":
    main(*(sys.argv[1:2] or ["C3"]), reps=int(sys.argv[2]) if len(sys.argv) > 2 else 3)
