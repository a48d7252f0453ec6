"""Forest-only workload for ncu captures: C3 model, 1M pool, rf_predict `reps` times."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))

from golden_io import cot_for, load, model  # noqa: E402
from paper_2212_11142_b200 import scenarios  # noqa: E402
from paper_2212_11142_b200.device import scorer  # noqa: E402

meta, arr, space = load("C3")
gp, feas = model(meta, arr, space)
sc = scorer()
sc.set_gp(gp)
sc.set_forest(feas)
rows = sc.to_device(scenarios.sample_rows_cot(sc.layout, cot_for("C3"), 1 << 20, np.random.default_rng(0)))
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    p = sc.rf_predict(rows, pairwise=False)
torch.cuda.synchronize()
print("ok", float(p.mean()))
