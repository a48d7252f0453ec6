"""Smallest end-to-end scoring run for compute-sanitizer (one tool per gpurun call):

    compute-sanitizer --tool synccheck python tools/sanitize_case.py
    compute-sanitizer --tool memcheck  python tools/sanitize_case.py

Scores a ragged pool (3 tiles + 17 rows) of the north-star M200 space and of C3 through the
device-resident path (posterior on the tensor cores, QuickScorer forest + summary, merge) and the
streamed packed host path, and one n = 300 (two column passes) posterior."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from golden_io import load, model  # noqa: E402
from paper_2212_11142_b200 import scenarios  # noqa: E402
from paper_2212_11142_b200.device import Scorer  # noqa: E402
from paper_2212_11142_b200.models import GPState, Hyper  # noqa: E402

q = 3 * 128 + 17
for case in ("M200", "C3"):
    meta, arr, space = load(case)
    gp, feas = model(meta, arr, space)
    sc = Scorer()
    sc.set_gp(gp)
    sc.set_forest(feas)
    rows_h = scenarios.sample_rows_uniform(sc.layout, q, np.random.default_rng(1))
    f = gp.objective_to_model(meta["f_best"])
    s, v, p = sc.score(sc.to_device(rows_h), f, meta["eps_f"], k=10, want_values=True)
    pk = torch.from_numpy(sc.pack(rows_h).view(np.int32)).pin_memory().numpy().view(np.uint32)
    s2 = sc.score_host(pk, f, meta["eps_f"], k=10, packed=True)
    assert [c.index for c in s.top] == [c.index for c in s2.top]
    print(case, "ok", sc.gp_kernel(), sc.distance_ksteps(), s.n_finite)
    sc.close()
space = scenarios.build_space("C5")
sc = Scorer()
lay = sc.set_space(space)
rng = np.random.default_rng(3)
cfgs = list(dict.fromkeys(lay.decode(scenarios.sample_rows_uniform(lay, 400, rng))))[:300]
gp = GPState.fit(space, cfgs, [scenarios.objective("C5", c) for c in cfgs],
                 Hyper(1.2, 1e-3, tuple(rng.uniform(0.8, 2.0, 10))), log_objective=True, scorer=sc)
sc.set_gp(gp)
m, var = sc.predict(sc.to_device(scenarios.sample_rows_uniform(lay, q, rng)))
torch.cuda.synchronize()
print("n=300 ok", sc.gp_kernel(), sc.distance_ksteps(), float(var.min()))
