"""Forest-only timing on the M200 / C3 forests at small and large pool sizes (rf_qs_kernel through
bx_rf_predict, CUDA events, 200 repetitions): the fixed per-launch cost (table load) against the
per-candidate cost.  python tools/rf_small_q.py"""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2212_11142_b200.device import Scorer  # noqa: E402

sc = Scorer(0)
for name in ("M200", "C3"):
    meta, space, gp, feas, cot = bench.load_workload(name, scorer=sc)
    sc.set_gp(gp)
    sc.set_forest(feas)
    if cot is not None:
        sc.set_cot(cot)
    rows_all = sc.generate(1 << 20, seed=5, mode=bench.CONFIGS[name]["mode"])
    for q in (1, 32, 320, 1024, 4096, 1 << 16, 1 << 20):
        rows = rows_all[:q].contiguous()
        for pw in (False, True) if q <= 320 else (False,):
            for _ in range(5):
                sc.rf_predict(rows, pw)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 200 if q <= 1 << 16 else 20
            a.record()
            for _ in range(reps):
                sc.rf_predict(rows, pw)
            b.record()
            torch.cuda.synchronize()
            us = a.elapsed_time(b) * 1e3 / reps
            print(f"{name} q={q:8d} pairwise={int(pw)}: {us:9.2f} us per launch, {1e3 * us / q:9.2f} ns per candidate")
