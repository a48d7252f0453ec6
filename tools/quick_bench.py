"""Quick device timing of the fused scorer on a golden model (development aid, not the bench)."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))

from golden_io import cot_for, load, model  # noqa: E402
from paper_2212_11142_b200 import scenarios  # noqa: E402
from paper_2212_11142_b200.device import scorer  # noqa: E402


def main(case="C3", q=1 << 20, reps=5):
    meta, arr, space = load(case)
    gp, feas = model(meta, arr, space)
    sc = scorer()
    sc.set_gp(gp)
    sc.set_forest(feas)
    lay = sc.layout
    rng = np.random.default_rng(0)
    cot = cot_for(case)
    rows_h = scenarios.sample_rows_cot(lay, cot, q, rng) if cot else scenarios.sample_rows_uniform(lay, q, rng)
    rows = sc.to_device(rows_h)
    f_model = gp.objective_to_model(meta["f_best"])
    for name, fn in [
        ("score+summary", lambda: sc.score(rows, f_model, meta["eps_f"], k=10)),
        ("score no-summary", lambda: sc.score(rows, f_model, meta["eps_f"], k=10, summary=False)),
        ("rf only", lambda: sc.rf_predict(rows, pairwise=False)),
        ("gp predict", lambda: sc.predict(rows)),
    ]:
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ms = min(ts)
        print(f"{case} n={gp._cho[0].shape[0]} q={q} {name:18s} {ms:8.3f} ms  {q / ms * 1e3:,.0f} cand/s")
    sc.score(rows, f_model, meta["eps_f"], k=10, timing=True)
    print("kernel timing (ms):", {k: round(v, 3) for k, v in sc.last_timing().items()})
    pinned = torch.from_numpy(rows_h.view(np.int32)).pin_memory()
    sc.score_host(pinned.numpy().view(np.uint32), f_model, meta["eps_f"], k=10)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        sc.score_host(pinned.numpy().view(np.uint32), f_model, meta["eps_f"], k=10)
    dt = (time.perf_counter() - t0) / reps
    print(f"{case} e2e host pool        {dt * 1e3:8.3f} ms  {q / dt:,.0f} cand/s")


if __name__ == "__main__":
    main(*(sys.argv[1:2] or ["C3"]))
