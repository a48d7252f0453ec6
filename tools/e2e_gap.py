"""Where the end-to-end leg's extra time goes (M200): per-step event times of bx_score on device
rows, bx_score_host on packed pinned rows (zero-copy) and the same call's host-side overhead
(wall clock around the call minus the device span).  python tools/e2e_gap.py [steps]"""
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2212_11142_b200.device import Scorer  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
sc = Scorer(0)
meta, space, gp, feas, cot = bench.load_workload("M200", scorer=sc)
sc.set_gp(gp)
sc.set_forest(feas)
q = 1 << 20
rows = sc.generate(q, seed=1000, mode=0)
rows_h = rows.cpu().numpy().view(np.uint32)
packed_h = torch.from_numpy(sc.pack(rows_h).view(np.int32)).pin_memory().numpy().view(np.uint32)
f_model = gp.objective_to_model(meta["f_best"])
eps = meta["eps_f"]
stream = torch.cuda.current_stream()


def run(name, fn):
    for _ in range(3):
        fn()
    ev, wall = [], []
    for _ in range(steps):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t = time.perf_counter()
        a.record(stream)
        fn()
        b.record(stream)
        b.synchronize()
        wall.append((time.perf_counter() - t) * 1e3)
        ev.append(a.elapsed_time(b))
    print(f"{name:34s} events {np.median(ev):.3f} ms  wall {np.median(wall):.3f} ms")


run("bx_score device rows", lambda: sc.score(rows, f_model, eps, k=10))
run("bx_score device rows + timing", lambda: sc.score(rows, f_model, eps, k=10, timing=True))
print("   kernels:", sc.last_timing())
run("bx_score_host packed pinned", lambda: sc.score_host(packed_h, f_model, eps, k=10, packed=True))
rows_pinned = torch.from_numpy(rows_h.view(np.int32)).pin_memory().numpy().view(np.uint32)
run("bx_score_host encoded pinned", lambda: sc.score_host(rows_pinned, f_model, eps, k=10))
