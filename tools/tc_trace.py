"""Role timeline of CTA 0 of the tensor-core posterior kernel (development aid).

    python tools/tc_trace.py [case] [q]          -> gpurun_out/tc_trace.bin, then
    python tools/tc_trace.py --show gpurun_out/tc_trace.bin
"""
import os
import sys
from pathlib import Path

import numpy as np

ROLES = ["producer", "mma", "epilogue", "tma"]
CODES = {"producer": {1: "tile-start", 2: "decoded", 3: "slice-computed", 4: "slice-free", 5: "slice-sync",
                      6: "cand-full"},
         "mma": {1: "wait-cand", 2: "cand-ok", 3: "chunk-issued"},
         "epilogue": {1: "acc-ready", 2: "acc-drained"},
         "tma": {1: "stage-free"}}


def show(path, tiles=3):
    t = np.fromfile(path, dtype=np.int64).reshape(4, 4096, 2)
    t0 = min(int(t[r, 0, 0]) for r in range(4) if t[r, 0, 0])
    for r, name in enumerate(ROLES):
        ev = t[r][t[r, :, 0] != 0]
        print(f"== {name}: {len(ev)} events")
        lim = {"producer": 40 * tiles, "mma": 10 * tiles, "epilogue": 16 * tiles, "tma": 30 * tiles}[name]
        for clk, code in ev[:lim]:
            print(f"  {clk - t0:>9d}  {CODES[name].get(int(code) >> 16, '?'):15s} {int(code) & 0xFFFF}")
        if name == "mma" and len(ev) > 4:
            starts = ev[(ev[:, 1] >> 16) == 2][:, 0]
            if len(starts) > 2:
                print("  tile period (clk):", np.diff(starts)[:12].tolist(), "mean", float(np.diff(starts).mean()))


def run(case="C3", q=1 << 20):
    sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
    sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
    import torch
    from golden_io import cot_for, load, model
    from paper_2212_11142_b200 import scenarios
    from paper_2212_11142_b200.device import scorer
    meta, arr, space = load(case)
    gp, feas = model(meta, arr, space)
    os.environ["BX_TC_TRACE"] = ""  # present at handle creation (enables the per-launch check), empty = off
    sc = scorer()
    sc.set_gp(gp)
    rng = np.random.default_rng(0)
    cot = cot_for(case)
    rows_h = (scenarios.sample_rows_cot(sc.layout, cot, q, rng) if cot
              else scenarios.sample_rows_uniform(sc.layout, q, rng))
    rows = sc.to_device(rows_h)
    sc.predict(rows)
    torch.cuda.synchronize()
    Path("gpurun_out").mkdir(exist_ok=True)
    os.environ["BX_TC_TRACE"] = "gpurun_out/tc_trace.bin"
    sc.predict(rows)
    torch.cuda.synchronize()
    del os.environ["BX_TC_TRACE"]
    print("kernel:", sc.gp_kernel())
    show("gpurun_out/tc_trace.bin")


if __name__ == "__main__":
    if sys.argv[1:2] == ["--show"]:
        show(sys.argv[2])
    else:
        run(*(sys.argv[1:2] or ["C3"]))
