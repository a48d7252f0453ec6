"""BASELINE.json configs[4]: the candidate-pool sweep 1M .. 1B on one GPU, pools generated on the
device chunk by chunk (bx_score_generated: Philox rows -> posterior -> forest + summary, running
merge; nothing materialised beyond a 2^22-row chunk), CUDA-event timed.

    python tools/sweep_generated.py [C5|M200|C3] [max log2 pool] > profiles/r02_sweep_<config>.txt
"""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import bench  # noqa: E402
from paper_2212_11142_b200.device import Scorer  # noqa: E402


def main(name="C5", max_log2=30):
    sc = Scorer()
    meta, space, gp, feas, cot = bench.load_workload(name, scorer=sc)
    sc.set_gp(gp)
    sc.set_forest(feas)
    if cot is not None:
        sc.set_cot(cot)
    f = gp.objective_to_model(meta["f_best"])
    mode = bench.CONFIGS[name]["mode"]
    print(f"{name}: n = {len(gp.configs)}, d = {len(space.parameters)}, kernel {sc.gp_kernel()}, "
          f"k-steps {sc.distance_ksteps()}; device-generated pools (mode {mode}), top-10 + trackers")
    sc.score_generated(1 << 22, seed=1, f_model=f, eps_f=meta["eps_f"], k=10, mode=mode)  # warm-up
    for lg in range(20, max_log2 + 1, 2 if max_log2 - 20 > 6 else 1):
        q = 1 << lg
        runs = []
        with bench.ClockSampler(sc.device) as clocks:
            for _ in range(3 if lg <= 26 else 1):
                torch.cuda.synchronize()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                s = sc.score_generated(q, seed=7, f_model=f, eps_f=meta["eps_f"], k=10, mode=mode)
                b.record()
                b.synchronize()
                runs.append(a.elapsed_time(b))
        ms = min(runs)
        c = clocks.summary()
        print(f"  pool 2^{lg:2d} = {q:>13,d}: {ms:10.2f} ms  {q / ms * 1e3:14,.0f} cand/s  "
              f"(n_finite {s.n_finite:,d}, best {s.top[0].value:.6g} at index {s.top[0].index}; runs "
              f"{', '.join(f'{r:.1f}' for r in runs)} ms; SM {c['sm_mhz']} MHz {c['reasons']})")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "C5", int(sys.argv[2]) if len(sys.argv) > 2 else 30)
