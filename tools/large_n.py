"""C5 (d=10 mixed, n training points) on the device: which posterior kernel runs, its time on a
2^20 pool, and agreement with the oracle on a sample.  python tools/large_n.py [n]"""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import oracle  # noqa: E402  (checker only)
from paper_2212_11142_b200 import scenarios  # noqa: E402
from paper_2212_11142_b200.device import Scorer  # noqa: E402
from paper_2212_11142_b200.models import GPState, Hyper  # noqa: E402


def main(n=500, q=1 << 20):
    import os
    trace = os.environ.pop("LARGE_N_TRACE", None)  # file: CTA 0's role timeline of one predict
    if trace:
        os.environ["BX_TC_TRACE"] = ""
    space = scenarios.build_space("C5")
    rng = np.random.default_rng(5)
    sc = Scorer()
    lay = sc.set_space(space)
    train_rows = scenarios.sample_rows_uniform(lay, n, rng)
    cfgs = lay.decode(train_rows)
    y = np.array([scenarios.objective("C5", c) for c in cfgs])
    hyp = Hyper(outputscale=1.7, noise_variance=1e-4, lengthscales=tuple(rng.uniform(0.8, 3.0, len(space.parameters))))
    gp = GPState.fit(space, cfgs, y, hyp, scorer=sc)
    sc.set_gp(gp)
    print("n", n, "kernel", sc.gp_kernel())
    rows = sc.to_device(scenarios.sample_rows_uniform(lay, q, rng))
    sc.predict(rows)
    torch.cuda.synchronize()
    ts = []
    for _ in range(6):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        mean, var = sc.predict(rows)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = float(np.median(ts))
    if trace:
        os.environ["BX_TC_TRACE"] = trace
        sc.predict(rows)
        torch.cuda.synchronize()
        del os.environ["BX_TC_TRACE"]
    print(f"predict 2^20: {ms:.3f} ms  {q / ms * 1e3:,.0f} cand/s  (runs: {' '.join(f'{t:.2f}' for t in ts)})")
    sample = lay.decode(rows[:2000].cpu().numpy().view(np.uint32))
    og = oracle.OracleGP(space, gp.configs, hyp.outputscale, hyp.noise_variance, hyp.lengthscales,
                         L=gp._cho[0], alpha=gp.alpha, y_mean=gp.y_mean, y_std=gp.y_std)
    m0, v0 = oracle.gp.predict(og, sample)
    m1, v1 = mean[:2000].cpu().numpy(), var[:2000].cpu().numpy()
    print("max rel mean err %.2e var err %.2e" % (np.max(np.abs(m1 - m0) / np.maximum(np.abs(m0), 1e-12)),
                                                   np.max(np.abs(v1 - v0) / np.abs(v0))))

if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 500)
