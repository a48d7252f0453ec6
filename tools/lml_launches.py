"""One batched bx_lml_core call (8 settings, C4 space, n = 200) repeated, for an ncu launch list:
    ncu --metrics gpu__time_duration.sum --csv python tools/lml_launches.py"""
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from golden_io import ref  # noqa: E402
from paper_2212_11142_b200 import scenarios  # noqa: E402
from paper_2212_11142_b200.device import scorer  # noqa: E402


def main(n=200, c=8, reps=5):
    bt = ref()
    space = scenarios.build_space("C4", bt.space)
    rng = np.random.default_rng(n)
    cfgs = list(dict.fromkeys(bt.space.sample_uniform(space, n + 20, rng)))[:n]
    y = np.array([scenarios.objective("C4", cfg) for cfg in cfgs])
    S = bt.surrogate
    z, _, _ = S._standardize(np.log(y))
    sc = scorer()
    lay = sc.set_space(space)
    rows = sc.to_device(lay.encode(cfgs))
    sq = sc.pairwise_sq(rows, rows)
    zd = torch.as_tensor(z, device="cuda")
    prm = torch.as_tensor(np.exp(rng.uniform(-1, 1, size=(c, 2 + space.dimension))), device="cuda")
    prior = S.LengthscalePrior()
    for _ in range(2):
        sc.lml_core(sq, zd, prm, True, prior)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        v, g, ok = sc.lml_core(sq, zd, prm, True, prior)
        v.cpu()
    print(f"n {n} c {c}: {(time.perf_counter() - t) / reps * 1e3:.3f} ms per call (wall, incl. the D2H sync)")


if __name__ == "__main__":
    main(*(int(a) for a in sys.argv[1:]))
