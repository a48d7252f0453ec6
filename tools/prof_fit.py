import cProfile, pstats, sys, numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
from golden_io import ref
from paper_2212_11142_b200 import hyperfit, scenarios
from paper_2212_11142_b200.patch import install
bt = ref(); space = scenarios.build_space("C4", bt.space)
install(bt, whole_path=False, lml=True, fit=False, rf=False)
rng = np.random.default_rng(200)
cfgs = list(dict.fromkeys(bt.space.sample_uniform(space, 220, rng)))[:200]
y = np.array([scenarios.objective("C4", c) for c in cfgs])
hyperfit.gp_fit(space, cfgs, y, np.random.default_rng(1))
cProfile.run("for _ in range(3): hyperfit.gp_fit(space, cfgs, y, np.random.default_rng(1))", "/tmp/fit.prof")
pstats.Stats("/tmp/fit.prof").sort_stats("tottime").print_stats(18)
