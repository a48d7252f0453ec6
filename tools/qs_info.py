import sys; sys.path.insert(0,'.')
import bench
from paper_2212_11142_b200.device import Scorer
sc=Scorer(0)
for name in ("M200","C3"):
    meta, space, gp, feas, cot = bench.load_workload(name, scorer=sc)
    sc.set_gp(gp); sc.set_forest(feas)
    print(name, [(p.name, p.kind) for p in space.parameters], flush=True)
