"""CPU oracle for the candidate-acquisition hot path — TEST INFRASTRUCTURE ONLY.

A NumPy/pure-Python restatement of the reference algorithms (boxtune, arXiv 2212.11142 desk
re-implementation; file:line citations refer to /root/reference/pkg/src/boxtune/).  Only `tests/`,
`__graft_entry__.smoke()` and bench.py's cpu_baseline / `--impl reference` leg may import it, and
only as the checker or the timed CPU baseline.  The product path (`paper_2212_11142_b200`) never
imports it.

Parity pinning: the oracle is checked against golden vectors produced by running the reference
itself in the build container (tests/golden/make_golden.py -> tests/golden/*.json|npz; tests in
tests/test_oracle_golden.py).  The reference's floating-point arithmetic lives in third-party
numpy 2.3 / scipy 1.18 (OpenBLAS potrf/trtrs/gemv, cephes ndtr); the oracle uses the same
libraries, so GP/EI values agree to rounding, and integer paths (neighbours, chain of trees,
constraints, forest leaves) agree exactly.
"""
from .gp import OracleGP, expected_improvement, pairwise_sq, predict, scores  # noqa: F401
from .forest import OracleForest, features, predict_proba  # noqa: F401
from .moves import cot_contains, eval_constraint, neighbors  # noqa: F401
from .lml import coarse_lml, lml_core, prior_term  # noqa: F401
from .search import optimize  # noqa: F401
