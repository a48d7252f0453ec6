"""B200-native candidate-acquisition scoring for BaCO (arXiv 2212.11142), behind the reference
("boxtune") Python API.  See DESIGN.md and INTEGRATION.md."""
from .acquisition import (  # noqa: F401
    MAX_CLIMB_STEPS, N_CANDIDATES, N_STARTS, SpaceExhausted, acquisition_value, batched_coarse_lml,
    constraints_batch, contains_batch, neighbors, optimize_acquisition, predict_batch,
    predict_proba_batch, scores)
from .device import Scorer, scorer  # noqa: F401
from .layout import SpaceLayout  # noqa: F401

__version__ = "0.1.0"
