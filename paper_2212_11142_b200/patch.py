"""Install the B200 path into a loaded reference package.

    import boxtune
    from paper_2212_11142_b200.patch import install
    undo = install(boxtune)          # every hot-path call site now runs on the GPU
    ...
    undo()                           # restore the reference functions

Patch targets are where the reference binds the names it calls.
"""
from __future__ import annotations

from . import acquisition as gpu
from . import forest_fit, hyperfit

TARGETS = (
    ("engine", "optimize_acquisition", gpu.optimize_acquisition),
    ("acquisition", "_scores", gpu.scores),
    ("acquisition", "neighbors", gpu.neighbors),
)
# hyperparameter-fit objectives: opt-in, because their values are FP64 but not bit-identical to
# LAPACK's, and they feed argsort / L-BFGS-B (surrogate.py:505-530), so the fitted hyperparameters
# - and with them the BO history - may drift from the reference's in the last bits
LML_TARGETS = (
    ("surrogate", "_batched_coarse_lml", gpu.batched_coarse_lml),
    ("surrogate", "_lml_core", gpu.lml_core),
)
# the feasibility forest's tree building on the GPU (forest_fit.py; bit-exact, so on by default);
# the engine binds rf_fit at import (engine.py:19)
RF_TARGETS = (
    ("engine", "rf_fit", forest_fit.rf_fit),
)
# the whole hyperparameter fit with its L-BFGS-B restarts batched on the GPU (hyperfit.py); the
# engine binds gp_fit at import (engine.py:21)
FIT_TARGETS = (
    ("engine", "gp_fit", hyperfit.gp_fit),
)
METHODS = (
    ("surrogate", "GPModel", "predict_batch", gpu.predict_batch),
    ("feasibility", "FeasibilityModel", "predict_proba_batch", gpu.predict_proba_batch),
)


def install(boxtune, whole_path: bool = True, lml: bool = False, fit: bool = False, rf: bool = True):
    """Replace the reference's hot-path functions; returns a callable that undoes it.
    With whole_path=False the engine keeps the reference optimize_acquisition (which then calls
    the GPU _scores / neighbors): the per-call parity mode.  lml=True also moves the
    hyperparameter-fit objectives (_batched_coarse_lml, _lml_core) to the GPU; fit=True replaces
    the engine's gp_fit with the batched-restart one (hyperfit.gp_fit); rf=True (default) builds
    the feasibility forest on the GPU (forest_fit.rf_fit, bit-exact)."""
    saved = []
    targets = TARGETS + (LML_TARGETS if lml else ()) + (FIT_TARGETS if fit else ()) + (RF_TARGETS if rf else ())
    for mod_name, attr, fn in targets:
        if not whole_path and attr == "optimize_acquisition":
            continue
        mod = getattr(boxtune, mod_name)
        saved.append((mod, attr, getattr(mod, attr)))
        setattr(mod, attr, fn)
    for mod_name, cls_name, attr, fn in METHODS:
        cls = getattr(getattr(boxtune, mod_name), cls_name)
        saved.append((cls, attr, getattr(cls, attr)))
        setattr(cls, attr, fn)

    def uninstall():
        for owner, attr, old in reversed(saved):
            setattr(owner, attr, old)

    return uninstall
