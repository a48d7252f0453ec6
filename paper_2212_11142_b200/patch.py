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

TARGETS = (
    ("engine", "optimize_acquisition", gpu.optimize_acquisition),
    ("acquisition", "_scores", gpu.scores),
    ("acquisition", "neighbors", gpu.neighbors),
    ("surrogate", "_batched_coarse_lml", gpu.batched_coarse_lml),
    ("surrogate", "_lml_core", gpu.lml_core),
)
METHODS = (
    ("surrogate", "GPModel", "predict_batch", gpu.predict_batch),
    ("feasibility", "FeasibilityModel", "predict_proba_batch", gpu.predict_proba_batch),
)


def install(boxtune, whole_path: bool = True):
    """Replace the reference's hot-path functions; returns a callable that undoes it.
    With whole_path=False the engine keeps the reference optimize_acquisition (which then calls
    the GPU _scores / neighbors): the per-call parity mode."""
    saved = []
    for mod_name, attr, fn in TARGETS:
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
