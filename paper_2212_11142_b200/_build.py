"""Build libbx_sm100.so (all CUDA sources, sm_100a) in-tree with nvcc.

The shared library lands next to this file so that it travels with the repo snapshot to the GPU
box; it is git-ignored.  Rebuilds only when a source or header is newer than the library.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
INCLUDE = PKG.parent / "include"
LIB = PKG / "libbx_sm100.so"
SOURCES = ["host_rng.cu", "host_rows.cu", "bx_api.cu", "bx_model.cu", "bx_score.cu", "bx_lml.cu", "score.cu", "score_summary.cu", "gp_fused.cu", "gp_tc.cu", "forest.cu", "feasible.cu",
           "gp_linalg.cu", "probe.cu", "merge.cu", "generate.cu", "lml_wide.cu", "forest_fit.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
         "--expt-relaxed-constexpr"]


def nvcc() -> str:
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not Path(cand).exists():
        raise RuntimeError("nvcc not found: cannot build the sm_100a library")
    return cand


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES] + list(CSRC.glob("*.cuh")) + list(INCLUDE.glob("*.h"))
    return any(p.stat().st_mtime > t for p in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not _stale():
        return LIB
    tmp = LIB.with_suffix(".so.tmp")
    objs, cmds = [], []
    for src in SOURCES:
        obj = PKG / "csrc" / (Path(src).stem + ".o")
        cmds.append([nvcc(), *ARCH, *FLAGS, "-I", str(INCLUDE), "-c", str(CSRC / src), "-o", str(obj)])
        objs.append(str(obj))
    # one nvcc per translation unit, in parallel (gp_tc.cu and forest.cu dominate)
    from concurrent.futures import ThreadPoolExecutor

    def run(cmd):
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)

    with ThreadPoolExecutor(max_workers=max(1, min(len(cmds), os.cpu_count() or 1))) as pool:
        list(pool.map(run, cmds))
    cmd = [nvcc(), *ARCH, "-shared", "-o", str(tmp), *objs, "-cudart", "static"]
    subprocess.run(cmd, check=True)
    os.replace(tmp, LIB)
    for o in objs:
        Path(o).unlink(missing_ok=True)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
