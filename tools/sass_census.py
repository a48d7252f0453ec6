"""SASS opcode census of the hot kernels in libbx_sm100.so (cuobjdump -sass): the instructions
that prove the Blackwell paths - UTCIMMA (tcgen05.mma kind::i8), LDTM / STTM (tcgen05.ld / st,
TMEM), UBLKCP (cp.async.bulk), SYNCS (mbarrier), DMMA (FP64 tensor MMA), DFMA / DMUL / DADD (FP64
pipe), LDS (shared loads).

    python tools/sass_census.py [lib] > profiles/r02_sass_census.txt
"""
import collections
import re
import subprocess
import sys
from pathlib import Path

LIB = Path(sys.argv[1]) if len(sys.argv) > 1 else Path(__file__).resolve().parent.parent / "paper_2212_11142_b200" / "libbx_sm100.so"
KERNELS = ("gp_tc_kernel", "rf_qs_summary_kernel", "rf_qs_kernel", "merge_fast_kernel", "climb_update_kernel",
           "neighbors_kernel", "generate_kernel", "gp_fused_kernel", "lw_chol_kernel", "lw_grad_kernel")
OPS = ("UTCIMMA", "UTCBAR", "LDTM", "STTM", "UBLKCP", "SYNCS", "DMMA", "DFMA", "DMUL", "DADD", "LDS", "STS",
       "LDG", "STG", "MUFU", "I2F", "F2I", "POPC", "IDP")

out = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True, check=True).stdout
func, counts = None, collections.defaultdict(collections.Counter)
for line in out.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        func = m.group(1)
        continue
    m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(?:\.[A-Z0-9_.]+)?", line)
    if func and m:
        counts[func][m.group(1)] += 1
print(f"SASS census of {LIB.name} (static instruction counts per kernel instance)")
print(f"{'kernel':70s} " + " ".join(f"{o:>7s}" for o in OPS))
for f in sorted(counts):
    if not any(k in f for k in KERNELS):
        continue
    name = subprocess.run(["c++filt", f], capture_output=True, text=True).stdout.strip()
    name = re.sub(r"bx::\(anonymous namespace\)::", "", name)[:70]
    print(f"{name:70s} " + " ".join(f"{counts[f][o]:7d}" for o in OPS))
