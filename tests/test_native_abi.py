"""The C-ABI library loads without a GPU and exports exactly what include/bx_sm100.h declares,
with struct layouts that match the ctypes binding."""
import ctypes as C
import re
import subprocess
from pathlib import Path

import pytest

from paper_2212_11142_b200 import _native as N

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "bx_sm100.h"


def declared():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(bx_[a-z0-9_]+)\s*\(", text)))


def test_library_loads_and_exports_every_declared_symbol():
    lib = N.lib()
    names = declared()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), name
    assert set(N.EXPORTED) == set(names)
    assert lib.bx_abi_version() == 1


def test_struct_layouts_match_ctypes(tmp_path):
    src = tmp_path / "layout.c"
    src.write_text(f'''
#include <stdio.h>
#include <stddef.h>
#include "{HEADER}"
int main(void) {{
  printf("%zu %zu %zu\\n", sizeof(bx_param_desc), sizeof(bx_cand), sizeof(bx_score_summary));
  printf("%zu %zu %zu %zu\\n", offsetof(bx_param_desc, lo), offsetof(bx_param_desc, raw_mx),
         offsetof(bx_cand, row), offsetof(bx_score_summary, best_prob));
  return 0;
}}''')
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-o", str(exe), str(src)], check=True)
    a, b = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split("\n")[:2]
    sizes, offs = list(map(int, a.split())), list(map(int, b.split()))
    assert sizes == [C.sizeof(N.ParamDesc), C.sizeof(N.Cand), C.sizeof(N.ScoreSummary)]
    assert offs == [N.ParamDesc.lo.offset, N.ParamDesc.raw_mx.offset, N.Cand.row.offset,
                    N.ScoreSummary.best_prob.offset]


def test_create_without_device_fails_cleanly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    assert not N.lib().bx_create(0)
    assert N.lib().bx_last_error(None) == b"null handle"
    # every entry point rejects a null handle with BX_ERR_ARG instead of crashing
    assert N.lib().bx_set_evaluated(None, None, 0) == N.BX_ERR_ARG
    assert N.lib().bx_score(None, None, 1, 0, 0.0, 0.0, 1, 0, None, None, None, None) == N.BX_ERR_ARG


def test_package_refuses_cpu_execution():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2212_11142_b200.device import Scorer
    with pytest.raises(RuntimeError, match="CUDA"):
        Scorer()


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_unique_rows_is_dict_fromkeys_order(seed):
    """bx_unique_rows (host code) keeps the first occurrence of every row in draw order, as
    list(dict.fromkeys(raw)) does (acquisition.py:173) - pools full of repeats, ragged widths."""
    import numpy as np

    from paper_2212_11142_b200 import sampling
    rng = np.random.default_rng(seed)
    for _ in range(60):
        q, w = int(rng.integers(2, 4000)), int(rng.integers(1, 20))
        rows = rng.integers(0, int(rng.integers(2, 5)), size=(q, w)).astype(np.uint32)
        want = np.array(list(dict.fromkeys(map(tuple, rows))), dtype=np.uint32).reshape(-1, w)
        assert np.array_equal(sampling.unique_rows(rows), want)
    assert N.lib().bx_unique_rows(None, -1, 4, None) < 0
