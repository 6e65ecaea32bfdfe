"""C-ABI library checks that need no GPU (-m "not gpu"): the library loads, exports
every entry point include/hydro.h declares, and its own (binary128) basis tables
agree bit for bit with the oracle's independent (mpmath) tables."""
from __future__ import annotations

import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "hydro.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hydro_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2104_11404_b200 import hydro
    L = hydro.lib()
    names = _declared()
    assert len(names) >= 18
    for n in names:
        assert hasattr(L, n), n
    assert set(names) == set(hydro.EXPORTED)
    assert b"sm_100a" in L.hydro_version()


def test_library_is_sm100a_cubin():
    import subprocess
    from paper_2104_11404_b200 import hydro
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", hydro.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("k,q", [(2, 4), (3, 6)])
def test_tables_bitwise_equal_to_oracle(oracle_lib, k, q):
    from paper_2104_11404_b200 import hydro
    mine = hydro.basis_tables(k, q)
    ref = oracle_lib.tables(k, q)
    for key in ("xi", "w", "B", "G", "Bl"):
        assert np.array_equal(np.asarray(mine[key]), np.asarray(ref[key])), key


def test_unsupported_combination_rejected():
    from paper_2104_11404_b200 import hydro
    import ctypes
    d = hydro._MeshDesc(3, 4, 8, 1, 1, None, None, None)
    assert hydro.lib().hydro_ctx_workspace_bytes(ctypes.byref(d)) == 0
