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
    # declarations of diagnostic builds only (not exported by the production library)
    src = re.sub(r"#ifdef HYDRO_COUNT_ROT.*?#endif", "", src, flags=re.S)
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


def _desc(dim, k, q, n_elem, n_nodes):
    from paper_2104_11404_b200 import hydro
    return hydro._MeshDesc(dim, k, q, n_elem, n_nodes, None, None, None)


def test_empty_and_oversized_meshes_rejected():
    """Edge cases of the boundary (no GPU needed): an empty mesh and a mesh whose
    element->node slot count overflows the int32 indexing are rejected up front
    (workspace size 0 = invalid description); valid sizes return a positive size."""
    import ctypes
    from paper_2104_11404_b200 import hydro
    L = hydro.lib()
    ws = lambda d: L.hydro_ctx_workspace_bytes(ctypes.byref(d))
    assert ws(_desc(3, 2, 4, 0, 10)) == 0                        # no elements
    assert ws(_desc(3, 2, 4, 10, 0)) == 0                        # no nodes
    assert ws(_desc(3, 2, 4, (1 << 31) // 27 + 1, 1000)) == 0    # n_elem * 27 >= 2^31
    assert ws(_desc(3, 2, 4, 262144, 129 ** 3)) > 0              # C2 size
    assert ws(_desc(3, 3, 6, 258048, 337 * 145 * 145)) > 0       # C3 size
    assert ws(_desc(2, 2, 5, 10, 100)) == 0                      # unsupported q for k = 2


def test_null_arguments_rejected_without_gpu():
    """Argument errors return synchronously, before any device work."""
    from paper_2104_11404_b200 import hydro
    L = hydro.lib()
    assert L.hydro_force_full(None, None, None, None, None, None, hydro.Visc(0.5, 2.0, 1).c(),
                              hydro.Cfl(0.5, 2.5).c(), None, None, None, None) == hydro.HYDRO_ERR_ARG
    assert L.hydro_sample_create(None, None, 0, 1, None) == hydro.HYDRO_ERR_ARG
    assert L.hydro_rom_lift(10, 0, 4, None, None, 0, None, None, None) == hydro.HYDRO_ERR_ARG
    assert L.hydro_selftest_ieee_fast(1, -1, 0, 0, None, None) == hydro.HYDRO_ERR_ARG


def test_time_loop_and_offline_arguments_rejected_without_gpu():
    """The time loops, the offline routines and the stage-state export validate their
    arguments before any device work: NULL objects, non-positive steps, reversed time
    intervals, out-of-range controller constants, empty bases."""
    import ctypes
    from paper_2104_11404_b200 import hydro
    L = hydro.lib()
    ERR = hydro.HYDRO_ERR_ARG
    visc, cfl, ctrl = hydro.Visc().c(), hydro.Cfl().c(), hydro.DtCtrl().c()
    dt = ctypes.c_double(1e-3)
    assert L.hydro_fom_advance(None, None, None, None, None, visc, cfl, ctrl, 0.0, 1.0,
                               ctypes.byref(dt), 10, 1e-12, 100, None, None, None, None) == ERR
    bad = hydro.DtCtrl(beta1=1.5).c()   # beta1 must lie in (0, 1)
    assert L.hydro_fom_advance(None, None, None, None, None, visc, cfl, bad, 0.0, 1.0,
                               ctypes.byref(dt), 10, 1e-12, 100, None, None, None, None) == ERR
    h = (ctypes.c_double * 2)(1e-3, 1e-3)
    assert L.hydro_rom_advance(None, None, None, None, None, visc, cfl, ctrl, 1.0, 0.0, h, 10,
                               None, None, None, None, None) == ERR
    k = ctypes.c_int(0)
    assert L.hydro_pod(None, 4, 100, 0.9999, 4, None, None, ctypes.byref(k), None) == ERR
    assert L.hydro_pod(None, 4, 100, 1.5, 4, None, None, ctypes.byref(k), None) == ERR
    idx = (ctypes.c_int64 * 4)()
    assert L.hydro_deim(None, 100, 4, idx, None) == ERR
    assert L.hydro_qdeim(None, 100, 4, idx, None) == ERR
    assert L.hydro_deim_oversampled(None, 100, 4, 8, idx, None) == ERR
    assert L.hydro_mass_e_apply(None, None, None, None) == ERR
    z = (ctypes.c_int64 * 2)(0, 1)
    eta = (ctypes.c_double * 2)()
    assert L.hydro_rom_indicator(None, None, None, None, None, visc, cfl, 2, None, 2, None, 2, None, 2, z,
                                 2, None, 2, z, eta, None) == ERR
    assert L.hydro_window_ops(None, 0, 100, 4, 4, 1, None, None, None, None, None, None, None) == ERR
    vp8 = ctypes.c_void_p(8)
    assert L.hydro_window_ops(None, 3, 100, 4, 4, 1, vp8, vp8, vp8, vp8, vp8, vp8, None) == ERR  # field
    assert L.hydro_deim_oversampled(ctypes.c_void_p(8), 100, 4, 3, idx, None) == ERR   # n_s < m
    assert L.hydro_fom_stage_state(None, None, None, None, None) == ERR
