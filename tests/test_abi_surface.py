"""CPU-side checks of the boundary: libdpm.so loads and exports every symbol include/dpm.h declares.
No compute calls (no GPU here)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "dpm.h")
LIB = os.path.join(ROOT, "paper_1811_03557_b200", "libdpm.so")


def declared_symbols():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(dpm_[a-z_0-9]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        import paper_1811_03557_b200.build as b
        b.build()
    return ctypes.CDLL(LIB)


def test_header_declares_the_north_star_calls():
    syms = declared_symbols()
    for s in ["dpm_create", "dpm_aux_solve_batch", "dpm_build_projection", "dpm_boundary_lsq", "dpm_pks_step"]:
        assert s in syms


def test_library_exports_every_declared_symbol(lib):
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_binding_covers_every_symbol(lib):
    from paper_1811_03557_b200 import _lib
    assert sorted(_lib.EXPORTED) == declared_symbols()


def test_sm100a_code_in_library():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    assert "DMMA.8x8x4" in sass     # fp64 tensor-core transforms


def test_create_rejects_invalid_without_gpu(lib):
    # argument validation happens before any CUDA call
    from paper_1811_03557_b200 import _lib as L
    h = ctypes.c_void_p()
    g = L.Grid(2, -1.0, 1.0)
    d = L.Domain(L.SPHERE, (ctypes.c_double * 3)(0, 0, 0), (ctypes.c_double * 3)(0.5, 0.5, 0.5))
    assert L.lib.dpm_create(ctypes.byref(g), ctypes.byref(d), 2, 1e-3, 0, 0, ctypes.byref(h)) == L.DPM_ERR_INVALID
    g = L.Grid(16, -1.0, 1.0)
    d = L.Domain(L.SPHERE, (ctypes.c_double * 3)(0, 0, 0), (ctypes.c_double * 3)(1.5, 1.5, 1.5))
    assert L.lib.dpm_create(ctypes.byref(g), ctypes.byref(d), 2, 1e-3, 0, 0, ctypes.byref(h)) == L.DPM_ERR_INVALID
    assert b"inside" in L.lib.dpm_last_error(None)
    d = L.Domain(L.SPHERE, (ctypes.c_double * 3)(0, 0, 0), (ctypes.c_double * 3)(0.5, 0.5, 0.5))
    assert L.lib.dpm_create(ctypes.byref(g), ctypes.byref(d), 2, -1.0, 0, 0, ctypes.byref(h)) == L.DPM_ERR_INVALID


def test_dd_creators_reject_invalid_without_gpu(lib):
    # dpm_create_octant / dpm_create_dd1 validate before any CUDA call (NEXT-3: 0 < r1 < r2, sub in {0, 1},
    # the subdomain strictly inside its box; octant index 0..7)
    from paper_1811_03557_b200 import _lib as L
    h = ctypes.c_void_p()
    g = L.Grid(20, -0.328125, 0.328125)      # the paper's N1 = 20 mesh for r1 = 0.25
    bad = [(2, 0.25, 0.5), (0, 0.5, 0.25), (0, 0.0, 0.5), (0, 0.4, 0.5)]   # bad sub, r2 <= r1, r1 = 0, ball > box
    for sub, r1, r2 in bad:
        st = L.lib.dpm_create_dd1(ctypes.byref(g), sub, r1, r2, 0, 0, 1e-8, 0, ctypes.byref(h))
        assert st == L.DPM_ERR_INVALID, (sub, r1, r2)
    assert L.lib.dpm_create_dd1(ctypes.byref(g), 0, 0.25, 0.5, -1, 0, 1e-8, 0, ctypes.byref(h)) == L.DPM_ERR_INVALID
    go = L.Grid(16, -0.1, 1.1)
    assert L.lib.dpm_create_octant(ctypes.byref(go), 8, 1.0, 4, 4, 1e-3, 0, ctypes.byref(h)) == L.DPM_ERR_INVALID
    assert L.lib.dpm_create_octant(ctypes.byref(go), 0, 2.0, 4, 4, 1e-3, 0, ctypes.byref(h)) == L.DPM_ERR_INVALID
    assert not h.value
