"""The C-ABI library loads on a CPU-only host and exports exactly the
functions include/dgswe_b200.h declares; argument validation needs no GPU."""

import ctypes
import os
import re

import pytest

from paper_2303_11767_b200 import _lib


def _declared():
    src = open(_lib.HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return set(re.findall(r"\b(dgswe_[a-z0-9_]+)\s*\(", src))


def test_library_built_in_tree():
    assert os.path.exists(_lib.LIB_PATH), "run __graft_entry__.build() first"
    assert os.path.dirname(_lib.LIB_PATH).endswith("paper_2303_11767_b200")


def test_exports_every_declared_symbol():
    lib = _lib.load()
    declared = _declared()
    assert declared, "header parse found no declarations"
    assert declared == set(_lib.SIGNATURES), declared ^ set(_lib.SIGNATURES)
    for name in declared:
        assert hasattr(lib, name), name


def test_abi_version_and_error_string():
    lib = _lib.load()
    assert lib.dgswe_abi_version() == _lib.ABI_VERSION == 5
    assert isinstance(lib.dgswe_last_error(), bytes)


def _tables():
    buf = (ctypes.c_double * 64)()
    p = ctypes.cast(buf, ctypes.POINTER(ctypes.c_double))
    return _lib.Tables(*([p] * 9)), buf


def test_create_validates_without_gpu():
    lib = _lib.load()
    tabs, keep = _tables()
    h = ctypes.c_void_p()
    bad = [
        dict(nx=0, ny=4, nz=1, p=2, nrows=4, jlo=0, jhi=4),
        dict(nx=4, ny=4, nz=1, p=9, nrows=4, jlo=0, jhi=4),
        dict(nx=4, ny=4, nz=1, p=2, nrows=4, jlo=2, jhi=2),
        dict(nx=4, ny=4, nz=1, p=2, nrows=4, jlo=0, jhi=5),
        dict(nx=4, ny=8, nz=1, p=2, nrows=4, jlo=0, jhi=4, row0=2),   # needs a southern halo
    ]
    for kw in bad:
        kw.setdefault("row0", 0)
        cfg = _lib.Cfg(radius=6.4e6, gravity=9.81, h_floor=1e-5, dx=0.1, dy=0.1, **kw)
        rc = lib.dgswe_create(ctypes.byref(cfg), ctypes.byref(tabs), ctypes.byref(h))
        assert rc in (-1, -4), (kw, rc)
        assert lib.dgswe_last_error()
    assert lib.dgswe_create(None, None, None) == -1
    assert lib.dgswe_rhs(None, None, None, None) == -1
    assert lib.dgswe_state_elems(None) == 0
    assert lib.dgswe_launch_count(None) == 0


def test_context_requires_gpu_loudly():
    """No CPU fallback: the device API refuses to run without CUDA."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2303_11767_b200 as P
    setup = P.build_case(P.default_config("williamson_tc6").override(nx=8, ny=4, p=1))
    with pytest.raises(RuntimeError):
        P.SpatialOperator(setup.mesh, 1, setup.model)
