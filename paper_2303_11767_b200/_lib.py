"""ctypes binding of the C ABI in include/dgswe_b200.h.

The shared library is built in-tree (``paper_2303_11767_b200/libdgswe_b200.so``,
see :mod:`.build`).  There is no fallback: if the library is missing or the
GPU is absent every device call raises.
"""

from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libdgswe_b200.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "dgswe_b200.h")

ABI_VERSION = 5            # DGSWE_ABI_VERSION
STRIP = 32                 # DGSWE_STRIP: longitude elements per strip block
STATUS_POSITIVITY = 0x1
STATUS_NONFINITE = 0x2
STATUS_MEAN_NONPOS = 0x4
STATUS_PEER_TIMEOUT = 0x8
STATUS_BITS = 4

ALPHA_LOCAL, ALPHA_GLOBAL_PINNED, ALPHA_GLOBAL = 0, 1, 2

_D = ctypes.c_double
_PD = ctypes.POINTER(ctypes.c_double)
_VP = ctypes.c_void_p
_I = ctypes.c_int


class Cfg(ctypes.Structure):
    _fields_ = [
        ("nx", _I), ("ny", _I), ("nz", _I), ("p", _I),
        ("row0", _I), ("nrows", _I), ("jlo", _I), ("jhi", _I),
        ("radius", _D), ("gravity", _D), ("h_floor", _D), ("dx", _D), ("dy", _D),
        ("alpha_mode", _I), ("alpha", _D), ("row_chunk", _I), ("periodic_y", _I),
    ]


class AdvCfg(ctypes.Structure):
    _fields_ = [("nx", _I), ("ny", _I), ("nz", _I), ("p", _I), ("dx", _D), ("dy", _D),
                ("beta_x", _D), ("beta_y", _D)]


class Tables(ctypes.Structure):
    _fields_ = [(name, _PD) for name in (
        "leg", "dleg", "weights", "cos_r_int", "sin_r_int", "fcos_int",
        "cos_r_edge", "cos_edge", "minv", "orog")]


# name -> (restype, argtypes); the single source for the symbol-export test
SIGNATURES = {
    "dgswe_abi_version": (_I, []),
    "dgswe_last_error": (ctypes.c_char_p, []),
    "dgswe_create": (_I, [ctypes.POINTER(Cfg), ctypes.POINTER(Tables), ctypes.POINTER(_VP)]),
    "dgswe_destroy": (None, [_VP]),
    "dgswe_adv_create": (_I, [ctypes.POINTER(AdvCfg), _PD, _PD, _PD, ctypes.POINTER(_VP)]),
    "dgswe_adv_stage": (_I, [_VP, _D, _VP, _D, _VP, _D, _VP, _VP]),
    "dgswe_adv_set_alpha": (_I, [_VP, _D]),
    "dgswe_adv_destroy": (None, [_VP]),
    "dgswe_state_elems": (ctypes.c_int64, [_VP]),
    "dgswe_rhs": (_I, [_VP, _VP, _VP, _VP]),
    "dgswe_set_basis": (_I, [_VP, _I]),
    "dgswe_convert": (_I, [_VP, _VP, _I, _I, _I, _VP]),
    "dgswe_stage": (_I, [_VP, _D, _VP, _D, _VP, _D, _VP, _I, _VP]),
    "dgswe_stage_rows": (_I, [_VP, _D, _VP, _D, _VP, _D, _VP, _I, _I, _I, _VP]),
    "dgswe_stage_rows2": (_I, [_VP, _D, _VP, _D, _VP, _D, _VP, _I, _I, _I, _I, _I, _VP]),
    "dgswe_stage_rows_checked": (_I, [_VP, _D, _VP, _D, _VP, _D, _VP, _I, _I, _I, _I, _I, _VP]),
    "dgswe_set_exchange": (_I, [_VP, ctypes.c_longlong, _VP, ctypes.c_longlong, _VP, _VP, _VP]),
    "dgswe_stage_band": (_I, [_VP, _D, _VP, _D, _VP, _D, _VP, _I, _VP, _VP, _VP]),
    "dgswe_dev_alloc": (_I, [ctypes.c_size_t, ctypes.POINTER(ctypes.c_void_p)]),
    "dgswe_dev_free": (_I, [_VP]),
    "dgswe_ipc_handle": (_I, [_VP, ctypes.c_char_p]),
    "dgswe_ipc_open": (_I, [ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)]),
    "dgswe_ipc_close": (_I, [_VP]),
    "dgswe_axpy": (_I, [_VP, _D, _VP, _VP, _I, _I, _VP]),
    "dgswe_ssprk3": (_I, [_VP, _VP, _VP, _VP, _D, _I, _I, _VP]),
    "dgswe_rk_steps": (_I, [_VP, _I, _VP, _VP, _VP, _VP, _D, _I, _I, _VP]),
    "dgswe_mass": (_I, [_VP, _VP, _I, _I, _PD, _PD, _VP]),
    "dgswe_l2_sums": (_I, [_VP, _VP, _I, _I, _PD, _I, _PD, _VP, _PD, _VP]),
    "dgswe_project": (_I, [_VP, _VP, _PD, _D, _VP, _VP]),
    "dgswe_stage2": (_I, [_VP, _D, _VP, _D, _VP, _D, _VP, _VP, _D, _VP, _I, _I, _I, _VP]),
    "dgswe_alpha_prepass": (_I, [_VP, _VP, _VP]),
    "dgswe_alpha_buffer": (_VP, [_VP]),
    "dgswe_set_external_alpha": (_I, [_VP, _I]),
    "dgswe_status": (_I, [_VP, ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(ctypes.c_int32),
                          _I, _VP]),
    "dgswe_status_tags": (_I, [_VP, ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(ctypes.c_int32),
                               _I, _VP]),
    "dgswe_set_peer_timeout": (_I, [_VP, ctypes.c_ulonglong]),
    "dgswe_launch_count": (ctypes.c_int64, [_VP]),
}

_lib = None


class DGSWEError(RuntimeError):
    """A C-ABI call failed (message from dgswe_last_error)."""


def load():
    """Load (once) the in-tree library; raises if it was not built."""
    global _lib
    if _lib is None:
        path = os.environ.get("DGSWE_LIB", LIB_PATH)   # experiment builds (same ABI)
        if not os.path.exists(path):
            raise DGSWEError(
                f"{path} not found: build the CUDA library first "
                "(python -c 'import __graft_entry__ as g; g.build()')")
        lib = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.dgswe_abi_version() != ABI_VERSION:
            raise DGSWEError("libdgswe_b200.so ABI version mismatch")
        _lib = lib
    return _lib


def check(rc: int, what: str):
    if rc != 0:
        msg = load().dgswe_last_error()
        raise DGSWEError(f"{what} failed ({rc}): {msg.decode() if msg else ''}")
