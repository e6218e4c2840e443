"""Conservation and accuracy monitors used as parity gates.

``mass_integral`` and ``l2_error`` keep the reference's signatures
(/root/reference/pkg/src/dgswe/diagnostics.py:42-107).  On a device state
of this package's SpatialOperator they run on the GPU (dgswe_mass /
dgswe_l2_sums: per-element contributions, then a fixed-order double-double
reduction -- deterministic, no host copy of the state).  The ``*_host``
variants keep the reference's exact reduction order (a sequential sum in
ascending element order) on a host copy, for bitwise comparisons.
"""

from __future__ import annotations

import ctypes
import math

import numpy as np
import torch

from . import _lib
from .geometry import build_vander, element_node_coords, gauss_legendre


def _ordered_sum(cell: np.ndarray) -> float:
    total = 0.0
    for v in cell.reshape(-1):    # (nx, ny) C order == i-major, j-minor
        total += v
    return total


def _device_ctx(state, op):
    ctx = getattr(op, "_ctx", None)
    data = getattr(state, "data", None)
    if ctx is None or not isinstance(data, torch.Tensor) or not data.is_cuda:
        return None
    return ctx


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def mass_integral_host(state, op, var: str | None = None, level: int = 0) -> float:
    """Sum over elements of (M_j c)_0 in the reference's order (diagnostics.py:92-107)."""
    var = var or state.names[0]
    coeffs = state.interior_coeffs(var)[:, :, level, :]
    cell = np.einsum("ym,xym->xy", op.M_rows[:, 0, :], coeffs)
    return _ordered_sum(cell)


def mass_integral(state, op, var: str | None = None, level: int = 0) -> float:
    """Sum over elements of (M_j c)_0, the cos-weighted integral of var."""
    ctx = _device_ctx(state, op)
    if ctx is None:
        return mass_integral_host(state, op, var, level)
    var = var or state.names[0]
    m0 = np.ascontiguousarray(op.M_rows[:, 0, :], dtype=np.float64)
    out = ctypes.c_double(0.0)
    _lib.check(ctx.lib.dgswe_mass(ctx.h, ctypes.c_void_p(state.data.data_ptr()), state.names.index(var),
                                  int(level), _dptr(m0), ctypes.byref(out), ctx.stream()), "dgswe_mass")
    return out.value


def _error_rule(op):
    quad = gauss_legendre(op.p + 2)
    return quad, build_vander(op.p, quad)


def _weight_rows(mesh, quad, th) -> np.ndarray:
    """(ny, n*n) quadrature weights per element row: w_i w_j cos(theta_j)
    on the sphere, w_i w_j on the plane (diagnostics.py:66-75)."""
    n = quad.n_1d
    w2 = np.outer(quad.weights, quad.weights)
    metric = np.cos(th) if mesh.kind == "latlon" else np.ones_like(th)
    return np.ascontiguousarray((w2[None, :, :] * metric[:, None, :]).reshape(mesh.ny, n * n))


def l2_error_host(state, reference_fn, op, var: str | None = None, relative: bool = False,
                  level: int = 0) -> float:
    """L2 norm of (numerical - reference), p+2 Gauss rule, cos(theta) metric
    on the sphere, reference reduction order (diagnostics.py:42-80)."""
    mesh = op.mesh
    var = var or state.names[0]
    quad, vander = _error_rule(op)
    n = quad.n_1d
    coeffs = state.interior_coeffs(var)[:, :, level, :]
    vals = np.einsum("qm,xym->xyq", vander.phi, coeffs)
    lam, th = element_node_coords(mesh, quad.nodes)
    ref = np.broadcast_to(reference_fn(lam[:, None, :, None], th[None, :, None, :]),
                          (mesh.nx, mesh.ny, n, n)).reshape(mesh.nx, mesh.ny, n * n)
    w_rows = _weight_rows(mesh, quad, th)
    err = _ordered_sum(mesh.determ * np.einsum("xyq,yq->xy", (vals - ref) ** 2, w_rows))
    norm = _ordered_sum(mesh.determ * np.einsum("xyq,yq->xy", ref**2, w_rows))
    e = math.sqrt(max(err, 0.0))
    return e / math.sqrt(max(norm, 1e-300)) if relative else e


def reference_nodal(reference_fn, lam: np.ndarray, th: np.ndarray, device) -> torch.Tensor:
    """reference_fn at the tensor nodes of every element, as a device array
    [ny][nx][n*n] (q = qi*n + qj, qi along lambda): evaluated on the GPU when
    the function accepts torch tensors, else with numpy and uploaded."""
    nx, n = lam.shape
    ny = th.shape[0]
    L = torch.from_numpy(lam).to(device)[None, :, :, None]        # (1, nx, n, 1)
    T = torch.from_numpy(th).to(device)[:, None, None, :]         # (ny, 1, 1, n)
    try:
        vals = reference_fn(L, T)
        if not isinstance(vals, torch.Tensor):
            raise TypeError
        vals = torch.broadcast_to(vals.to(torch.float64), (ny, nx, n, n))
    except Exception:
        v = reference_fn(lam[None, :, :, None], th[:, None, None, :])
        vals = torch.from_numpy(np.array(np.broadcast_to(v, (ny, nx, n, n)), dtype=np.float64)).to(device)
    return vals.reshape(ny, nx, n * n).contiguous()


def l2_error(state, reference_fn, op, var: str | None = None, relative: bool = False,
             level: int = 0) -> float:
    """L2 norm of (numerical - reference) with a p+2 Gauss rule and the
    cos(theta) metric (diagnostics.py:42-80)."""
    ctx = _device_ctx(state, op)
    if ctx is None:
        return l2_error_host(state, reference_fn, op, var, relative, level)
    mesh = op.mesh
    var = var or state.names[0]
    quad, vander = _error_rule(op)
    n = quad.n_1d
    lam, th = element_node_coords(mesh, quad.nodes)
    ref = reference_nodal(reference_fn, lam, th, state.data.device)
    w_rows = _weight_rows(mesh, quad, th)
    phi2 = np.ascontiguousarray(vander.phi, dtype=np.float64)
    out = (ctypes.c_double * 2)()
    _lib.check(ctx.lib.dgswe_l2_sums(ctx.h, ctypes.c_void_p(state.data.data_ptr()), state.names.index(var),
                                     int(level), _dptr(phi2), int(n * n), _dptr(w_rows),
                                     ctypes.c_void_p(ref.data_ptr()),
                                     ctypes.cast(out, ctypes.POINTER(ctypes.c_double)), ctx.stream()),
               "dgswe_l2_sums")
    e = math.sqrt(max(mesh.determ * out[0], 0.0))
    return e / math.sqrt(max(mesh.determ * out[1], 1e-300)) if relative else e


def convergence_rate(eps1: float, h1: float, eps2: float, h2: float) -> float:
    if min(eps1, eps2, h1, h2) <= 0.0:
        raise ValueError("errors and mesh sizes must be positive")
    if h1 == h2:
        raise ValueError("mesh sizes must differ")
    return (math.log(eps1) - math.log(eps2)) / (math.log(h1) - math.log(h2))
