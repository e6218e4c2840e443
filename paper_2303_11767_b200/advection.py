"""Linear advection on the doubly periodic plane: the reference's
``advection_model`` and ``advection_sine`` case (models.py:114-140,
cases.py:99-110), on the GPU through ``dgswe_adv_stage``
(csrc/dgswe_adv.cuh, include/dgswe_b200.h).

A one-variable scalar model next to the shallow-water hot path: the
operator keeps the reference's API (``project_state``, ``zero_state``,
``state_from_coeffs``, ``assemble_rhs``, ``max_physical_speed``) so
``rk_step`` / ``integrate`` drive it through their generic path (Butcher
form with the reference's two-rounding axpy on device tensors).  States
hold the modal coefficients of u, device layout [nz][ny][nphi][nx].
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib, tracing
from .geometry import Mesh, build_vander, gauss_legendre, project_initial, row_mass_matrices


class AdvectionModel:
    """F = beta_x u, G = beta_y u (models.py:114-140)."""

    n_vars = 1
    var_names = ("u",)
    has_source = False
    is_spherical = False

    def __init__(self, beta):
        self.beta = tuple(float(b) for b in beta)
        if len(self.beta) != 2 or not all(np.isfinite(self.beta)):
            raise ValueError("advection velocity must be two finite numbers")

    def wavespeed_nodes(self, U, coords, direction):
        return np.full(np.shape(U["u"]), abs(self.beta[direction]))

    def max_physical_speed(self, U=None, coords=None) -> float:
        return max(abs(self.beta[0]), abs(self.beta[1]))


def advection_model(beta) -> AdvectionModel:
    """Linear constant-coefficient advection, F = beta1 u, G = beta2 u (models.py:137-140)."""
    return AdvectionModel(beta)


class AdvState:
    """Modal coefficients of u on the device, [nz][ny][nphi][nx]."""

    names = ("u",)

    def __init__(self, data: torch.Tensor, nx: int, ny: int, nz: int, nphi: int):
        if data.dtype != torch.float64 or not data.is_cuda or tuple(data.shape) != (nz, ny, nphi, nx):
            raise ValueError(f"state must be a CUDA float64 tensor of shape {(nz, ny, nphi, nx)}")
        self.data = data
        self.nx, self.ny, self.nz, self.nphi = nx, ny, nz, nphi

    def interior_coeffs(self, name: str = "u") -> np.ndarray:
        """(nx, ny, nz, nphi) host copy, the reference's interior layout."""
        if name != "u":
            raise KeyError(name)
        return np.ascontiguousarray(self.data.detach().cpu().numpy().transpose(3, 1, 0, 2))

    def to_numpy(self) -> np.ndarray:
        """(1, nx, ny, nz, nphi): the reference's stacked interior layout."""
        return self.interior_coeffs("u")[None]

    def copy(self) -> "AdvState":
        return AdvState(self.data.clone(), self.nx, self.ny, self.nz, self.nphi)

    def max_abs(self) -> float:
        return float(self.data.abs().max().item())


class AdvectionOperator:
    """DG operator of linear advection on a periodic planar mesh
    (the reference's SpatialOperator with an advection model, dg.py:166-543)."""

    def __init__(self, mesh: Mesh, p: int, model: AdvectionModel, rusanov=None, nz: int = 1, device=None):
        """``rusanov``: RusanovParams (dg.py:47-57); "local" and "global" coincide
        for constant beta (alpha = |beta_d| on every face), a pinned global
        alpha replaces it in both directions."""
        from .operator import RusanovParams
        if mesh.kind != "planar" or not isinstance(model, AdvectionModel):
            raise ValueError("linear advection runs on the periodic planar mesh")
        self.rusanov = rusanov if rusanov is not None else RusanovParams()
        if not torch.cuda.is_available():
            raise RuntimeError("AdvectionOperator needs a CUDA device (no CPU fallback)")
        self.mesh, self.p, self.model, self.nz = mesh, int(p), model, int(nz)
        self.device = torch.device("cuda") if device is None else torch.device(device)
        if self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        self.quad = gauss_legendre(self.p + 1)
        self.vander = build_vander(self.p, self.quad)
        self.nphi = self.vander.nphi
        self.M_rows, self.Minv_rows = row_mass_matrices(self.p, mesh, self.quad)   # monitors (host path)
        self.lib = _lib.load()
        keep = [np.ascontiguousarray(a, dtype=np.float64) for a in (self.vander.leg, self.vander.dleg,
                                                                    self.quad.weights)]
        cfg = _lib.AdvCfg(nx=mesh.nx, ny=mesh.ny, nz=self.nz, p=self.p, dx=mesh.dx, dy=mesh.dy,
                          beta_x=model.beta[0], beta_y=model.beta[1])
        handle = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _lib.check(self.lib.dgswe_adv_create(ctypes.byref(cfg), *[k.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
                                                                      for k in keep], ctypes.byref(handle)),
                       "dgswe_adv_create")
        self._h = handle
        self._ws = None
        if self.rusanov.mode == "global" and self.rusanov.alpha is not None:
            _lib.check(self.lib.dgswe_adv_set_alpha(self._h, float(self.rusanov.alpha)), "dgswe_adv_set_alpha")

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                self.lib.dgswe_adv_destroy(h)
            except Exception:
                pass
            self._h = None

    @property
    def state_shape(self):
        return (self.nz, self.mesh.ny, self.nphi, self.mesh.nx)

    def zero_state(self) -> AdvState:
        return AdvState(torch.zeros(self.state_shape, dtype=torch.float64, device=self.device),
                        self.mesh.nx, self.mesh.ny, self.nz, self.nphi)

    def state_from_coeffs(self, coeffs: dict) -> AdvState:
        """{"u": (nx, ny, nphi) or (nx, ny, nz, nphi)} modal coefficients."""
        a = np.asarray(coeffs["u"], dtype=np.float64)
        if a.ndim == 3:
            a = np.broadcast_to(a[:, :, None, :], (self.mesh.nx, self.mesh.ny, self.nz, self.nphi))
        d = torch.from_numpy(np.ascontiguousarray(a.transpose(2, 1, 3, 0))).to(self.device)
        return AdvState(d, self.mesh.nx, self.mesh.ny, self.nz, self.nphi)

    def project_state(self, ic_funcs: dict) -> AdvState:
        """L2 projection of the initial condition (basis.py:206-233, planar)."""
        return self.state_from_coeffs({"u": project_initial(ic_funcs["u"], self.mesh, self.vander)})

    def stage(self, a: float, U: AdvState | None, b: float, X: AdvState, g: float, Y: AdvState):
        """Y = a U + b X + g RHS(X) in one launch (U may alias Y, X may not)."""
        for s in (U, X, Y):
            if s is not None and (tuple(s.data.shape) != self.state_shape or s.data.device != self.device
                                  or not s.data.is_contiguous()):
                raise ValueError(f"states must be contiguous {self.state_shape} float64 tensors on {self.device}")
        with torch.cuda.device(self.device):
            _lib.check(self.lib.dgswe_adv_stage(self._h, float(a), ctypes.c_void_p(U.data.data_ptr() if U else 0),
                                                float(b), ctypes.c_void_p(X.data.data_ptr()), float(g),
                                                ctypes.c_void_p(Y.data.data_ptr()),
                                                ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)),
                       "dgswe_adv_stage")
        if tracing.get_op_recorder() is not None:
            rgn = tracing.LaunchRegion((self.mesh.nx, self.mesh.ny, self.nz), self.p, nvars=1)
            tracing.record("stage", "dgswe_adv_stage", rgn, 24.0 if (U is not None and a != 0.0) else 16.0,
                           tracing.adv_stage_flops_per_dof(self.p))

    def assemble_rhs(self, state: AdvState, out: AdvState | None = None) -> AdvState:
        """M^-1 (volume - boundary) of the advection operator (dg.py:504-523)."""
        if out is None:
            out = self.zero_state()
        self.stage(0.0, None, 0.0, state, 1.0, out)
        return out

    def rk_steps(self, state: AdvState, dt: float, nsteps: int, order: int = 3):
        """nsteps fused steps in place: forward Euler, Heun / SSPRK3 in
        Shu-Osher form, one launch per stage (Y = a U + b X + g RHS(X); the
        last stage writes u^{n+1} over u^n element by element)."""
        if order not in (1, 2, 3):
            raise ValueError("fused advection steps support orders 1..3 (use rk_step for tableau(4))")
        if self._ws is None:
            self._ws = [self.zero_state(), self.zero_state()]
        b0, b1 = self._ws
        for _ in range(int(nsteps)):
            self.stage(0.0, None, 1.0, state, dt, b0)
            if order == 1:
                state.data.copy_(b0.data)
            elif order == 2:
                self.stage(0.5, state, 0.5, b0, 0.5 * dt, state)
            else:
                self.stage(0.75, state, 0.25, b0, 0.25 * dt, b1)
                self.stage(1.0 / 3.0, state, 2.0 / 3.0, b1, (2.0 / 3.0) * dt, state)
        return state

    def max_physical_speed(self, state=None) -> float:
        return self.model.max_physical_speed()
