"""Device-resident DG operator with the reference's solver API.

``SpatialOperator`` and ``State`` mirror /root/reference/pkg/src/dgswe/
dg.py:47-89 and 166-543 (constructor, attributes, ``zero_state``,
``state_from_coeffs``, ``project_state``, ``assemble_rhs``,
``max_physical_speed``); the right-hand side itself is one fused CUDA launch
through the C ABI (include/dgswe_b200.h, ``dgswe_rhs``).

Device layout of a state: one fp64 tensor ``data[z, j, v, s, m, l]``
(level, latitude row, variable, strip, mode, lane) with longitude element
i = 32 s + l -- a strip-blocked structure of arrays: a warp's 32 lanes read
32 consecutive elements of one mode, and one variable's row tile of a strip
is a single contiguous block (the unit of the kernel's TMA copies).  The
last strip is zero-padded past nx.  There is no halo ring: the periodic
longitude wrap is an index wrap inside the kernel (replaces
``_halo_exchange``, dg.py:330-346).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib, tracing
from .geometry import (Mesh, build_vander, gauss_legendre, node_latitudes, project_initial,
                       row_mass_matrices)
from .physics import PositivityError, SphereSWEModel

VAR_NAMES = ("h", "hu", "hv")


@dataclass(frozen=True)
class RusanovParams:
    """Per-interface local alpha (default) or one global alpha per
    direction, optionally pinned (dg.py:47-57)."""

    mode: str = "local"
    alpha: float | None = None

    def __post_init__(self):
        if self.mode not in ("local", "global"):
            raise ValueError(f"mode must be 'local' or 'global', got {self.mode!r}")


STRIP = _lib.STRIP


def nstrips(nx: int) -> int:
    return (nx + STRIP - 1) // STRIP


def device_shape(nz: int, nrows: int, nphi: int, nx: int) -> tuple:
    """Shape of a device state buffer: (nz, nrows, 3, nstrip, nphi, STRIP)."""
    return (nz, nrows, 3, nstrips(nx), nphi, STRIP)


def _to_device_layout(stack: np.ndarray) -> np.ndarray:
    """(3, nx, ny, nz, nphi) reference interior layout -> (nz, ny, 3, nstrip, nphi, STRIP)."""
    _, nx, ny, nz, nphi = stack.shape
    ns = nstrips(nx)
    pad = np.zeros((3, ns * STRIP, ny, nz, nphi), dtype=np.float64)
    pad[:, :nx] = stack
    pad = pad.reshape(3, ns, STRIP, ny, nz, nphi)
    return np.ascontiguousarray(np.transpose(pad, (4, 3, 0, 1, 5, 2)))


def lon_major(data: torch.Tensor, nx: int) -> torch.Tensor:
    """View-transform of a device state to (nz, nrows, 3, nphi, nx) (a copy)."""
    nz, nr, nv, ns, nphi, L = data.shape
    return data.permute(0, 1, 2, 4, 3, 5).reshape(nz, nr, nv, nphi, ns * L)[..., :nx]


def _to_reference_layout(data: torch.Tensor, nx: int) -> np.ndarray:
    """(nz, ny, 3, nstrip, nphi, STRIP) device tensor -> (3, nx, ny, nz, nphi) host."""
    return np.ascontiguousarray(lon_major(data, nx).detach().cpu().numpy().transpose(2, 4, 1, 0, 3))


class _VarView:
    """Host view object standing in for a reference ``Field`` (``.data`` is
    the halo-padded (nx+2, ny+2, nz, nphi) array, copied from the device)."""

    def __init__(self, state: "State", v: int):
        self._s, self._v = state, v

    @property
    def data(self) -> np.ndarray:
        s = self._s
        inner = s.interior_coeffs(s.names[self._v])
        out = np.zeros((s.nx + 2, s.ny + 2, s.nz, s.nphi))
        out[1:-1, 1:-1] = inner
        out[0, 1:-1] = inner[-1]
        out[-1, 1:-1] = inner[0]
        return out


class State:
    """Modal coefficients of (h, hu, hv) on the device.

    ``interior_coeffs(name)`` returns a host copy shaped like the
    reference's (nx, ny, nz, nphi) view; writes to it do not reach the
    device (use :meth:`set_interior_coeffs`).

    Between consecutive fused ``rk_step`` calls the buffer may hold the
    values at the Gauss nodes instead of the modal coefficients (the stage
    kernels' own basis): every read through ``data``
    (and so every method below, the diagnostics and the Butcher path)
    converts it back first, in place, with one elementwise kernel.  The
    raw buffer is ``_data``; ``_nodal`` is the operator whose nodal basis
    it currently holds (None: modal).
    """

    def __init__(self, data: torch.Tensor, nx: int, ny: int, nz: int, nphi: int):
        if data.dtype != torch.float64 or not data.is_cuda:
            raise TypeError("State data must be a CUDA float64 tensor")
        if tuple(data.shape) != device_shape(nz, ny, nphi, nx) or not data.is_contiguous():
            raise ValueError(f"State data must be contiguous {device_shape(nz, ny, nphi, nx)} "
                             f"(nz, ny, 3, nstrip, nphi, {STRIP}), got {tuple(data.shape)}")
        if data.data_ptr() % 16:
            raise ValueError("State data must be 16-byte aligned (the kernels move row tiles by TMA)")
        self._data = data
        self._nodal = None
        self.names = VAR_NAMES
        self.nx, self.ny, self.nz, self.nphi = nx, ny, nz, nphi

    @property
    def data(self) -> torch.Tensor:
        """The modal coefficients (converted back in place if the buffer holds nodal values)."""
        if self._nodal is not None:
            op, self._nodal = self._nodal, None
            op._ctx.convert(self._data, False, 0, self.ny)
        return self._data

    @data.setter
    def data(self, value: torch.Tensor):
        self._data = value
        self._nodal = None

    def _as_nodal(self, op) -> torch.Tensor:
        """The raw buffer holding ``op``'s nodal values (converted in place if modal)."""
        if self._nodal is not op:
            raw = self.data                      # modal (converting back from another operator's basis)
            op._ctx.convert(raw, True, 0, self.ny)
            self._nodal = op
        return self._data

    @property
    def fields(self) -> dict:
        return {n: _VarView(self, v) for v, n in enumerate(self.names)}

    @property
    def interior(self):
        return (self.nx, self.ny, self.nz)

    def interior_coeffs(self, name: str) -> np.ndarray:
        v = self.names.index(name)
        return np.ascontiguousarray(
            lon_major(self.data, self.nx)[:, :, v].detach().cpu().numpy().transpose(3, 1, 0, 2))

    def set_interior_coeffs(self, name: str, arr) -> None:
        v = self.names.index(name)
        a = np.broadcast_to(np.asarray(arr, dtype=np.float64), (self.nx, self.ny, self.nz, self.nphi))
        stack = np.zeros((3, self.nx, self.ny, self.nz, self.nphi))
        stack[0] = a
        dev = torch.from_numpy(_to_device_layout(stack)).to(self.data.device)
        self.data[:, :, v].copy_(dev[:, :, 0])

    def to_numpy(self) -> np.ndarray:
        """(3, nx, ny, nz, nphi) host copy in the reference's interior layout."""
        return _to_reference_layout(self.data, self.nx)

    def copy(self) -> "State":
        return State(self.data.clone(), self.nx, self.ny, self.nz, self.nphi)

    def max_abs(self) -> float:
        return float(self.data.abs().max().item())


class _Context:
    """Owns one dgswe_ctx (C ABI) for a band of latitude rows."""

    def __init__(self, mesh: Mesh, p: int, model: SphereSWEModel, rusanov: RusanovParams, nz: int,
                 quad, vander, Minv, row0=0, nrows=None, jlo=None, jhi=None, row_chunk=0, bottom=None):
        lib = _lib.load()
        ny = mesh.ny
        nrows = ny if nrows is None else nrows
        jlo = 0 if jlo is None else jlo
        jhi = nrows if jhi is None else jhi
        n = quad.nodes.shape[0]
        if mesh.kind == "planar":
            # the plane as the lat-lon operator with cos = 1, sin = 0, R = 1:
            # F, G and the mass unweighted, the source f (hv, -hu)
            # (models.py:176-227), rows wrapping instead of poles
            R = 1.0
            arrs = {
                "leg": vander.leg, "dleg": vander.dleg, "weights": quad.weights,
                "cos_r_int": np.ones((ny, n)), "sin_r_int": np.zeros((ny, n)),
                "fcos_int": np.full((ny, n), model.coriolis_f),
                "cos_r_edge": np.ones(ny + 1), "cos_edge": np.ones(ny + 1),
                "minv": Minv,
            }
        else:
            const = model.constants
            th = node_latitudes(mesh, quad.nodes)                 # (ny, n)
            R = const.radius
            arrs = {
                "leg": vander.leg, "dleg": vander.dleg, "weights": quad.weights,
                "cos_r_int": np.cos(th) / R, "sin_r_int": np.sin(th) / R,
                "fcos_int": 2.0 * const.omega * np.sin(th) * np.cos(th),
                "cos_r_edge": np.cos(mesh.y_edges) / R, "cos_edge": np.cos(mesh.y_edges),
                "minv": Minv,
            }
        if bottom is not None:
            arrs["orog"] = bottom                             # (ny, nx, n*n) b at the Gauss nodes
        keep = {k: np.ascontiguousarray(v, dtype=np.float64) for k, v in arrs.items()}
        tabs = _lib.Tables(**{k: v.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
                              for k, v in keep.items()})
        if rusanov.mode == "local":
            mode, alpha = _lib.ALPHA_LOCAL, 0.0
        elif rusanov.alpha is not None:
            mode, alpha = _lib.ALPHA_GLOBAL_PINNED, float(rusanov.alpha)
        else:
            mode, alpha = _lib.ALPHA_GLOBAL, 0.0
        cfg = _lib.Cfg(nx=mesh.nx, ny=ny, nz=nz, p=p, row0=row0, nrows=nrows, jlo=jlo, jhi=jhi,
                       radius=R, gravity=model.gravity, h_floor=model.h_floor,
                       dx=mesh.dx, dy=mesh.dy, alpha_mode=mode, alpha=alpha,
                       row_chunk=int(row_chunk), periodic_y=int(mesh.kind == "planar"))
        handle = ctypes.c_void_p()
        _lib.check(lib.dgswe_create(ctypes.byref(cfg), ctypes.byref(tabs), ctypes.byref(handle)),
                   "dgswe_create")
        self.lib, self.h = lib, handle
        self.row0, self.nrows, self.jlo, self.jhi = row0, nrows, jlo, jhi
        self.device = torch.cuda.current_device()

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value:
            try:
                self.lib.dgswe_destroy(h)
            except Exception:
                pass
            self.h = None

    @staticmethod
    def stream():
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)

    def status(self, reset=True):
        """(flags, smallest tag over the raised bits)."""
        flags, tags = self.status_tags(reset)
        return flags, min(tags)

    def status_tags(self, reset=True):
        """(flags, [smallest tag per status bit]) -- POSITIVITY, NONFINITE,
        MEAN_NONPOS, PEER_TIMEOUT (INT32_MAX where the bit is clear)."""
        flags = ctypes.c_uint32(0)
        tags = (ctypes.c_int32 * _lib.STATUS_BITS)()
        _lib.check(self.lib.dgswe_status_tags(self.h, ctypes.byref(flags), tags, int(reset),
                                              self.stream()), "dgswe_status_tags")
        return flags.value, list(tags)

    def launches(self) -> int:
        return int(self.lib.dgswe_launch_count(self.h))

    def set_basis(self, nodal: bool):
        """Basis of the states the stage entry points take (include/dgswe_b200.h)."""
        _lib.check(self.lib.dgswe_set_basis(self.h, int(bool(nodal))), "dgswe_set_basis")

    def convert(self, data: torch.Tensor, to_nodal: bool, r0: int, r1: int):
        """In-place modal <-> nodal change of basis of local rows [r0, r1)."""
        _lib.check(self.lib.dgswe_convert(self.h, ctypes.c_void_p(data.data_ptr()), int(bool(to_nodal)),
                                          int(r0), int(r1), self.stream()), "dgswe_convert")


def _ptr(t: torch.Tensor | None):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


class _NullTimer:
    def begin(self, phase):
        pass

    def end(self, phase):
        pass


class SpatialOperator:
    """Precomputed DG discretisation of the spherical SWE on one mesh, with
    the right-hand side evaluated by the fused sm_100a kernel.

    Quadrature: p+1 Gauss points per direction for interior and edges,
    weights and Jacobians folded into the device contraction constants.
    """

    def __init__(self, mesh: Mesh, p: int, model: SphereSWEModel, rusanov: RusanovParams | None = None,
                 nz: int = 1, timers=None, device=None, row_chunk: int = 0):
        if bool(getattr(model, "is_spherical", False)) != (mesh.kind == "latlon") or \
                mesh.kind not in ("latlon", "planar"):
            raise ValueError("model/mesh geometry mismatch (lat-lon sphere or periodic plane)")
        if not torch.cuda.is_available():
            raise RuntimeError("SpatialOperator needs a CUDA device (no CPU fallback)")
        self.mesh, self.p, self.model = mesh, int(p), model
        self.rusanov = rusanov or RusanovParams()
        self.nz = int(nz)
        self.timers = timers or _NullTimer()
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else \
            torch.device(device)
        self.quad = gauss_legendre(self.p + 1)
        self.vander = build_vander(self.p, self.quad)
        self.nphi, self.n1, self.nq = self.vander.nphi, self.vander.n_1d, self.vander.n_q
        self.halo_shape = (mesh.nx + 2, mesh.ny + 2, self.nz)
        self.M_rows, self.Minv_rows = row_mass_matrices(self.p, mesh, self.quad)
        self.M_planar = self.M_rows[0] if mesh.kind == "planar" else None
        self.bottom_nodal = self._bottom_at_nodes()
        with torch.cuda.device(self.device):
            self._ctx = _Context(mesh, self.p, model, self.rusanov, self.nz, self.quad, self.vander,
                                 self.Minv_rows, row_chunk=row_chunk, bottom=self.bottom_nodal)
        self._phi_dev = None
        self._scratch = {}
        self._replayed = 0          # kernel launches replayed from Python-captured CUDA graphs

    def _bottom_at_nodes(self):
        """(ny, nx, n*n) orography b at every element's Gauss nodes (q = qi n + qj,
        qi along lambda), or None without orography (the reference's model)."""
        b = getattr(self.model, "bottom", None)
        if b is None:
            return None
        from .geometry import element_node_coords
        lam, th = element_node_coords(self.mesh, self.quad.nodes)      # (nx, n), (ny, n)
        n = self.p + 1
        vals = np.asarray(b(lam[None, :, :, None], th[:, None, None, :]), dtype=np.float64)
        vals = np.broadcast_to(vals, (self.mesh.ny, self.mesh.nx, n, n))
        return np.ascontiguousarray(vals.reshape(self.mesh.ny, self.mesh.nx, n * n))

    # -- state construction -------------------------------------------------

    @property
    def state_shape(self):
        return device_shape(self.nz, self.mesh.ny, self.nphi, self.mesh.nx)

    def zero_state(self) -> State:
        d = torch.zeros(self.state_shape, dtype=torch.float64, device=self.device)
        return State(d, self.mesh.nx, self.mesh.ny, self.nz, self.nphi)

    def state_from_coeffs(self, coeffs: dict) -> State:
        """Per-variable (nx, ny, nphi) (or (nx, ny, nz, nphi)) arrays."""
        stack = np.zeros((3, self.mesh.nx, self.mesh.ny, self.nz, self.nphi))
        for name, arr in coeffs.items():
            a = np.asarray(arr, dtype=np.float64)
            stack[VAR_NAMES.index(name)] = a[:, :, None, :] if a.ndim == 3 else a
        return self.state_from_array(stack)

    def state_from_array(self, stack: np.ndarray) -> State:
        """(3, nx, ny, nz, nphi) host array in the reference's interior layout."""
        d = torch.from_numpy(_to_device_layout(np.asarray(stack, dtype=np.float64)))
        return State(d.to(self.device), self.mesh.nx, self.mesh.ny, self.nz, self.nphi)

    def state_from_reference(self, ref_state) -> State:
        """Adopt a reference ``dgswe.dg.State`` (interior coefficients)."""
        return self.state_from_array(np.stack([ref_state.interior_coeffs(n) for n in VAR_NAMES]))

    def project_state(self, ic_funcs: dict, device: bool = False) -> State:
        """cos-weighted L2 projection of the initial condition (basis.py:206-233).

        ``device=False`` (default): numpy on the host in the reference's
        operation order (bitwise equal to the reference).  ``device=True``:
        the functions are evaluated on the GPU (torch-capable callables, else
        numpy and upload) and projected by ``dgswe_project`` -- for grids
        where host setup is slow; equal to the host result to rounding."""
        if not device:
            return self.state_from_coeffs({name: project_initial(f, self.mesh, self.vander)
                                           for name, f in ic_funcs.items()})
        from .geometry import element_node_coords
        from .monitors import reference_nodal
        lam, th = element_node_coords(self.mesh, self.quad.nodes)
        zero = lambda lam_, th_: 0.0 * lam_ + 0.0 * th_     # noqa: E731
        f = torch.stack([reference_nodal(ic_funcs.get(name, zero), lam, th, self.device)
                         for name in VAR_NAMES])               # (3, ny, nx, n*n)
        out = self.zero_state()
        cosn = np.ascontiguousarray(np.ones_like(th) if self.mesh.kind == "planar" else np.cos(th),
                                    dtype=np.float64)
        c = self._ctx
        _lib.check(c.lib.dgswe_project(c.h, _ptr(f), cosn.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                       float(self.mesh.determ), _ptr(out.data), c.stream()),
                   "dgswe_project")
        return out

    # -- device entry points ------------------------------------------------

    def _check(self, state: State):
        if tuple(state.data.shape) != self.state_shape or (state.nx, state.ny, state.nz, state.nphi) != \
                (self.mesh.nx, self.mesh.ny, self.nz, self.nphi):
            raise ValueError(f"state shape {tuple(state.data.shape)} != operator {self.state_shape}")

    def raise_on_status(self, flags: int):
        if flags & _lib.STATUS_POSITIVITY:
            raise PositivityError("non-positive water height at a quadrature node")
        if flags & _lib.STATUS_PEER_TIMEOUT:
            raise RuntimeError("a latitude-band neighbour's halo rows never arrived")

    def assemble_rhs(self, state: State, out: State | None = None, check: bool = True) -> State:
        """Full right-hand side M^-1 (volume - boundary + source); raises
        PositivityError like the reference when ``check`` (one device sync)."""
        self._check(state)
        if out is None:
            out = self.zero_state()
        self._check(out)
        self.timers.begin("main")
        c = self._ctx
        _lib.check(c.lib.dgswe_rhs(c.h, _ptr(state.data), _ptr(out.data), c.stream()), "dgswe_rhs")
        self.timers.end("main")
        self._record("rhs", "dgswe_rhs", 16.0)
        if check:
            flags, _ = c.status(reset=True)
            self.raise_on_status(flags)
        return out

    def stage(self, a: float, U: State | None, b: float, X: State, g: float, Y: State, tag: int = 0):
        """Y = a U + b X + g RHS(X) in one launch (no sync)."""
        c = self._ctx
        _lib.check(c.lib.dgswe_stage(c.h, float(a), _ptr(U.data if U is not None else None),
                                     float(b), _ptr(X.data), float(g), _ptr(Y.data), int(tag),
                                     c.stream()), "dgswe_stage")
        self._record("stage", "dgswe_stage", 24.0 if U is not None and a != 0.0 else 16.0)

    def axpy(self, coef: float, x: State, y: State, check_finite: bool = False, tag: int = 0):
        """y += x*coef with the reference's two roundings (timestep.py:137-141)."""
        c = self._ctx
        _lib.check(c.lib.dgswe_axpy(c.h, float(coef), _ptr(x.data), _ptr(y.data),
                                    int(check_finite), int(tag), c.stream()), "dgswe_axpy")
        self._record("axpy", "dgswe_axpy", 24.0, flops=2.0)

    def rk_steps(self, state: State, dt: float, nsteps: int, order: int = 3, check_mean: bool = False):
        """nsteps fused steps of tableau(order) (1..4) in place, one CUDA graph:
        Euler, Heun / SSPRK3 in Shu-Osher form, classical RK4 with the
        accumulator as the stage kernel's second output."""
        self._check(state)
        key = state.data.data_ptr()
        ws = self._scratch.get(key)
        if ws is None:
            # zeroed once: the strip padding past nx is read but never written
            ws = tuple(torch.zeros_like(state.data) for _ in range(3))
            self._scratch = {k: v for k, v in self._scratch.items() if not isinstance(k, int)}
            self._scratch[key] = ws
        c = self._ctx
        _lib.check(c.lib.dgswe_rk_steps(c.h, int(order), _ptr(state.data), _ptr(ws[0]), _ptr(ws[1]),
                                        _ptr(ws[2]), float(dt), int(nsteps), int(check_mean), c.stream()),
                   "dgswe_rk_steps")
        # stage bytes per step: Euler 16, Heun 16 + 24, SSPRK3 16 + 24 + 24, RK4 (accumulator) 32 + 40 + 40 + 24
        per_step = {1: 16.0, 2: 40.0, 3: 64.0, 4: 136.0}[int(order)]
        self._record("rk_steps", f"dgswe_rk_steps(order={int(order)})", per_step * nsteps,
                     flops=tracing.stage_flops_per_dof(self.p) * int(order) * nsteps)

    def ssprk3_steps(self, state: State, dt: float, nsteps: int, check_mean: bool = False):
        """nsteps fused Shu-Osher SSPRK3 steps in place (one CUDA graph)."""
        self.rk_steps(state, dt, nsteps, 3, check_mean)

    def ssprk3_step_host(self, host: torch.Tensor, dt: float, tag: int = 0, check_mean: bool = False,
                         chunks: int | None = None, graph: bool = True):
        """One SSPRK3 step of a host-resident (pinned) modal state, in place:
        the reference's ``rk_step`` contract on a host array
        (timestep.py:149-167), row-pipelined.  The state moves in latitude
        chunks; chunk c's host->device copy, chunk c-1's stage 1, c-2's
        stage 2, c-3's stage 3 and the device->host copy of finished chunks
        overlap (two copy streams: PCIe is full duplex).  Bitwise equal to
        ``ssprk3_steps(state, dt, 1)`` on the device copy.  Enqueued on the
        current stream (which waits for the last copy); ``status()`` syncs.
        With ``graph`` the ~10 launches per chunk are captured once per
        (host buffer, dt, tag, check_mean) and replayed as one CUDA graph."""
        mesh = self.mesh
        ny, nz = mesh.ny, self.nz
        # argument checks before any graph lookup: a replay must never run on
        # a buffer the capture was not made for
        if tuple(host.shape) != tuple(self.state_shape) or host.dtype != torch.float64:
            raise ValueError(f"host state must be float64 {tuple(self.state_shape)}")
        if host.device.type != "cpu" or not host.is_pinned() or not host.is_contiguous():
            raise ValueError("host state must be a contiguous pinned CPU tensor")
        if chunks is not None and not 1 <= int(chunks) <= ny:
            raise ValueError(f"chunks must be in [1, ny={ny}], got {chunks}")
        if self.rusanov.mode == "global" and self.rusanov.alpha is None:
            raise ValueError("global-alpha mode needs the whole state before a stage: use ssprk3_steps")
        if graph:
            gkey = ("hostgraph", host.data_ptr(), float(dt), int(tag), bool(check_mean), chunks)
            g = self._scratch.get(gkey)
            if g is None:
                if sum(1 for k in self._scratch if isinstance(k, tuple) and k[0] == "hostgraph") >= 8:
                    for k in [k for k in self._scratch if isinstance(k, tuple) and k[0] == "hostgraph"]:
                        del self._scratch[k]
                self.ssprk3_step_host(host, dt, tag, check_mean, chunks, graph=False)   # warm-up step
                torch.cuda.current_stream().synchronize()
                g = torch.cuda.CUDAGraph()             # captured, not run: this call's step was the eager one
                with torch.cuda.graph(g):
                    self.ssprk3_step_host(host, dt, tag, check_mean, chunks, graph=False)
                self._scratch[gkey] = g
                return
            g.replay()
            return
        nch = chunks if chunks is not None else max(1, min(16, ny // 4))
        bounds = [ny * c // nch for c in range(nch + 1)]
        key = ("host", tuple(host.shape))
        ws = self._scratch.get(key)
        if ws is None:
            ws = tuple(torch.zeros(self.state_shape, dtype=torch.float64, device=self.device) for _ in range(3))
            ws = ws + (torch.cuda.Stream(), torch.cuda.Stream())
            self._scratch[key] = ws
        u, w1, w2, s_in, s_out = ws
        c = self._ctx
        cur = torch.cuda.current_stream()
        s_in.wait_stream(cur)
        s_out.wait_stream(cur)
        ev_in = [torch.cuda.Event() for _ in range(nch)]

        def rows(k):
            return bounds[k], bounds[k + 1]

        def launch(fn, a, U, b, X, g, Y, k, last=False):
            r0, r1 = rows(k)
            if last:
                _lib.check(c.lib.dgswe_stage_rows_checked(
                    c.h, float(a), _ptr(U), float(b), _ptr(X), float(g), _ptr(Y), int(tag), r0, r1, 1,
                    int(check_mean), c.stream()), "dgswe_stage_rows_checked")
            else:
                _lib.check(c.lib.dgswe_stage_rows(
                    c.h, float(a), _ptr(U), float(b), _ptr(X), float(g), _ptr(Y), int(tag), r0, r1,
                    c.stream()), "dgswe_stage_rows")

        c.set_basis(True)
        try:
            for it in range(nch + 3):
                if it < nch:
                    r0, r1 = rows(it)
                    with torch.cuda.stream(s_in):
                        for z in range(nz):
                            u[z, r0:r1].copy_(host[z, r0:r1], non_blocking=True)
                        ev_in[it].record(s_in)
                    cur.wait_event(ev_in[it])
                    c.convert(u, True, r0, r1)
                if 0 <= it - 1 < nch:
                    launch(None, 0.0, None, 1.0, u, dt, w1, it - 1)
                if 0 <= it - 2 < nch:
                    launch(None, 0.75, u, 0.25, w1, 0.25 * dt, w2, it - 2)
                k3 = it - 3
                if 0 <= k3 < nch:
                    launch(None, 1.0 / 3.0, u, 2.0 / 3.0, w2, (2.0 / 3.0) * dt, u, k3, last=True)
                    r0, r1 = rows(k3)
                    c.convert(u, False, r0, r1)
                    ev = torch.cuda.Event()
                    ev.record(cur)
                    s_out.wait_event(ev)
                    with torch.cuda.stream(s_out):
                        for z in range(nz):
                            host[z, r0:r1].copy_(u[z, r0:r1], non_blocking=True)
        finally:
            c.set_basis(False)
        cur.wait_stream(s_out)
        cur.wait_stream(s_in)

    def rk_step_fused(self, state: State, dt: float, order: int, bufs, tag: int = 0) -> torch.Tensor:
        """One step of tableau(order) (1..4) in fused stage form on the
        nodal values: ``state`` is converted to nodal values in place if it
        holds modes (once; it stays nodal until it is read, see State), then
        ``order`` stage kernels -- the same launches as a step of
        ``rk_steps`` (no other kernel, no allocation) -- the last one writing
        the new state into ``bufs[order-1]`` with the non-finite check.
        Returns that raw (nodal) buffer; ``state`` keeps u^n (the caller
        swaps on success, so a PositivityError leaves u^n in place like the
        reference)."""
        c = self._ctx
        if state._nodal is self:
            u = state._data
        else:
            # first fused step of a modal state: convert a copy (the spare
            # buffer), so a PositivityError leaves the caller's modes untouched
            spare = bufs[-1]
            spare._data.copy_(state.data)
            spare._nodal = None
            u = spare._as_nodal(self)
            bufs = bufs[:-1]

        def stage(a, U, b, X, g, Y, check=False):
            _lib.check(c.lib.dgswe_stage_rows_checked(
                c.h, float(a), _ptr(U), float(b), _ptr(X), float(g), _ptr(Y), int(tag), 0, self.mesh.ny,
                int(check), 0, c.stream()), "dgswe_stage_rows_checked")

        def stage2(a, U, b, X, g, Y, A, g2, Y2):
            _lib.check(c.lib.dgswe_stage2(c.h, float(a), _ptr(U), float(b), _ptr(X), float(g), _ptr(Y),
                                          _ptr(A), float(g2), _ptr(Y2), int(tag), 0, self.mesh.ny, c.stream()),
                       "dgswe_stage2")

        b = [x._data if isinstance(x, State) else x for x in bufs]
        if order not in (1, 2, 3, 4):
            raise ValueError(f"unsupported RK order {order}; choose 1..4")
        # the step's launches are captured once per (buffers, dt, order) and
        # replayed as one CUDA graph (the state/workspace swap alternates
        # between two buffer assignments, so two graphs serve a run)
        key = ("rkstep", order, float(dt), int(tag), u.data_ptr(), tuple(x.data_ptr() for x in b[:order]))
        g = self._scratch.get(key)
        if g is not None and self.rusanov.mode == "local":
            g.replay()
            self._replayed += order
            return b[order - 1]
        out = self._rk_stages(u, b, dt, order, tag, stage, stage2)
        if self.rusanov.mode == "local":
            if sum(1 for k in self._scratch if isinstance(k, tuple) and k[0] == "rkstep") >= 8:
                for k in [k for k in self._scratch if isinstance(k, tuple) and k[0] == "rkstep"]:
                    del self._scratch[k]
            g = torch.cuda.CUDAGraph()              # captured, not run: this call's step was the eager one
            with torch.cuda.graph(g):
                self._rk_stages(u, b, dt, order, tag, stage, stage2)
            self._replayed -= order                 # the C counter counted the captured launches
            self._scratch[key] = g
        return out

    def _rk_stages(self, u, b, dt, order, tag, stage, stage2):
        c = self._ctx
        c.set_basis(True)
        try:
            if order == 1:
                stage(0.0, None, 1.0, u, dt, b[0], check=True)
                return b[0]
            if order == 2:
                stage(0.0, None, 1.0, u, dt, b[0])
                stage(0.5, u, 0.5, b[0], 0.5 * dt, b[1], check=True)
                return b[1]
            if order == 3:
                stage(0.0, None, 1.0, u, dt, b[0])
                stage(0.75, u, 0.25, b[0], 0.25 * dt, b[1])
                stage(1.0 / 3.0, u, 2.0 / 3.0, b[1], (2.0 / 3.0) * dt, b[2], check=True)
                return b[2]
            w1, w2, acc, out = b[0], b[1], b[2], b[3]
            stage2(0.0, None, 1.0, u, 0.5 * dt, w1, u, dt / 6.0, acc)
            stage2(1.0, u, 0.0, w1, 0.5 * dt, w2, acc, dt / 3.0, acc)
            stage2(1.0, u, 0.0, w2, dt, w1, acc, dt / 3.0, acc)
            stage(1.0, acc, 0.0, w1, dt / 6.0, out, check=True)
            return out
        finally:
            c.set_basis(False)

    def stage2(self, a: float, U: State | None, b: float, X: State, g: float, Y: State, A: State,
               g2: float, Y2: State, tag: int = 0):
        """Y = a U + b X + g RHS(X) and Y2 = A + g2 RHS(X) in one launch (no sync)."""
        c = self._ctx
        _lib.check(c.lib.dgswe_stage2(c.h, float(a), _ptr(U.data if U is not None else None), float(b),
                                      _ptr(X.data), float(g), _ptr(Y.data), _ptr(A.data), float(g2),
                                      _ptr(Y2.data), int(tag), 0, self.mesh.ny, c.stream()),
                   "dgswe_stage2")

    def status(self, reset: bool = True):
        return self._ctx.status(reset)

    def status_tags(self, reset: bool = True):
        return self._ctx.status_tags(reset)

    def _record(self, kind: str, op: str, bytes_per_dof: float, flops: float | None = None):
        """One op-recorder entry (tracing.set_op_recorder) for a launch over all rows."""
        if tracing.get_op_recorder() is not None:
            rgn = tracing.LaunchRegion((self.mesh.nx, self.mesh.ny, self.nz), self.p)
            tracing.record(kind, op, rgn, bytes_per_dof,
                           tracing.stage_flops_per_dof(self.p) if flops is None else flops)

    def launch_count(self) -> int:
        return self._ctx.launches() + self._replayed

    # -- host-side helpers (diagnostics / step control) ---------------------

    def interior_nodal_values(self, state: State) -> dict:
        """(nx, ny, nz, nq) nodal values per variable."""
        if self._phi_dev is None:
            self._phi_dev = torch.from_numpy(self.vander.phi).to(self.device)
        U = torch.einsum("qm,zjvmi->vijzq", self._phi_dev, lon_major(state.data, self.mesh.nx))
        return {n: U[v].cpu().numpy() for v, n in enumerate(VAR_NAMES)}

    def max_physical_speed(self, state: State) -> float:
        """max over interior nodes of max(|u|,|v|) + sqrt(g h) (models.py:282-285)."""
        if self._phi_dev is None:
            self._phi_dev = torch.from_numpy(self.vander.phi).to(self.device)
        U = torch.einsum("qm,zjvmi->vzjqi", self._phi_dev, lon_major(state.data, self.mesh.nx))
        h = U[0]
        hf = torch.clamp_min(h, self.model.h_floor)
        c = torch.sqrt(self.model.gravity * torch.clamp_min(h, 0.0))
        vel = torch.maximum((U[1] / hf).abs(), (U[2] / hf).abs())
        return float((vel + c).max().item())
