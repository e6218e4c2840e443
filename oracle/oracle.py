"""CPU oracle for the DG shallow-water time-stepping path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference``) may import
this module, and only as the checker / CPU baseline.  The product package
``paper_2303_11767_b200`` never imports it.

Two layers:

* numpy restatement of the reference's host-side setup (mesh, Gauss rule,
  Legendre recurrences, Vandermonde tables, per-row cos-weighted mass
  matrices, node metric tables, Williamson ICs and their L2 projection,
  mass integral, L2 error), in the reference's operation order so every
  table is bit-identical (pinned by tests/test_oracle_golden.py);
* ctypes binding of ``oracle/dgswe_oracle.c`` (built into
  ``oracle/liboracle.so``), the RHS + Butcher RK step in the reference's
  exact operation order, OpenMP over elements.

Parity pin: SHA-256 of the oracle's coefficients equals the fixtures
generated from the unmodified reference (tests/golden/golden.json), e.g.
TC2 40x20 p=2 dt=10 RK3: IC 5923f725ddeb20c9 -> 100 steps 438852d718a262a2.

Reference citations are to /root/reference/pkg/src/dgswe/<file>:<line>.
"""

from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")

# physical constants (mesh.py:28-36) and Williamson constants (cases.py:32-45)
RADIUS = 6.37122e6
OMEGA = 7.292e-5
GRAVITY = 9.81
DAY = 86400.0
TC2_U0 = 2.0 * math.pi * RADIUS / (12.0 * DAY)
TC2_GH0 = 2.94e4
TC6_OMEGA = 7.848e-6
TC6_K = 7.848e-6
TC6_H0 = 8.0e3
TC6_R = 4

LEFT, RIGHT, BOTTOM, TOP = range(4)


# --------------------------------------------------------------------------
# setup (basis.py, mesh.py, dg.py:186-283)

def legendre(j, x):
    """P_j by the three-term recurrence (basis.py:58-66)."""
    x = np.asarray(x, dtype=np.float64)
    if j == 0:
        return np.ones_like(x)
    a, b = np.ones_like(x), x.copy()
    for k in range(1, j):
        a, b = b, ((2 * k + 1) * x * b - k * a) / (k + 1)
    return b


def legendre_d(j, x):
    """P_j' with P'_{k+1} = P'_{k-1} + (2k+1) P_k (basis.py:69-81)."""
    x = np.asarray(x, dtype=np.float64)
    if j == 0:
        return np.zeros_like(x)
    a, b = np.ones_like(x), x.copy()
    da, db = np.zeros_like(x), np.ones_like(x)
    for k in range(1, j):
        nb = ((2 * k + 1) * x * b - k * a) / (k + 1)
        ndb = da + (2 * k + 1) * b
        a, b = b, nb
        da, db = db, ndb
    return db


def vander_tables(p, nodes):
    """phi, d/dxi, d/deta and edge traces (basis.py:109-143)."""
    n = len(nodes)
    nphi = (p + 1) ** 2
    P = np.stack([legendre(a, nodes) for a in range(p + 1)])
    D = np.stack([legendre_d(a, nodes) for a in range(p + 1)])
    Pm = np.array([legendre(a, -1.0) for a in range(p + 1)]).reshape(p + 1)
    Pp = np.array([legendre(a, 1.0) for a in range(p + 1)]).reshape(p + 1)
    phi = np.empty((n * n, nphi))
    gx = np.empty_like(phi)
    gy = np.empty_like(phi)
    E = [np.empty((n, nphi)) for _ in range(4)]
    for a in range(p + 1):
        for b in range(p + 1):
            m = a * (p + 1) + b
            for qi in range(n):
                for qj in range(n):
                    q = qi * n + qj
                    phi[q, m] = P[a, qi] * P[b, qj]
                    gx[q, m] = D[a, qi] * P[b, qj]
                    gy[q, m] = P[a, qi] * D[b, qj]
            for q in range(n):
                E[LEFT][q, m] = Pm[a] * P[b, q]
                E[RIGHT][q, m] = Pp[a] * P[b, q]
                E[BOTTOM][q, m] = P[a, q] * Pm[b]
                E[TOP][q, m] = P[a, q] * Pp[b]
    return phi, gx, gy, E


@dataclass
class Tables:
    nx: int
    ny: int
    p: int
    nz: int
    h_floor: float
    alpha_mode: int
    alpha: float
    x_edges: np.ndarray
    y_edges: np.ndarray
    dx: float
    dy: float
    determ: float
    nodes: np.ndarray
    weights: np.ndarray
    phi: np.ndarray
    edge: list
    volx: np.ndarray
    voly: np.ndarray
    bnd: list
    src: np.ndarray
    M_rows: np.ndarray
    Minv: np.ndarray
    coords: dict        # name -> (cos_over_r, sin_over_r, f_cos), shape (ny+2, k)
    cos_yb: np.ndarray  # (ny,) np.cos(bottom edge latitude)
    cos_yt: np.ndarray

    @property
    def n1(self):
        return self.p + 1

    @property
    def nphi(self):
        return (self.p + 1) ** 2


def row_mass(p, tb, tt, nodes, weights, dlam, phi):
    """cos-weighted per-row mass matrix and inverse (basis.py:159-176)."""
    theta_q = 0.5 * (tb + tt) + 0.5 * (tt - tb) * nodes
    cos_q = np.cos(theta_q)
    w_metric = np.outer(weights, weights * cos_q).reshape(-1)
    determ = dlam * (tt - tb) / 4.0
    M = determ * (phi.T * w_metric) @ phi
    M = 0.5 * (M + M.T)
    np.linalg.cholesky(M)
    return M, np.linalg.inv(M)


def make_tables(nx, ny, p, h_ref, nz=1, alpha_mode="local", alpha=None):
    x_edges = np.linspace(0.0, 2.0 * math.pi, nx + 1)
    y_edges = np.linspace(-math.pi / 2.0, math.pi / 2.0, ny + 1)
    dx = float(x_edges[1] - x_edges[0])
    dy = float(y_edges[1] - y_edges[0])
    determ = dx * dy / 4.0
    bdx, bdy = dx / 2.0, dy / 2.0
    nodes, weights = np.polynomial.legendre.leggauss(p + 1)
    phi, gx, gy, E = vander_tables(p, nodes)
    w2 = np.outer(weights, weights).reshape(-1)
    volx = (determ / bdx) * (w2[:, None] * gx)
    voly = (determ / bdy) * (w2[:, None] * gy)
    we = weights[:, None]
    bnd = [-bdy * (we * E[LEFT]), +bdy * (we * E[RIGHT]),
           -bdx * (we * E[BOTTOM]), +bdx * (we * E[TOP])]
    src = determ * (w2[:, None] * phi)
    nphi = (p + 1) ** 2
    M = np.empty((ny, nphi, nphi))
    Minv = np.empty_like(M)
    for j in range(ny):
        M[j], Minv[j] = row_mass(p, y_edges[j], y_edges[j + 1], nodes, weights, dx, phi)
    # node latitudes per row slot (dg.py:264-283); halo rows clamp
    nyh = ny + 2
    ylo = np.empty(nyh)
    ylo[1:ny + 1] = y_edges[:-1]
    ylo[0], ylo[-1] = y_edges[0], y_edges[-2]
    th_nodes = ylo[:, None] + 0.5 * dy * (1.0 + nodes)[None, :]
    n1 = p + 1
    th_int = np.repeat(th_nodes[:, None, :], n1, axis=1).reshape(nyh, n1 * n1)
    yb = np.empty(nyh)
    yb[1:ny + 1] = y_edges[:-1]
    yb[0], yb[-1] = y_edges[0], y_edges[-2]
    yt = np.empty(nyh)
    yt[1:ny + 1] = y_edges[1:]
    yt[0], yt[-1] = y_edges[1], y_edges[-1]

    def trig(th):
        return (np.cos(th) / RADIUS, np.sin(th) / RADIUS, 2.0 * OMEGA * np.sin(th) * np.cos(th))

    coords = {"int": trig(th_int), "xe": trig(th_nodes), "yb": trig(yb[:, None]),
              "yt": trig(yt[:, None])}
    mode = {"local": 0, "global": 1 if alpha is not None else 2}[alpha_mode]
    return Tables(nx=nx, ny=ny, p=p, nz=nz, h_floor=1e-8 * float(h_ref), alpha_mode=mode,
                  alpha=float(alpha) if alpha is not None else 0.0,
                  x_edges=x_edges, y_edges=y_edges, dx=dx, dy=dy, determ=determ,
                  nodes=nodes, weights=weights, phi=phi, edge=E, volx=volx, voly=voly,
                  bnd=bnd, src=src, M_rows=M, Minv=Minv, coords=coords,
                  cos_yb=np.cos(yb[1:ny + 1]), cos_yt=np.cos(yt[1:ny + 1]))


# --------------------------------------------------------------------------
# Williamson initial conditions (cases.py:126-179) and projection

def ic_tc2():
    a, g = RADIUS, GRAVITY
    u0 = TC2_U0
    coef = a * OMEGA * u0 + 0.5 * u0 * u0

    def height(lam, th):
        return (TC2_GH0 - coef * np.sin(th) ** 2) / g + 0.0 * lam

    def h_u(lam, th):
        return height(lam, th) * u0 * np.cos(th)

    def zero(lam, th):
        return np.zeros(np.broadcast(lam, th).shape)

    return {"h": height, "hu": h_u, "hv": zero}, height


def ic_tc6():
    a, g, Om = RADIUS, GRAVITY, OMEGA
    w, K, R = TC6_OMEGA, TC6_K, TC6_R

    def winds(lam, th):
        cth = np.cos(th)
        u = a * w * cth + a * K * cth ** (R - 1) * (
            R * np.sin(th) ** 2 - cth**2) * np.cos(R * lam)
        v = -a * K * R * cth ** (R - 1) * np.sin(th) * np.sin(R * lam)
        return u, v

    def height(lam, th):
        cth = np.cos(th)
        A = 0.5 * w * (2.0 * Om + w) * cth**2 + 0.25 * K**2 * cth ** (2 * R) * (
            (R + 1) * cth**2 + (2 * R**2 - R - 2) - 2.0 * R**2 * cth ** (-2))
        B = (2.0 * (Om + w) * K) / ((R + 1) * (R + 2)) * cth**R * (
            (R**2 + 2 * R + 2) - (R + 1) ** 2 * cth**2)
        C = 0.25 * K**2 * cth ** (2 * R) * ((R + 1) * cth**2 - (R + 2))
        return TC6_H0 + (a * a / g) * (A + B * np.cos(R * lam) + C * np.cos(2 * R * lam))

    return {"h": height,
            "hu": lambda lam, th: height(lam, th) * winds(lam, th)[0],
            "hv": lambda lam, th: height(lam, th) * winds(lam, th)[1]}


# Williamson TC5 (zonal flow over an isolated mountain, Williamson et al. 1992
# section 3.5).  EXTENSION: the reference has no orography, so
# this case is "parity unpinned" -- the oracle restates the same source the
# CUDA path adds, -g h grad b, with grad b the derivative of b's degree-p
# nodal interpolant (see orography_factors).
TC5_U0 = 20.0
TC5_H0 = 5960.0
TC5_HS0 = 2000.0
TC5_RM = math.pi / 9.0
TC5_LC = 1.5 * math.pi
TC5_TC = math.pi / 6.0


def tc5_bottom(lam, th):
    r = np.minimum(TC5_RM, np.sqrt((lam - TC5_LC) ** 2 + (th - TC5_TC) ** 2))
    return TC5_HS0 * (1.0 - r / TC5_RM)


def ic_tc5():
    coef = RADIUS * OMEGA * TC5_U0 + 0.5 * TC5_U0 * TC5_U0

    def depth(lam, th):
        return (GRAVITY * TC5_H0 - coef * np.sin(th) ** 2) / GRAVITY - tc5_bottom(lam, th)

    return {"h": depth,
            "hu": lambda lam, th: depth(lam, th) * TC5_U0 * np.cos(th),
            "hv": lambda lam, th: np.zeros(np.broadcast(lam, th).shape)}


H_REF = {"williamson_tc2": TC2_GH0 / GRAVITY, "williamson_tc6": TC6_H0, "williamson_tc5": TC5_H0}


def ic_funcs(case):
    if case == "williamson_tc5":
        return ic_tc5()
    return ic_tc2()[0] if case == "williamson_tc2" else ic_tc6()


def orography_factors(t, bottom):
    """(nx, ny, nq) factors -(g/R) db/dlambda and -(g cos/R) db/dtheta at the
    interior nodes, grad b from the nodal interpolant of b:
    db/dxi(x_i, x_j) = sum_k l_k'(x_i) b(x_k, x_j), l_k' from the Legendre
    expansion l_k(x) = sum_a (2a+1)/2 w_k P_a(x_k) P_a(x)."""
    n = t.p + 1
    x, y = node_coords(t, t.nodes)
    b = np.broadcast_to(bottom(x[:, None, :, None], y[None, :, None, :]), (t.nx, t.ny, n, n))
    P = np.stack([legendre(a, t.nodes) for a in range(n)])          # [a][k]
    dP = np.stack([legendre_d(a, t.nodes) for a in range(n)])       # [a][i]
    scale = np.array([(2 * a + 1) / 2.0 for a in range(n)])
    D = np.einsum("a,ai,ak,k->ik", scale, dP, P, t.weights)           # D[i][k] = l_k'(x_i)
    dxi = np.einsum("ik,xykj->xyij", D, b)
    deta = np.einsum("jk,xyik->xyij", D, b)
    cos_n = np.cos(y)                                               # (ny, n) node latitudes
    ox = -(GRAVITY / RADIUS) * dxi * (2.0 / t.dx)
    oy = -(GRAVITY / RADIUS) * cos_n[None, :, None, :] * deta * (2.0 / t.dy)
    return (np.ascontiguousarray(ox.reshape(t.nx, t.ny, n * n)),
            np.ascontiguousarray(oy.reshape(t.nx, t.ny, n * n)))


def node_coords(t: Tables, nodes):
    x = t.x_edges[:-1][:, None] + 0.5 * t.dx * (1.0 + nodes)[None, :]
    y = t.y_edges[:-1][:, None] + 0.5 * t.dy * (1.0 + nodes)[None, :]
    return x, y


def project(t: Tables, f):
    """L2 projection with the cos metric (basis.py:206-233); (nx, ny, nphi)."""
    n1 = t.n1
    x, y = node_coords(t, t.nodes)
    fv = f(x[:, None, :, None], y[None, :, None, :])
    fv = np.broadcast_to(fv, (t.nx, t.ny, n1, n1)).reshape(t.nx, t.ny, n1 * n1)
    qw = np.outer(t.weights, t.weights).reshape(-1)
    cos_q = np.cos(y)
    w_rows = (qw.reshape(n1, n1)[None, :, :] * cos_q[:, None, :]).reshape(t.ny, n1 * n1)
    rhs = t.determ * np.einsum("xyq,yq,qm->xym", fv, w_rows, t.phi)
    Minv = np.empty((t.ny, t.nphi, t.nphi))
    for j in range(t.ny):
        Minv[j] = row_mass(t.p, t.y_edges[j], t.y_edges[j + 1], t.nodes, t.weights,
                           t.dx, t.phi)[1]
    return np.ascontiguousarray(np.einsum("ymn,xyn->xym", Minv, rhs))


def initial_state(t: Tables, case):
    """(3, nx, ny, nz, nphi) projected IC, same on every level."""
    f = ic_funcs(case)
    out = np.empty((3, t.nx, t.ny, t.nz, t.nphi))
    for v, name in enumerate(("h", "hu", "hv")):
        out[v] = project(t, f[name])[:, :, None, :]
    return out


# --------------------------------------------------------------------------
# diagnostics (diagnostics.py:42-107)

def mass_integral(t: Tables, X, level=0):
    coeffs = X[0, :, :, level, :]
    cell = np.einsum("ym,xym->xy", t.M_rows[:, 0, :], coeffs)
    total = 0.0
    for i in range(t.nx):
        for j in range(t.ny):
            total += cell[i, j]
    return total


def l2_error(t: Tables, X, ref_fn, var=0, relative=False, level=0):
    n1 = t.p + 2
    nodes, weights = np.polynomial.legendre.leggauss(n1)
    phi = vander_tables(t.p, nodes)[0]
    coeffs = X[var, :, :, level, :]
    vals = np.einsum("qm,xym->xyq", phi, coeffs)
    x, y = node_coords(t, nodes)
    ref = ref_fn(x[:, None, :, None], y[None, :, None, :])
    ref = np.broadcast_to(ref, (t.nx, t.ny, n1, n1)).reshape(t.nx, t.ny, n1 * n1)
    w2 = np.outer(weights, weights).reshape(-1)
    w_rows = (w2.reshape(n1, n1)[None, :, :] * np.cos(y)[:, None, :]).reshape(t.ny, n1 * n1)
    cell = t.determ * np.einsum("xyq,yq->xy", (vals - ref) ** 2, w_rows)
    cell_ref = t.determ * np.einsum("xyq,yq->xy", ref**2, w_rows)
    total = 0.0
    total_ref = 0.0
    for i in range(t.nx):
        for j in range(t.ny):
            total += cell[i, j]
            total_ref += cell_ref[i, j]
    err = math.sqrt(max(total, 0.0))
    return err / math.sqrt(max(total_ref, 1e-300)) if relative else err


# --------------------------------------------------------------------------
# C core binding

_P = ctypes.POINTER(ctypes.c_double)


class _Cfg(ctypes.Structure):
    _fields_ = [
        ("nx", ctypes.c_int), ("ny", ctypes.c_int), ("nz", ctypes.c_int), ("p", ctypes.c_int),
        ("radius", ctypes.c_double), ("inv_r", ctypes.c_double),
        ("gravity", ctypes.c_double), ("half_g", ctypes.c_double),
        ("h_floor", ctypes.c_double), ("alpha_mode", ctypes.c_int), ("alpha", ctypes.c_double),
        ("phi", _P), ("edge", _P * 4), ("volx", _P), ("voly", _P), ("src", _P),
        ("bnd", _P * 4), ("minv", _P), ("cr_int", _P), ("sr_int", _P), ("fc_int", _P),
        ("cr_yb", _P), ("cr_yt", _P), ("cos_yb", _P), ("cos_yt", _P),
        ("orog_x", _P), ("orog_y", _P),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"oracle library missing: build with `make -C {HERE}`")
        _lib = ctypes.CDLL(LIB_PATH)
        _lib.oracle_rhs.argtypes = [ctypes.POINTER(_Cfg), _P, _P, ctypes.c_int]
        _lib.oracle_rhs.restype = ctypes.c_int
        _lib.oracle_rk_steps.argtypes = [ctypes.POINTER(_Cfg), _P, ctypes.c_double, ctypes.c_int,
                                         _P, _P, ctypes.c_int, ctypes.c_int,
                                         ctypes.POINTER(ctypes.c_int)]
        _lib.oracle_rk_steps.restype = ctypes.c_int
        _lib.oracle_max_threads.restype = ctypes.c_int
    return _lib


def max_threads():
    return lib().oracle_max_threads()


def _ptr(a):
    return a.ctypes.data_as(_P)


class Oracle:
    """Bound oracle for one Tables instance (keeps the C arrays alive)."""

    POSITIVITY = 1
    NONFINITE = 2

    def __init__(self, t: Tables, bottom=None):
        self.t = t
        ny = t.ny
        c = lambda a: np.ascontiguousarray(a, dtype=np.float64)
        ci, cx, cb, ct = t.coords["int"], t.coords["xe"], t.coords["yb"], t.coords["yt"]
        keep = {
            "phi": c(t.phi), "volx": c(t.volx), "voly": c(t.voly), "src": c(t.src),
            "minv": c(t.Minv),
            "cr_int": c(ci[0][1:ny + 1]), "sr_int": c(ci[1][1:ny + 1]),
            "fc_int": c(ci[2][1:ny + 1]),
            "cr_yb": c(cb[0][1:ny + 1, 0]), "cr_yt": c(ct[0][1:ny + 1, 0]),
            "cos_yb": c(t.cos_yb), "cos_yt": c(t.cos_yt),
        }
        edges = [c(e) for e in t.edge]
        bnds = [c(b) for b in t.bnd]
        orog = orography_factors(t, bottom) if bottom is not None else None
        self._keep = (keep, edges, bnds, orog)
        cfg = _Cfg()
        cfg.nx, cfg.ny, cfg.nz, cfg.p = t.nx, t.ny, t.nz, t.p
        cfg.radius = RADIUS
        cfg.inv_r = 1.0 / RADIUS
        cfg.gravity = GRAVITY
        cfg.half_g = 0.5 * GRAVITY
        cfg.h_floor = t.h_floor
        cfg.alpha_mode = t.alpha_mode
        cfg.alpha = t.alpha
        for k, v in keep.items():
            setattr(cfg, k, _ptr(v))
        for e in range(4):
            cfg.edge[e] = _ptr(edges[e])
            cfg.bnd[e] = _ptr(bnds[e])
        if orog is not None:
            cfg.orog_x, cfg.orog_y = _ptr(orog[0]), _ptr(orog[1])
        self.cfg = cfg

    def rhs(self, X, nthreads=0):
        X = np.ascontiguousarray(X, dtype=np.float64)
        K = np.empty_like(X)
        st = lib().oracle_rhs(ctypes.byref(self.cfg), _ptr(X), _ptr(K), nthreads)
        if st < 0:
            raise MemoryError("oracle workspace allocation failed")
        if st & self.POSITIVITY:
            raise ArithmeticError("oracle: non-positive water height")
        return K

    def rk_steps(self, X, dt, order, nsteps, nthreads=0):
        """Butcher steps in place on a copy; returns (state, status, steps_done)."""
        A, b = TABLEAUX[order]
        s = len(b)
        u = np.array(X, dtype=np.float64, order="C", copy=True)
        a = np.ascontiguousarray(np.array(A, dtype=np.float64).reshape(s * s))
        bb = np.ascontiguousarray(np.array(b, dtype=np.float64))
        done = ctypes.c_int(0)
        st = lib().oracle_rk_steps(ctypes.byref(self.cfg), _ptr(u), float(dt), s, _ptr(a),
                                   _ptr(bb), int(nsteps), nthreads, ctypes.byref(done))
        if st < 0:
            raise MemoryError("oracle workspace allocation failed")
        return u, st, done.value


# timestep.py:57-82
TABLEAUX = {
    1: (((0.0,),), (1.0,)),
    2: (((0.0, 0.0), (1.0, 0.0)), (0.5, 0.5)),
    3: (((0.0, 0.0, 0.0), (1.0, 0.0, 0.0), (0.25, 0.25, 0.0)),
        (1.0 / 6.0, 1.0 / 6.0, 2.0 / 3.0)),
    4: (((0.0, 0.0, 0.0, 0.0), (0.5, 0.0, 0.0, 0.0), (0.0, 0.5, 0.0, 0.0), (0.0, 0.0, 1.0, 0.0)),
        (1.0 / 6.0, 1.0 / 3.0, 1.0 / 3.0, 1.0 / 6.0)),
}


def sha16(X):
    import hashlib
    h = hashlib.sha256()
    for v in range(X.shape[0]):
        h.update(np.ascontiguousarray(X[v]).tobytes())
    return h.hexdigest()[:16]


def build_case(case, nx, ny, p, nz=1, alpha_mode="local", alpha=None):
    """(Tables, Oracle, initial state) for a Williamson case (TC5: with its
    orography, an extension of the reference)."""
    t = make_tables(nx, ny, p, H_REF[case], nz=nz, alpha_mode=alpha_mode, alpha=alpha)
    return t, Oracle(t, tc5_bottom if case == "williamson_tc5" else None), initial_state(t, case)
