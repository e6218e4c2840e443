"""Host-side discretisation setup: lat-lon mesh, Gauss rule, modal Legendre
basis tables and per-row cos-weighted mass matrices.

Mirrors the reference setup API (``build_latlon_mesh``, ``gauss_legendre``,
``build_vander``, ``mass_matrix_sphere``, ``sphere_row_mass_matrices``,
``project_initial``; /root/reference/pkg/src/dgswe/mesh.py:136-174 and
basis.py:50-233).  Everything is computed once in fp64 numpy and then
uploaded to the device by :mod:`.operator`; tables are bit-identical to the
reference's (tests/test_host_setup.py pins them against the golden
fixtures), so the device sees exactly the reference's constants.

The lat-lon sphere is the north star's geometry; the doubly periodic
planar mesh of the reference's f-plane case (mesh.py:120-132,
basis.py:152-156) runs on the same kernels with cos = 1, sin = 0, R = 1
and wrapped rows.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

LEFT, RIGHT, BOTTOM, TOP = 0, 1, 2, 3
EDGE_NAMES = ("left", "right", "bottom", "top")


@dataclass(frozen=True)
class PhysicalConstants:
    """Williamson-suite Earth parameters (mesh.py:24-36)."""

    radius: float = 6.37122e6
    omega: float = 7.292e-5
    gravity: float = 9.81

    def coriolis(self, theta):
        return 2.0 * self.omega * np.sin(theta)


EARTH = PhysicalConstants()


@dataclass(frozen=True)
class NeighborRef:
    kind: str                 # "interior" | "periodic_wrap" | "pole_closed"
    index: tuple | None = None


@dataclass
class Mesh:
    """Uniform lat-lon element grid: lambda in [0, 2pi] (periodic), theta in
    [-pi/2, pi/2] (pole-closed).  x = longitude, y = latitude."""

    kind: str
    nx: int
    ny: int
    x_edges: np.ndarray
    y_edges: np.ndarray
    radius: float | None = None
    periodic_y: bool = False

    # the spacings are differences of the linspace edges, not 2pi/nx, so
    # every derived constant matches the reference to the last bit
    @property
    def dx(self) -> float:
        return float(self.x_edges[1] - self.x_edges[0])

    @property
    def dy(self) -> float:
        return float(self.y_edges[1] - self.y_edges[0])

    @property
    def determ(self) -> float:
        return self.dx * self.dy / 4.0

    @property
    def bd_det_x(self) -> float:
        return self.dx / 2.0

    @property
    def bd_det_y(self) -> float:
        return self.dy / 2.0

    @property
    def n_elements(self) -> int:
        return self.nx * self.ny

    def element_bounds(self, i: int, j: int):
        return ((float(self.x_edges[i]), float(self.x_edges[i + 1])),
                (float(self.y_edges[j]), float(self.y_edges[j + 1])))

    def neighbor(self, i: int, j: int, edge: int) -> NeighborRef:
        if edge in (LEFT, RIGHT):
            step = -1 if edge == LEFT else 1
            k = i + step
            if 0 <= k < self.nx:
                return NeighborRef("interior", (k, j))
            return NeighborRef("periodic_wrap", (k % self.nx, j))
        if edge in (BOTTOM, TOP):
            step = -1 if edge == BOTTOM else 1
            k = j + step
            if 0 <= k < self.ny:
                return NeighborRef("interior", (i, k))
            if self.periodic_y:
                return NeighborRef("periodic_wrap", (i, k % self.ny))
            return NeighborRef("pole_closed")
        raise ValueError(f"edge must be one of 0..3, got {edge}")


def build_latlon_mesh(nx: int, ny: int, radius: float = EARTH.radius) -> Mesh:
    if nx < 1 or ny < 1:
        raise ValueError("element counts must be at least 1")
    return Mesh("latlon", int(nx), int(ny),
                np.linspace(0.0, 2.0 * math.pi, nx + 1),
                np.linspace(-math.pi / 2.0, math.pi / 2.0, ny + 1),
                float(radius), False)


def build_planar_mesh(nx: int, ny: int, length: float) -> Mesh:
    """Uniform periodic mesh of the square [0, length]^2 (mesh.py:120-132)."""
    if nx < 1 or ny < 1:
        raise ValueError("element counts must be at least 1")
    if length <= 0:
        raise ValueError("domain length must be positive")
    return Mesh("planar", int(nx), int(ny), np.linspace(0.0, length, nx + 1),
                np.linspace(0.0, length, ny + 1), None, True)


def min_effective_diameter(mesh: Mesh) -> float:
    """min over rows of R*dtheta and R*cos(theta_far)*dlambda, the far
    latitude replaced by the near one on pole rows (mesh.py:155-174);
    min(dx, dy) on the plane."""
    if mesh.kind == "planar":
        return min(mesh.dx, mesh.dy)
    R = mesh.radius
    best = math.inf
    for j in range(mesh.ny):
        c0, c1 = math.cos(mesh.y_edges[j]), math.cos(mesh.y_edges[j + 1])
        far = min(c0, c1)
        if far <= 1e-14:
            far = max(c0, c1)
        best = min(best, R * mesh.dy, R * far * mesh.dx)
    return best


# ---------------------------------------------------------------------------
# basis

@dataclass(frozen=True)
class Quadrature:
    n_1d: int
    nodes: np.ndarray
    weights: np.ndarray


def gauss_legendre(n: int) -> Quadrature:
    if n < 1:
        raise ValueError("need at least one quadrature point")
    x, w = np.polynomial.legendre.leggauss(n)
    return Quadrature(n, x, w)


def _legendre_both(j: int, x):
    """(P_j, P_j') by the Bonnet recurrence and P'_{k+1} = P'_{k-1} + (2k+1)P_k."""
    x = np.asarray(x, dtype=np.float64)
    if j == 0:
        return np.ones_like(x), np.zeros_like(x)
    p_prev, p_cur = np.ones_like(x), x.copy()
    d_prev, d_cur = np.zeros_like(x), np.ones_like(x)
    for k in range(1, j):
        p_next = ((2 * k + 1) * x * p_cur - k * p_prev) / (k + 1)
        d_next = d_prev + (2 * k + 1) * p_cur
        p_prev, p_cur, d_prev, d_cur = p_cur, p_next, d_cur, d_next
    return p_cur, d_cur


def legendre_eval(j: int, x):
    return _legendre_both(j, x)[0]


def legendre_deriv(j: int, x):
    return _legendre_both(j, x)[1]


@dataclass(frozen=True)
class Vander:
    """Modal -> nodal matrices; modal index a*(p+1)+b (a: lambda degree),
    node index qi*n+qj (qi: lambda node), edges LEFT, RIGHT, BOTTOM, TOP."""

    p: int
    n_1d: int
    nphi: int
    phi: np.ndarray
    grad_x: np.ndarray
    grad_y: np.ndarray
    edges: tuple
    w: np.ndarray
    w_edge: np.ndarray
    nodes: np.ndarray
    leg: np.ndarray      # (p+1, n): P_a at the 1-d nodes
    dleg: np.ndarray     # (p+1, n): P'_a at the 1-d nodes

    @property
    def n_q(self) -> int:
        return self.phi.shape[0]


def build_vander(p: int, quad: Quadrature) -> Vander:
    n = quad.n_1d
    if n < p + 1:
        raise ValueError(f"quadrature with {n} points cannot resolve degree {p}")
    x = quad.nodes
    pairs = [_legendre_both(a, x) for a in range(p + 1)]
    P = np.stack([pv for pv, _ in pairs])
    D = np.stack([dv for _, dv in pairs])
    at_m1 = np.array([legendre_eval(a, -1.0) for a in range(p + 1)]).reshape(p + 1)
    at_p1 = np.array([legendre_eval(a, 1.0) for a in range(p + 1)]).reshape(p + 1)
    # tensor products, one rounding each: row q=(qi,qj), column m=(a,b)
    Pa, Pb = P[:, None, :, None], P[None, :, None, :]
    Da, Db = D[:, None, :, None], D[None, :, None, :]

    def mat(t):   # t indexed [a, b, qi, qj] -> [q, m]
        return np.ascontiguousarray(t.transpose(2, 3, 0, 1).reshape(n * n, (p + 1) ** 2))

    phi = mat(Pa * Pb)
    gx = mat(Da * Pb)
    gy = mat(Pa * Db)
    # edge traces: [k, (a, b)]
    eL = (at_m1[:, None, None] * P[None, :, :]).transpose(2, 0, 1).reshape(n, -1)
    eR = (at_p1[:, None, None] * P[None, :, :]).transpose(2, 0, 1).reshape(n, -1)
    eB = (P[:, None, :] * at_m1[None, :, None]).transpose(2, 0, 1).reshape(n, -1)
    eT = (P[:, None, :] * at_p1[None, :, None]).transpose(2, 0, 1).reshape(n, -1)
    edges = tuple(np.ascontiguousarray(e) for e in (eL, eR, eB, eT))
    return Vander(p=p, n_1d=n, nphi=(p + 1) ** 2, phi=phi, grad_x=gx, grad_y=gy,
                  edges=edges, w=np.outer(quad.weights, quad.weights).reshape(-1),
                  w_edge=quad.weights.copy(), nodes=x.copy(), leg=P, dleg=D)


@dataclass(frozen=True)
class MassMatrix:
    M: np.ndarray
    Minv: np.ndarray


def mass_matrix_sphere(p: int, theta_bounds, quad: Quadrature, dlam: float) -> MassMatrix:
    """M_ij = int phi_i phi_j cos(theta) over one element of a latitude row
    (basis.py:159-176): symmetrised, Cholesky-checked, inverted by LAPACK."""
    lo, hi = theta_bounds
    phi = build_vander(p, quad).phi
    cosw = np.cos(0.5 * (lo + hi) + 0.5 * (hi - lo) * quad.nodes)
    weighted = np.outer(quad.weights, quad.weights * cosw).reshape(-1)
    scale = dlam * (hi - lo) / 4.0
    M = scale * (phi.T * weighted) @ phi
    M = 0.5 * (M + M.T)
    np.linalg.cholesky(M)
    return MassMatrix(M, np.linalg.inv(M))


def mass_matrix_planar(p: int, determ: float) -> MassMatrix:
    """Diagonal mass matrix of the orthogonal tensor Legendre basis
    (basis.py:152-156)."""
    norms = np.array([2.0 / (2 * a + 1) for a in range(p + 1)])
    diag = determ * np.outer(norms, norms).reshape(-1)
    return MassMatrix(np.diag(diag), np.diag(1.0 / diag))


def row_mass_matrices(p: int, mesh: Mesh, quad: Quadrature):
    """(ny, nphi, nphi) mass matrices and inverses of every row: the
    cos-weighted ones on the sphere, the planar diagonal one repeated."""
    if mesh.kind == "planar":
        m = mass_matrix_planar(p, mesh.determ)
        return np.stack([m.M] * mesh.ny), np.stack([m.Minv] * mesh.ny)
    return sphere_row_mass_matrices(p, mesh, quad)


def sphere_row_mass_matrices(p: int, mesh: Mesh, quad: Quadrature):
    """(ny, nphi, nphi) mass matrices and inverses, one per latitude row."""
    out = [mass_matrix_sphere(p, (mesh.y_edges[j], mesh.y_edges[j + 1]), quad, mesh.dx)
           for j in range(mesh.ny)]
    return np.stack([m.M for m in out]), np.stack([m.Minv for m in out])


def element_node_coords(mesh: Mesh, nodes: np.ndarray):
    """lambda (nx, n) and theta (ny, n) of the 1-d nodes of every element."""
    half = 0.5 * mesh.dx
    lam = mesh.x_edges[:-1][:, None] + half * (1.0 + nodes)[None, :]
    half = 0.5 * mesh.dy
    th = mesh.y_edges[:-1][:, None] + half * (1.0 + nodes)[None, :]
    return lam, th


def project_initial(f, mesh: Mesh, vander: Vander) -> np.ndarray:
    """cos-weighted L2 projection of f(lambda, theta): (nx, ny, nphi); on
    the plane the unweighted one against the diagonal mass (basis.py:206-233)."""
    n = vander.n_1d
    lam, th = element_node_coords(mesh, vander.nodes)
    vals = np.broadcast_to(f(lam[:, None, :, None], th[None, :, None, :]),
                           (mesh.nx, mesh.ny, n, n)).reshape(mesh.nx, mesh.ny, n * n)
    w2 = np.outer(vander.w_edge, vander.w_edge).reshape(-1)
    if mesh.kind == "planar":
        rhs = mesh.determ * np.einsum("xyq,q,qm->xym", vals, w2, vander.phi)
        mm = mass_matrix_planar(vander.p, mesh.determ)
        return np.ascontiguousarray(rhs * (1.0 / np.diag(mm.M))[None, None, :])
    w_rows = (w2.reshape(n, n)[None, :, :] * np.cos(th)[:, None, :]).reshape(mesh.ny, n * n)
    moments = mesh.determ * np.einsum("xyq,yq,qm->xym", vals, w_rows, vander.phi)
    _, Minv = sphere_row_mass_matrices(vander.p, mesh, gauss_legendre(n))
    return np.ascontiguousarray(np.einsum("ymn,xyn->xym", Minv, moments))


def eval_modal_at_nodes(coeffs: np.ndarray, eval_matrix: np.ndarray) -> np.ndarray:
    return np.einsum("qm,...m->...q", eval_matrix, coeffs)


def node_latitudes(mesh: Mesh, nodes: np.ndarray) -> np.ndarray:
    """(ny, n) latitude of the 1-d nodes of each row, as the operator's
    coordinate tables form it: y_lo + (dy/2)(1+x) (dg.py:264-268)."""
    return mesh.y_edges[:-1][:, None] + 0.5 * mesh.dy * (1.0 + nodes)[None, :]
