"""Spherical shallow-water model description (host side).

The pointwise flux / source / wavespeed arithmetic of the hot path runs
inside the fused CUDA stage kernel (csrc/dgswe_kernels.cuh); this module
keeps the reference's model object API (``swe_sphere_model``,
``PositivityError``, ``max_physical_speed``; /root/reference/pkg/src/dgswe/
models.py:43-46, 149-170, 213-295) for step-size control and for callers
that inspect the model.

Flux-form SWE in lat-lon coordinates, conserved (h, hu, hv):
    F = (1/R) (hu, hu u + g h^2/2, hu v)
    G = (cos/R) (hv, hu v, hv v + g h^2/2)
    S = (0, t hv, -(g h^2/2) sin/R - t hu),  t = u sin/R + 2 Omega sin cos

Extension (not in the reference, whose SPEC.md:157 lists orography as a
non-goal): an optional bottom topography b(lambda, theta) adds the momentum
sources -(g h / R) db/dlambda and -(g h cos / R) db/dtheta -- the
cos-weighted form of -g h grad b -- for Williamson test case 5.  h is the
fluid depth; the free surface is h + b.
"""

from __future__ import annotations

import numpy as np

from .geometry import PhysicalConstants

X_DIR, Y_DIR = 0, 1


class PositivityError(RuntimeError):
    """Water height reached zero or below at a quadrature point."""


class SphereSWEModel:
    n_vars = 3
    var_names = ("h", "hu", "hv")
    has_source = True
    is_spherical = True

    def __init__(self, constants: PhysicalConstants, h_ref: float = 1.0, bottom=None):
        if constants.gravity <= 0:
            raise ValueError("gravity must be positive")
        self.constants = constants
        self.gravity = float(constants.gravity)
        self.h_floor = 1e-8 * float(h_ref)
        self.bottom = bottom          # None, or b(lambda, theta) in metres (numpy)

    def _floor_and_celerity(self, U):
        h = U["h"]
        return np.maximum(h, self.h_floor), np.sqrt(self.gravity * np.maximum(h, 0.0))

    def wavespeed_nodes(self, U, coords, direction):
        """Coordinate speeds d(lambda)/dt or d(theta)/dt."""
        R = self.constants.radius
        hf, c = self._floor_and_celerity(U)
        if direction == X_DIR:
            cos = np.maximum(np.cos(coords.theta), 1e-14)
            return (np.abs(U["hu"] / hf) + c) / (R * cos)
        return (np.abs(U["hv"] / hf) + c) / R

    def alpha_nodes(self, U, coords, direction):
        """Directional flux-Jacobian spectral radius (Rusanov bound)."""
        R = self.constants.radius
        hf, c = self._floor_and_celerity(U)
        if direction == X_DIR:
            return (np.abs(U["hu"] / hf) + c) / R
        return np.cos(coords.theta) * (np.abs(U["hv"] / hf) + c) / R

    def max_wavespeed(self, U, coords, direction) -> float:
        return float(np.max(self.wavespeed_nodes(U, coords, direction)))

    def max_physical_speed(self, U, coords=None) -> float:
        hf, c = self._floor_and_celerity(U)
        vel = np.maximum(np.abs(U["hu"] / hf), np.abs(U["hv"] / hf))
        return float(np.max(vel + c))


def swe_sphere_model(constants: PhysicalConstants, h_ref: float = 1.0, bottom=None) -> SphereSWEModel:
    """models.py:293-295; ``bottom`` (extension) is the orography b(lambda, theta)."""
    return SphereSWEModel(constants, h_ref, bottom)


class PlanarSWEModel:
    """Shallow water on the doubly periodic plane with an f-plane Coriolis
    source (models.py:176-227): the lat-lon operator with cos = 1, sin = 0
    and R = 1 -- the row tables the kernels read carry exactly that
    (operator.py) -- and rows that wrap instead of poles."""

    n_vars = 3
    var_names = ("h", "hu", "hv")
    has_source = True
    is_spherical = False
    bottom = None

    def __init__(self, gravity: float, coriolis_f: float, h_ref: float = 1.0):
        if gravity <= 0:
            raise ValueError("gravity must be positive")
        self.gravity = float(gravity)
        self.coriolis_f = float(coriolis_f)
        self.h_floor = 1e-8 * float(h_ref)

    def wavespeed_nodes(self, U, coords, direction):
        h = U["h"]
        mom = U["hu"] if direction == X_DIR else U["hv"]
        vel = mom / np.maximum(h, self.h_floor)
        return np.abs(vel) + np.sqrt(self.gravity * np.maximum(h, 0.0))

    def alpha_nodes(self, U, coords, direction):
        return self.wavespeed_nodes(U, coords, direction)

    def max_wavespeed(self, U, coords, direction) -> float:
        return float(np.max(self.wavespeed_nodes(U, coords, direction)))

    def max_physical_speed(self, U, coords=None) -> float:
        return max(self.max_wavespeed(U, coords, X_DIR), self.max_wavespeed(U, coords, Y_DIR))


def swe_planar_model(gravity: float, coriolis_f: float, h_ref: float = 1.0) -> PlanarSWEModel:
    """Planar shallow water with constant Coriolis parameter f (models.py:288-290)."""
    return PlanarSWEModel(gravity, coriolis_f, h_ref)
