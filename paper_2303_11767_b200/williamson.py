"""Williamson shallow-water test cases and run configurations.

API of /root/reference/pkg/src/dgswe/cases.py (``CaseConfig``,
``default_config``, ``build_case``, ``RunSetup``, ``ic_williamson_tc2``,
``ic_williamson_tc6``) for the two spherical cases of the reference.
Williamson et al. (1992) equations: TC2 (90)-(95) with alpha = 0,
TC6 (142)-(149).  The planar f-plane case (geostrophic adjustment,
cases.py:113-123) runs on the same kernels (y-periodic plane); the scalar
advection case (a one-variable model, cases.py:99-110) runs on its own
stage kernel (advection.py, csrc/dgswe_adv.cuh).
Williamson TC5 (flow over an isolated mountain) is an extension: the
reference has no orography; its bottom topography enters the
model's momentum sources (physics.py) and the oracle restates the same
discretisation (parity unpinned against the reference).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, replace

import numpy as np

from .geometry import EARTH, PhysicalConstants, build_latlon_mesh, build_planar_mesh
from .physics import swe_planar_model, swe_sphere_model

DAY = 86400.0
TC2_U0 = 2.0 * math.pi * EARTH.radius / (12.0 * DAY)
TC2_GH0 = 2.94e4
# geostrophic adjustment on the f-plane (cases.py:58-63)
ADJ_LENGTH = 1.0e7          # m
ADJ_H0 = 1000.0             # m
ADJ_H1 = 5.0                # m
ADJ_SIGMA = ADJ_LENGTH / 20.0
ADJ_F = 1.0e-4              # s^-1

TC6_OMEGA = 7.848e-6
TC6_K = 7.848e-6
TC6_H0 = 8.0e3
TC6_R = 4
# test case 5 (zonal flow over an isolated mountain), Williamson et al. (1992)
# section 3.5 -- EXTENSION: the reference has no orography
TC5_U0 = 20.0
TC5_H0 = 5960.0
TC5_HS0 = 2000.0
TC5_RM = math.pi / 9.0
TC5_LC = 1.5 * math.pi        # lambda_c = -pi/2 on [0, 2 pi)
TC5_TC = math.pi / 6.0

def _xp(*arrays):
    """numpy, or torch when the coordinates are torch tensors (the device
    initial-condition projection evaluates these functions on the GPU)."""
    for a in arrays:
        if type(a).__module__.startswith("torch"):
            import torch
            return torch
    return np


def _zeros(lam, th):
    xp = _xp(lam, th)
    if xp is np:
        return np.zeros(np.broadcast(lam, th).shape)
    return xp.zeros(xp.broadcast_shapes(lam.shape, th.shape), dtype=xp.float64, device=lam.device)


CASE_IDS = ("advection_sine", "geostrophic_adjustment", "williamson_tc2", "williamson_tc6",
            "williamson_tc5")
SPHERE_CASES = ("williamson_tc2", "williamson_tc6", "williamson_tc5")


@dataclass(frozen=True)
class CaseConfig:
    case: str
    nx: int
    ny: int
    p: int
    rk: int
    t_final: float
    dt: float | None = None
    courant: float | None = None
    nz: int = 1
    alpha_mode: str = "local"
    alpha: float | None = None

    def override(self, **kwargs) -> "CaseConfig":
        return replace(self, **{k: v for k, v in kwargs.items() if v is not None})


_DEFAULTS = {
    "advection_sine": dict(nx=20, ny=20, p=2, rk=4, t_final=1.0, courant=0.2),
    "geostrophic_adjustment": dict(nx=50, ny=50, p=3, rk=4, t_final=36000.0, dt=100.0),
    "williamson_tc2": dict(nx=20, ny=20, p=3, rk=4, t_final=2.0 * DAY, courant=0.2),
    "williamson_tc6": dict(nx=40, ny=20, p=3, rk=4, t_final=8.0 * DAY, dt=4.0),
    "williamson_tc5": dict(nx=40, ny=20, p=4, rk=3, t_final=15.0 * DAY, dt=2.0),
}


def default_config(case: str) -> CaseConfig:
    if case not in _DEFAULTS:
        raise ValueError(f"unknown case {case!r}; choose from {CASE_IDS}")
    return CaseConfig(case=case, **_DEFAULTS[case])


def ic_williamson_tc2(constants: PhysicalConstants = EARTH):
    """Steady zonal geostrophic flow: u = u0 cos(theta), v = 0,
    g h = g h0 - (R Omega u0 + u0^2/2) sin^2(theta)."""
    g = constants.gravity
    u0 = TC2_U0
    k = constants.radius * constants.omega * u0 + 0.5 * u0 * u0

    def height(lam, th):
        return (TC2_GH0 - k * _xp(th).sin(th) ** 2) / g + 0.0 * lam

    return ({"h": height,
             "hu": lambda lam, th: height(lam, th) * u0 * _xp(th).cos(th),
             "hv": _zeros},
            height)


def tc6_fields(constants: PhysicalConstants = EARTH):
    """Wavenumber-4 Rossby-Haurwitz height and winds."""
    a, g, Om = constants.radius, constants.gravity, constants.omega
    w, K, R = TC6_OMEGA, TC6_K, TC6_R

    def winds(lam, th):
        xp = _xp(lam, th)
        c = xp.cos(th)
        u = a * w * c + a * K * c ** (R - 1) * (R * xp.sin(th) ** 2 - c**2) * xp.cos(R * lam)
        v = -a * K * R * c ** (R - 1) * xp.sin(th) * xp.sin(R * lam)
        return u, v

    def height(lam, th):
        xp = _xp(lam, th)
        c = xp.cos(th)
        A = 0.5 * w * (2.0 * Om + w) * c**2 + 0.25 * K**2 * c ** (2 * R) * (
            (R + 1) * c**2 + (2 * R**2 - R - 2) - 2.0 * R**2 * c ** (-2))
        B = (2.0 * (Om + w) * K) / ((R + 1) * (R + 2)) * c**R * (
            (R**2 + 2 * R + 2) - (R + 1) ** 2 * c**2)
        C = 0.25 * K**2 * c ** (2 * R) * ((R + 1) * c**2 - (R + 2))
        return TC6_H0 + (a * a / g) * (A + B * xp.cos(R * lam) + C * xp.cos(2 * R * lam))

    return height, winds


def tc5_bottom(lam, th):
    """Isolated conical mountain: b = hs0 (1 - r/R_m), r = min(R_m, dist to
    (lambda_c, theta_c)) in the (lambda, theta) plane (Williamson eq. 134)."""
    xp = _xp(lam, th)
    d = xp.sqrt((lam - TC5_LC) ** 2 + (th - TC5_TC) ** 2)
    r = xp.minimum(d, xp.full_like(d, TC5_RM) if xp is not np else TC5_RM)
    return TC5_HS0 * (1.0 - r / TC5_RM)


def ic_williamson_tc5(constants: PhysicalConstants = EARTH):
    """TC2-like balanced zonal flow (u0 = 20 m/s, h0 = 5960 m) over the
    mountain: depth h = h0 - (R Omega u0 + u0^2/2) sin^2(theta)/g - b."""
    g = constants.gravity
    k = constants.radius * constants.omega * TC5_U0 + 0.5 * TC5_U0 * TC5_U0

    def depth(lam, th):
        return (g * TC5_H0 - k * _xp(th).sin(th) ** 2) / g - tc5_bottom(lam, th)

    return {"h": depth,
            "hu": lambda lam, th: depth(lam, th) * TC5_U0 * _xp(th).cos(th),
            "hv": _zeros}


def ic_williamson_tc6(constants: PhysicalConstants = EARTH):
    height, winds = tc6_fields(constants)
    return {"h": height,
            "hu": lambda lam, th: height(lam, th) * winds(lam, th)[0],
            "hv": lambda lam, th: height(lam, th) * winds(lam, th)[1]}


@dataclass
class RunSetup:
    config: CaseConfig
    mesh: object
    model: object
    ic: dict
    exact: object = None
    constants: PhysicalConstants = EARTH


ADV_BETA = (1.0, 1.0)


def ic_advection_sine():
    """sin(2 pi x) sin(2 pi y) on the periodic unit square; the exact
    solution is the profile translated by beta t (cases.py:99-110)."""
    beta = ADV_BETA

    def u0(x, y):
        return np.sin(2.0 * math.pi * x) * np.sin(2.0 * math.pi * y)

    def exact(t):
        return lambda x, y: u0(np.mod(x - beta[0] * t, 1.0), np.mod(y - beta[1] * t, 1.0))

    return {"u": u0}, beta, exact


def ic_geostrophic_adjustment():
    """Gaussian height bump at rest on the f-plane (cases.py:113-123)."""

    def h0(x, y):
        r2 = (x - ADJ_LENGTH / 2) ** 2 + (y - ADJ_LENGTH / 2) ** 2
        return ADJ_H0 + ADJ_H1 * np.exp(-r2 / (2.0 * ADJ_SIGMA ** 2))

    zero = lambda x, y: np.zeros(np.broadcast(x, y).shape)   # noqa: E731
    return {"h": h0, "hu": zero, "hv": zero}


def build_case(config: CaseConfig, constants: PhysicalConstants = EARTH) -> RunSetup:
    case = config.case
    if case == "williamson_tc2":
        ic, height = ic_williamson_tc2(constants)
        setup = RunSetup(config, build_latlon_mesh(config.nx, config.ny, constants.radius),
                         swe_sphere_model(constants, h_ref=TC2_GH0 / constants.gravity), ic,
                         None, constants)
        setup.exact = lambda t: height
        return setup
    if case == "williamson_tc6":
        return RunSetup(config, build_latlon_mesh(config.nx, config.ny, constants.radius),
                        swe_sphere_model(constants, h_ref=TC6_H0), ic_williamson_tc6(constants),
                        None, constants)
    if case == "williamson_tc5":
        model = swe_sphere_model(constants, h_ref=TC5_H0, bottom=tc5_bottom)
        return RunSetup(config, build_latlon_mesh(config.nx, config.ny, constants.radius), model,
                        ic_williamson_tc5(constants), None, constants)
    if case == "geostrophic_adjustment":
        model = swe_planar_model(constants.gravity, ADJ_F, h_ref=ADJ_H0)
        return RunSetup(config, build_planar_mesh(config.nx, config.ny, ADJ_LENGTH), model,
                        ic_geostrophic_adjustment(), None, constants)
    if case == "advection_sine":
        from .advection import advection_model
        ic, beta, exact = ic_advection_sine()
        return RunSetup(config, build_planar_mesh(config.nx, config.ny, 1.0), advection_model(beta),
                        ic, exact, constants)
    raise ValueError(f"unknown case {case!r}; choose from {CASE_IDS}")
