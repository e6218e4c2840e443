"""The reference's f-plane case (geostrophic adjustment on the doubly
periodic plane, cases.py:113-123, mesh.py:120-132, models.py:176-227): host
setup bit-identical to the unmodified reference (tests/golden/planar.npz,
made by tests/golden/make_planar_golden.py)."""

import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "planar.npz")


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLDEN)


def _names(gold):
    return sorted({k.split("/")[0] for k in gold.files})


def test_planar_projection_bit_identical(gold):
    import paper_2303_11767_b200 as P
    for name in _names(gold):
        nx, ny, p, dt, nsteps = gold[f"{name}/meta"]
        setup = P.build_case(P.default_config("geostrophic_adjustment").override(nx=int(nx), ny=int(ny), p=int(p)))
        vander = P.build_vander(int(p), P.gauss_legendre(int(p) + 1))
        x0 = np.stack([P.project_initial(setup.ic[v], setup.mesh, vander) for v in ("h", "hu", "hv")])
        assert np.array_equal(x0[:, :, :, None, :], gold[f"{name}/x0"]), name


def test_planar_mesh_and_model():
    import paper_2303_11767_b200 as P
    m = P.build_planar_mesh(10, 8, 1.0e7)
    assert m.kind == "planar" and m.periodic_y and m.dx == 1.0e6 and m.dy == 1.25e6
    assert P.min_effective_diameter(m) == 1.0e6
    assert m.neighbor(3, 7, P.TOP).index == (3, 0) and m.neighbor(3, 0, P.BOTTOM).index == (3, 7)
    mm = P.mass_matrix_planar(2, m.determ)
    assert np.allclose(np.diag(mm.M) * np.diag(mm.Minv), 1.0)
    model = P.swe_planar_model(9.81, 1e-4, h_ref=1000.0)
    assert not model.is_spherical and model.h_floor == 1e-5
    setup = P.build_case(P.default_config("advection_sine"))
    assert setup.model.beta == (1.0, 1.0) and setup.mesh.kind == "planar" and setup.mesh.dx == 0.05


ADV_GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "advection.npz")


def test_advection_projection_bit_identical():
    """advection_sine on the unit square (cases.py:99-110): mesh, model and
    the host L2 projection bit-identical to the reference's fixtures."""
    import paper_2303_11767_b200 as P
    gold = np.load(ADV_GOLDEN)
    for name in _names(gold):
        nx, ny, p = (int(v) for v in gold[f"{name}/meta"][:3])
        setup = P.build_case(P.default_config("advection_sine").override(nx=nx, ny=ny, p=p))
        assert setup.mesh.dx == 1.0 / nx and setup.model.max_physical_speed() == 1.0
        vander = P.build_vander(p, P.gauss_legendre(p + 1))
        x0 = P.project_initial(setup.ic["u"], setup.mesh, vander)
        assert np.array_equal(x0[None, :, :, None, :], gold[f"{name}/x0"]), name
        # the exact solution is the initial profile translated by beta t (period 1)
        assert np.allclose(setup.exact(1.0)(0.3, 0.7), setup.ic["u"](0.3, 0.7))


def test_advection_model_and_operator_guard():
    import torch
    import paper_2303_11767_b200 as P
    with pytest.raises(ValueError):
        P.advection_model((1.0, float("nan")))
    m = P.advection_model((2.0, -3.0))
    assert m.max_physical_speed() == 3.0 and m.n_vars == 1
    assert np.all(m.wavespeed_nodes({"u": np.zeros(4)}, None, 1) == 3.0)
    if not torch.cuda.is_available():
        with pytest.raises(RuntimeError):                       # no CPU fallback
            P.AdvectionOperator(P.build_planar_mesh(4, 4, 1.0), 1, m)


def test_advection_l2_error_matches_reference():
    """The planar L2 error (no cos metric) of the reference's own integrated
    state, in the reference's reduction order: bit-identical to its value."""
    import types
    import paper_2303_11767_b200 as P
    gold = np.load(ADV_GOLDEN)
    for name in _names(gold):
        nx, ny, p = (int(v) for v in gold[f"{name}/meta"][:3])
        setup = P.build_case(P.default_config("advection_sine").override(nx=nx, ny=ny, p=p))
        xT = gold[f"{name}/xT"][0]
        st = types.SimpleNamespace(names=("u",), interior_coeffs=lambda v, xT=xT: xT)
        op = types.SimpleNamespace(mesh=setup.mesh, p=p)
        err, err_rel = gold[f"{name}/errT"]
        assert P.l2_error_host(st, setup.exact(0.05), op) == err, name
        assert P.l2_error_host(st, setup.exact(0.05), op, relative=True) == err_rel, name
