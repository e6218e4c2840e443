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
    with pytest.raises(NotImplementedError):
        P.build_case(P.default_config("advection_sine"))
