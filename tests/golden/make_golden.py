"""Generate the golden fixtures from the UNMODIFIED reference package.

Run once in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

It imports ``dgswe`` from /root/reference/pkg/src read-only and writes

* ``tests/golden/golden.npz``  -- full arrays for the small cases
  (setup tables, initial coefficients, one RHS, states after N steps);
* ``tests/golden/golden.json`` -- case metadata, SHA-256 pins (first 16 hex
  of sha256 over h||hu||hv interior coefficient bytes), mass integrals and
  TC2 L2 errors, including cases too large to store in full.

Nothing here is imported by the product, the GPU tests read only the files
this script produced.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_dgswe")
sys.path.insert(0, REF)

from dgswe import basis, cases, dg, diagnostics, timestep  # noqa: E402


def coeffs_of(st):
    """(3, nx, ny, nz, nphi) stack of interior coefficients."""
    return np.stack([np.ascontiguousarray(st.interior_coeffs(n)) for n in st.names])


def sha16(st):
    h = hashlib.sha256()
    for n in st.names:
        h.update(np.ascontiguousarray(st.interior_coeffs(n)).tobytes())
    return h.hexdigest()[:16]


# name, case, nx, ny, p, nz, rk, dt, nsteps, rusanov(mode, alpha), store_full
CASES = [
    ("tc2_c1", "williamson_tc2", 40, 20, 2, 1, 3, 10.0, 100, ("local", None), True),
    ("tc6_40x20_p3", "williamson_tc6", 40, 20, 3, 1, 3, 4.0, 100, ("local", None), False),
    ("tc2_40x20_p3", "williamson_tc2", 40, 20, 3, 1, 3, 4.0, 100, ("local", None), False),
    ("tc6_p0", "williamson_tc6", 12, 6, 0, 1, 3, 60.0, 10, ("local", None), True),
    ("tc6_p1", "williamson_tc6", 12, 6, 1, 1, 3, 30.0, 10, ("local", None), True),
    ("tc6_p2", "williamson_tc6", 12, 6, 2, 1, 3, 20.0, 10, ("local", None), True),
    ("tc6_p3", "williamson_tc6", 12, 6, 3, 1, 3, 10.0, 10, ("local", None), True),
    ("tc6_p4", "williamson_tc6", 12, 6, 4, 1, 3, 6.0, 10, ("local", None), True),
    ("tc6_p5", "williamson_tc6", 12, 6, 5, 1, 3, 4.0, 10, ("local", None), True),
    ("tc2_p3_odd", "williamson_tc2", 35, 7, 3, 1, 3, 10.0, 10, ("local", None), True),
    ("tc6_rk1", "williamson_tc6", 10, 6, 2, 1, 1, 5.0, 10, ("local", None), True),
    ("tc6_rk2", "williamson_tc6", 10, 6, 2, 1, 2, 10.0, 10, ("local", None), True),
    ("tc6_rk4", "williamson_tc6", 10, 6, 2, 1, 4, 20.0, 10, ("local", None), True),
    ("tc6_ny1", "williamson_tc6", 8, 1, 2, 1, 3, 20.0, 5, ("local", None), True),
    ("tc2_nx1", "williamson_tc2", 1, 6, 2, 1, 3, 5.0, 5, ("local", None), True),
    ("tc6_nx2", "williamson_tc6", 2, 4, 3, 1, 3, 5.0, 5, ("local", None), True),
    ("tc6_global_pinned", "williamson_tc6", 12, 6, 2, 1, 3, 20.0, 5, ("global", 1.0e-4), True),
    ("tc6_global", "williamson_tc6", 12, 6, 2, 1, 3, 20.0, 5, ("global", None), True),
    ("tc6_nz2", "williamson_tc6", 12, 6, 2, 2, 3, 20.0, 5, ("local", None), True),
    ("tc6_wide", "williamson_tc6", 70, 8, 3, 1, 3, 2.0, 5, ("local", None), True),
    ("tc2_c2_shape", "williamson_tc2", 360, 180, 3, 1, 3, 0.05, 3, ("local", None), False),
    # BASELINE.json configs at full size (SHA / mass / L2 pins only; `--only` regenerates these
    # without rerunning the small cases): C2 100 steps, C3 20 steps, C4 shape 3 steps
    ("c2_full", "williamson_tc2", 360, 180, 3, 1, 3, 0.05, 100, ("local", None), False),
    ("c3_full", "williamson_tc6", 720, 360, 3, 1, 3, 5e-3, 20, ("local", None), False),
    ("c4_full", "williamson_tc6", 1440, 720, 4, 1, 3, 5e-4, 3, ("local", None), False),
]

TABLE_SHAPES = [(6, 4, 0), (8, 5, 1), (10, 6, 2), (12, 6, 3), (8, 4, 4), (6, 4, 5), (20, 10, 3)]


def build(case, nx, ny, p, nz, rus):
    cfg = cases.default_config(case).override(nx=nx, ny=ny, p=p, nz=nz)
    setup = cases.build_case(cfg)
    op = dg.SpatialOperator(setup.mesh, p, setup.model,
                            rusanov=dg.RusanovParams(*rus), nz=nz)
    return setup, op


def initial_state(setup, op, nz, name):
    st = op.project_state(setup.ic)
    if nz == 2:
        # second level: same flow with a perturbed mean height (keeps h > 0)
        c = st.fields["h"].data
        c[1:-1, 1:-1, 1, 0] += 25.0
        c[1:-1, 1:-1, 1, 1:] *= 0.9
        st.fields["hu"].data[1:-1, 1:-1, 1, :] *= 1.1
    return st


def main():
    only = None
    if "--only" in sys.argv:
        only = set(sys.argv[sys.argv.index("--only") + 1].split(","))
    arrays = {}
    meta = {"reference": REF, "numpy": np.__version__, "cases": {}, "tables": []}
    if only is not None:
        # merge into the existing fixtures: the npz is left untouched (no full arrays)
        meta = json.load(open(os.path.join(HERE, "golden.json")))
    try:
        import numba
        meta["numba"] = numba.__version__
    except ImportError:  # pragma: no cover
        meta["numba"] = None

    for (nx, ny, p) in (TABLE_SHAPES if only is None else ()):
        setup, op = build("williamson_tc6", nx, ny, p, 1, ("local", None))
        tag = f"tab_{nx}x{ny}_p{p}"
        meta["tables"].append(tag)
        v = op.vander
        arrays[f"{tag}/nodes"] = op.quad.nodes
        arrays[f"{tag}/weights"] = op.quad.weights
        arrays[f"{tag}/phi"] = v.phi
        arrays[f"{tag}/grad_x"] = v.grad_x
        arrays[f"{tag}/grad_y"] = v.grad_y
        for e in range(4):
            arrays[f"{tag}/edge{e}"] = v.edges[e]
            arrays[f"{tag}/bnd{e}"] = op.bnd_f[e].data[0, 0, 0]
        arrays[f"{tag}/volx"] = op.volx_f.data[0, 0, 0]
        arrays[f"{tag}/voly"] = op.voly_f.data[0, 0, 0]
        arrays[f"{tag}/src"] = op.src_f.data[0, 0, 0]
        arrays[f"{tag}/M_rows"] = op.M_rows
        arrays[f"{tag}/Minv"] = op.minv_f.data[0, 1:ny + 1, 0]
        for cname in ("coords_int", "coords_xe", "coords_yb", "coords_yt"):
            c = getattr(op, cname)
            for fld in ("cos_over_r", "sin_over_r", "f_cos"):
                arrays[f"{tag}/{cname}.{fld}"] = getattr(c, fld).data[0, :, 0]

    for (name, case, nx, ny, p, nz, rk, dt, nsteps, rus, full) in CASES:
        if only is not None and name not in only:
            continue
        if only is not None and full:
            raise SystemExit(f"{name} stores full arrays: regenerate everything instead")
        t0 = time.time()
        setup, op = build(case, nx, ny, p, nz, rus)
        st = initial_state(setup, op, nz, name)
        entry = {
            "case": case, "nx": nx, "ny": ny, "p": p, "nz": nz, "rk": rk,
            "dt": dt, "nsteps": nsteps, "rusanov": list(rus),
            "h_floor": op.model.h_floor,
            "sha_ic": sha16(st),
            "mass_ic": [diagnostics.mass_integral(st, op, "h", level=k) for k in range(nz)],
        }
        if full:
            arrays[f"{name}/ic"] = coeffs_of(st)
        k = op.assemble_rhs(st.copy())
        entry["sha_rhs"] = sha16(k)
        if full:
            arrays[f"{name}/rhs"] = coeffs_of(k)
        tab = timestep.tableau(rk)
        ws = timestep._RKWorkspace(st, tab.s)
        for _ in range(nsteps):
            timestep.rk_step(st, op.assemble_rhs, dt, tab, ws)
        entry["sha_final"] = sha16(st)
        entry["mass_final"] = [diagnostics.mass_integral(st, op, "h", level=k) for k in range(nz)]
        if case == "williamson_tc2":
            entry["l2_h_rel_final"] = diagnostics.l2_error(
                st, setup.exact(dt * nsteps), op, "h", relative=True)
        if full:
            arrays[f"{name}/final"] = coeffs_of(st)
        entry["seconds"] = round(time.time() - t0, 2)
        meta["cases"][name] = entry
        print(name, entry["sha_ic"], entry["sha_rhs"], entry["sha_final"], entry["seconds"], "s",
              flush=True)

    if only is None:
        np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
