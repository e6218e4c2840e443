"""Print GPU-vs-oracle error statistics for every golden case.

    python tools/parity_report.py            (on a GPU box)

For each case: one RHS (per-variable relative L2 error and error relative to
max|k|), N Butcher steps through rk_step, and N fused SSPRK3 steps.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
import paper_2303_11767_b200 as P  # noqa: E402


def rel(a, b):
    return [float(np.linalg.norm(a[v] - b[v]) / max(np.linalg.norm(b[v]), 1e-300)) for v in range(3)]


def main():
    meta = json.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))
    only = sys.argv[1:] or None
    for name, e in meta["cases"].items():
        if only and name not in only:
            continue
        t, orc, X = O.build_case(e["case"], e["nx"], e["ny"], e["p"], e["nz"], *e["rusanov"])
        if e["nz"] == 2:
            X[0, :, :, 1, 0] += 25.0
            X[0, :, :, 1, 1:] *= 0.9
            X[1, :, :, 1, :] *= 1.1
        cfg = P.default_config(e["case"]).override(nx=e["nx"], ny=e["ny"], p=e["p"], nz=e["nz"])
        setup = P.build_case(cfg)
        op = P.SpatialOperator(setup.mesh, e["p"], setup.model,
                               rusanov=P.RusanovParams(*e["rusanov"]), nz=e["nz"])
        st = op.state_from_array(X)
        k = op.assemble_rhs(st).to_numpy()
        kr = orc.rhs(X)
        r_rhs = rel(k, kr)
        nst = e["nsteps"]
        U, stc, _ = orc.rk_steps(X, e["dt"], e["rk"], nst)
        s2 = op.state_from_array(X)
        tab = P.tableau(e["rk"])
        for _ in range(nst):
            P.rk_step(s2, op.assemble_rhs, e["dt"], tab)
        r_but = rel(s2.to_numpy(), U)
        line = f"{name:18s} rhs {max(r_rhs):.2e} {['%.1e' % x for x in r_rhs]} butcher {max(r_but):.2e}"
        if e["rk"] == 3:
            s3 = op.state_from_array(X)
            op.ssprk3_steps(s3, e["dt"], nst)
            flags, _ = op.status()
            r_f = rel(s3.to_numpy(), U)
            nrm = np.linalg.norm(U[2]) / np.linalg.norm(U[1:3])
            line += f" fused {max(r_f):.2e} {['%.1e' % x for x in r_f]} flags {flags} |hv|/|m| {nrm:.1e}"
        print(line, flush=True)


if __name__ == "__main__":
    torch.cuda.set_device(0)
    main()
