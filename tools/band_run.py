"""Multi-rank latitude-band SSPRK3 run (used by tests/test_gpu_parity.py).

    torchrun --nproc-per-node N tools/band_run.py --transport host --out x.npy

Every rank owns a band of TC6 48x16 p=3, steps it with a halo exchange per
stage, and rank 0 gathers the owned rows into one (nz, ny, 3, nphi, nx)
array.  ``--transport host`` lets all ranks share GPU 0 (gloo);
``--transport p2p`` uses NCCL with one GPU per rank; ``--transport fused``
the in-kernel peer-memory exchange (``--same-gpu``: all ranks on GPU 0).
"""

from __future__ import annotations

import argparse
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2303_11767_b200 as P  # noqa: E402
from paper_2303_11767_b200.bands import BandLayout, BandOperator  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--transport", default="host")
    ap.add_argument("--out", required=True)
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--same-gpu", action="store_true", help="all ranks on GPU 0 (gloo process group)")
    ap.add_argument("--graph", action="store_true", help="capture the steps in one CUDA graph (fused)")
    ap.add_argument("--nz", type=int, default=1)
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    same = args.transport == "host" or args.same_gpu
    dev = 0 if same else int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo" if same else "nccl")
    setup = P.build_case(P.default_config("williamson_tc6").override(nx=48, ny=16, p=3, nz=args.nz))
    op = P.SpatialOperator(setup.mesh, 3, setup.model, nz=args.nz)
    full = op.project_state(setup.ic).data.cpu().numpy()
    if args.nz > 1:
        full[1:] *= 1.0001                        # distinct levels
    L = BandLayout(16, world, rank)
    bop = BandOperator(op, L, transport=args.transport)
    u = bop.empty()
    u.copy_(torch.from_numpy(L.scatter(full)))
    w1, w2 = bop.empty(), bop.empty()
    bop.attach(u, w1, w2)
    # one batch of args.steps steps (one modal <-> nodal conversion each way)
    if args.graph:
        bop.begin(u)
        bop.nodal_steps(u, w1, w2, 5.0, 1, tag=0)        # eager first step
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            bop.nodal_steps(u, w1, w2, 5.0, args.steps - 1, tag=1)
        g.replay()
        bop.end(u)
    else:
        bop.ssprk3_steps(u, w1, w2, 5.0, args.steps)
    flags, _ = bop.status()
    assert flags == 0, flags
    mine = u[:, L.jlo:L.jhi].cpu().contiguous()
    if rank == 0:
        parts = [mine]
        for r in range(1, world):
            Lr = BandLayout(16, world, r)
            buf = torch.empty((full.shape[0], Lr.owned) + full.shape[2:], dtype=torch.float64)
            dist.recv(buf, src=r)
            parts.append(buf)
        np.save(args.out, torch.cat(parts, dim=1).numpy())
    else:
        dist.send(mine, dst=0)
    dist.barrier()
    torch.cuda.synchronize()
    bop.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
