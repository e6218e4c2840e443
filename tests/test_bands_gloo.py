"""Latitude-band decomposition and halo exchange on CPU (gloo, world 2/3).

The exchange code is device-agnostic torch.distributed P2P; on the B200
node it runs with NCCL on device tensors.  Kernel-side band semantics are
covered on the GPU by tests/test_gpu_parity.py::test_band_decomposition_*.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2303_11767_b200.bands import BandLayout, HaloExchange, exchange_halos


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_split_covers_rows():
    for ny in (1, 5, 20, 360):
        for world in range(1, min(ny, 9) + 1):
            b = BandLayout.split(ny, world)
            assert b[0][0] == 0 and b[-1][1] == ny
            assert all(b[k][1] == b[k + 1][0] for k in range(world - 1))
            sizes = [hi - lo for lo, hi in b]
            assert max(sizes) - min(sizes) <= 1 and min(sizes) >= 1
    with pytest.raises(ValueError):
        BandLayout(3, 4, 0)


def test_layout_buffer_geometry():
    L = BandLayout(10, 3, 1)
    assert (L.j0, L.j1, L.nrows, L.row0, L.jlo, L.jhi) == (4, 7, 5, 3, 1, 4)
    assert (L.south, L.north) == (0, 2)
    assert BandLayout(10, 3, 0).south is None and BandLayout(10, 3, 2).north is None
    full = np.arange(2 * 10 * 3 * 4 * 5, dtype=np.float64).reshape(2, 10, 3, 4, 5)
    band = L.scatter(full)
    assert np.array_equal(band[:, 1:4], full[:, 4:7])
    assert np.array_equal(band[:, 0], full[:, 3]) and np.array_equal(band[:, 4], full[:, 7])
    south = BandLayout(10, 3, 0).scatter(full)
    assert np.all(south[:, 0] == 0)           # pole halo never filled


def _worker(rank, world, port, nz, ny, split, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        L = BandLayout(ny, world, rank)
        rng = np.random.default_rng(7)
        full = rng.normal(size=(nz, ny, 3, 4, 6))
        band = torch.from_numpy(L.scatter(full))
        truth = band.clone()
        band[:, 0] = -99.0                      # poison the halos
        band[:, L.jhi] = -99.0
        if split:
            ex = HaloExchange(L, "p2p")
            ex.start(band)
            ex.finish()
        else:
            exchange_halos(band, L, "p2p")
        ok = True
        if L.south is not None:
            ok &= torch.equal(band[:, 0], truth[:, 0])
        if L.north is not None:
            ok &= torch.equal(band[:, L.jhi], truth[:, L.jhi])
        ok &= torch.equal(band[:, 1:L.jhi], truth[:, 1:L.jhi])
        q.put((rank, bool(ok)))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as exc:  # pragma: no cover - reported to the parent
        q.put((rank, repr(exc)))


@pytest.mark.parametrize("world,nz,ny,split", [(2, 1, 6, False), (2, 2, 5, True), (3, 1, 7, True)])
def test_halo_exchange_gloo(world, nz, ny, split):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, nz, ny, split, q))
             for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert results == {r: True for r in range(world)}, results
