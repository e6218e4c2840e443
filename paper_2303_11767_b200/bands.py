"""Latitude-band decomposition over GPUs (one process per GPU).

The reference has no domain decomposition (its only exchange is the
in-memory periodic halo copy, /root/reference/pkg/src/dgswe/dg.py:330-346).
Here the element grid is split into contiguous latitude bands: longitude
stays periodic inside every band and the poles are closed, so a band has at
most a southern and a northern neighbour.  Per RK stage each band sends its
first and last owned rows of the stage input to those neighbours and
receives one halo row from each -- a one-element-deep exchange,
point-to-point only (no collective on the hot path).  Both bands evaluate
the shared face with identical operands and code, so the numerical flux is
bit-identical on both sides and results do not depend on the band count.

Band buffer (per state): [nz][nrows = owned + 2][3][nstrip][nphi][32] (the
strip-blocked layout of operator.py); buffer row 0
is the southern halo (global row j0-1), rows 1..owned are owned, the last
row is the northern halo.  Halo rows at a pole are never read.

Transports: ``"p2p"`` -- torch.distributed batched isend/irecv on the
device tensors (NCCL over NVLink/NVSwitch on a B200 node; also gloo for
CPU tensors); ``"host"`` -- rows staged through host memory and exchanged
with gloo (test transport: lets several ranks share one GPU).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import _lib


@dataclass(frozen=True)
class BandLayout:
    ny: int
    world: int
    rank: int

    def __post_init__(self):
        if not 0 <= self.rank < self.world:
            raise ValueError("rank outside world")
        if self.world > self.ny:
            raise ValueError(f"cannot split {self.ny} latitude rows over {self.world} ranks")

    @staticmethod
    def split(ny: int, world: int):
        """[j0, j1) per rank; the first ny % world ranks get one extra row."""
        base, extra = divmod(ny, world)
        bounds, j = [], 0
        for r in range(world):
            n = base + (1 if r < extra else 0)
            bounds.append((j, j + n))
            j += n
        return bounds

    @property
    def rows(self):
        return self.split(self.ny, self.world)[self.rank]

    @property
    def j0(self):
        return self.rows[0]

    @property
    def j1(self):
        return self.rows[1]

    @property
    def owned(self):
        return self.j1 - self.j0

    @property
    def nrows(self):
        return self.owned + 2

    @property
    def row0(self):
        """Global row of buffer row 0 (the southern halo)."""
        return self.j0 - 1

    @property
    def jlo(self):
        return 1

    @property
    def jhi(self):
        return 1 + self.owned

    @property
    def south(self):
        return self.rank - 1 if self.j0 > 0 else None

    @property
    def north(self):
        return self.rank + 1 if self.j1 < self.ny else None

    def scatter(self, full: np.ndarray) -> np.ndarray:
        """Band buffer (halos filled) from a global device-layout array (nz, ny, ...)."""
        nz = full.shape[0]
        out = np.zeros((nz, self.nrows) + full.shape[2:], dtype=full.dtype)
        lo, hi = max(self.j0 - 1, 0), min(self.j1 + 1, self.ny)
        out[:, lo - self.row0:hi - self.row0] = full[:, lo:hi]
        return out


def _row_buffers(data: torch.Tensor, r: int):
    view = data[:, r]
    return view, (view if view.is_contiguous() else view.contiguous())


def exchange_halos(data: torch.Tensor, layout: BandLayout, transport: str = "p2p", group=None):
    """Fill the band's halo rows of ``data`` from its neighbours (blocking
    for the caller's stream; see :class:`HaloExchange` for the split form)."""
    ex = HaloExchange(layout, transport, group)
    ex.start(data)
    ex.finish()


class HaloExchange:
    """start() posts the sends/receives, finish() completes them.  With NCCL
    the transfer runs on NCCL's stream while the caller launches interior
    rows; finish() makes the current stream wait for it."""

    def __init__(self, layout: BandLayout, transport: str = "p2p", group=None):
        if transport not in ("p2p", "host"):
            raise ValueError(f"unknown transport {transport!r}")
        self.layout, self.transport, self.group = layout, transport, group
        self._pending = None

    def _peer(self, r):
        return dist.get_global_rank(self.group, r) if self.group is not None else r

    def start(self, data: torch.Tensor):
        L = self.layout
        sends, recvs = [], []
        if L.south is not None:
            sends.append((_row_buffers(data, L.jlo)[1], L.south))
            recvs.append((data[:, 0], L.south))
        if L.north is not None:
            sends.append((_row_buffers(data, L.jhi - 1)[1], L.north))
            recvs.append((data[:, L.jhi], L.north))
        if self.transport == "host":
            sends = [(t.cpu(), p) for t, p in sends]
        rbufs = [(torch.empty(d.shape, dtype=d.dtype,
                              device="cpu" if self.transport == "host" else d.device), d, p)
                 for d, p in recvs]
        ops = [dist.P2POp(dist.isend, t, self._peer(p), self.group) for t, p in sends]
        ops += [dist.P2POp(dist.irecv, b, self._peer(p), self.group) for b, _, p in rbufs]
        reqs = dist.batch_isend_irecv(ops) if ops else []
        self._pending = (reqs, rbufs, sends)

    def finish(self):
        reqs, rbufs, _ = self._pending
        for r in reqs:
            r.wait()
        for buf, dst, _ in rbufs:
            dst.copy_(buf)
        self._pending = None


class BandOperator:
    """The fused stage kernel for one latitude band (C-ABI context with
    row0/nrows/jlo/jhi set to the band buffer)."""

    def __init__(self, op_host, layout: BandLayout, transport: str = "p2p", group=None,
                 row_chunk: int = 0, overlap: bool = True):
        from .operator import _Context
        self.op = op_host          # geometry / tables source (mesh, p, model, rusanov, nz)
        self.layout = layout
        self.transport = transport
        self.group = group
        self.overlap = overlap and transport == "p2p"
        mesh = op_host.mesh
        from .operator import device_shape
        self.shape = device_shape(op_host.nz, layout.nrows, op_host.nphi, mesh.nx)
        self.ctx = _Context(mesh, op_host.p, op_host.model, op_host.rusanov, op_host.nz,
                            op_host.quad, op_host.vander, op_host.Minv_rows, row0=layout.row0,
                            nrows=layout.nrows, jlo=layout.jlo, jhi=layout.jhi, row_chunk=row_chunk)
        self.global_alpha = op_host.rusanov.mode == "global" and op_host.rusanov.alpha is None
        if self.global_alpha:
            _lib.check(self.ctx.lib.dgswe_set_external_alpha(self.ctx.h, 1), "set_external_alpha")
        self.halo = HaloExchange(layout, transport, group)

    def empty(self, device=None):
        return torch.zeros(self.shape, dtype=torch.float64,
                           device=device or torch.device("cuda", torch.cuda.current_device()))

    def _alpha_tensor(self):
        ptr = self.ctx.lib.dgswe_alpha_buffer(self.ctx.h)

        class _Arr:
            __cuda_array_interface__ = {"shape": (2,), "typestr": "<f8", "data": (ptr, False),
                                        "version": 3}
        return torch.as_tensor(_Arr(), device="cuda")

    def _launch(self, a, U, b, X, g, Y, tag, r0, r1):
        c = self.ctx
        _lib.check(c.lib.dgswe_stage_rows(
            c.h, float(a), ctypes.c_void_p(U.data_ptr() if U is not None else 0), float(b),
            ctypes.c_void_p(X.data_ptr()), float(g), ctypes.c_void_p(Y.data_ptr()), int(tag),
            int(r0), int(r1), c.stream()), "dgswe_stage_rows")

    def _launch2(self, a, U, b, X, g, Y, tag, r0, r1, r2, r3):
        c = self.ctx
        _lib.check(c.lib.dgswe_stage_rows2(
            c.h, float(a), ctypes.c_void_p(U.data_ptr() if U is not None else 0), float(b),
            ctypes.c_void_p(X.data_ptr()), float(g), ctypes.c_void_p(Y.data_ptr()), int(tag),
            int(r0), int(r1), int(r2), int(r3), c.stream()), "dgswe_stage_rows2")

    def stage(self, a, U, b, X, g, Y, tag=0):
        """Halo exchange of X, then Y = a U + b X + g RHS(X) on owned rows."""
        L = self.layout
        self.halo.start(X)
        if self.global_alpha:
            self.halo.finish()
            _lib.check(self.ctx.lib.dgswe_alpha_prepass(self.ctx.h, ctypes.c_void_p(X.data_ptr()),
                                                        self.ctx.stream()), "alpha_prepass")
            if self.layout.world > 1:
                dist.all_reduce(self._alpha_tensor(), op=dist.ReduceOp.MAX, group=self.group)
            self._launch(a, U, b, X, g, Y, tag, L.jlo, L.jhi)
            return
        if self.overlap and L.owned > 2:
            self._launch(a, U, b, X, g, Y, tag, L.jlo + 1, L.jhi - 1)   # no halo needed
            self.halo.finish()
            # both boundary rows in one launch
            self._launch2(a, U, b, X, g, Y, tag, L.jlo, L.jlo + 1, L.jhi - 1, L.jhi)
        else:
            self.halo.finish()
            self._launch(a, U, b, X, g, Y, tag, L.jlo, L.jhi)

    def ssprk3_step(self, u, w1, w2, dt, tag=0):
        self.stage(0.0, None, 1.0, u, dt, w1, tag)
        self.stage(0.75, u, 0.25, w1, 0.25 * dt, w2, tag)
        self.stage(1.0 / 3.0, u, 2.0 / 3.0, w2, (2.0 / 3.0) * dt, u, tag)

    def status(self, reset=True):
        return self.ctx.status(reset)

    def launch_count(self):
        return self.ctx.launches()
