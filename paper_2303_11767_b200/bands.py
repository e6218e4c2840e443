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

Transports:
* ``"fused"`` -- no host collective on the path: one launch per stage
  (``dgswe_stage_band``) whose first CTAs compute the two edge rows and
  store them straight into the neighbours' halo rows over peer memory (CUDA
  IPC mappings: NVLink/NVSwitch on a B200 node), bumping the neighbours'
  receive counters; an edge row first waits (bounded) for its own counter
  to show the neighbour's previous-stage rows.  The interior CTAs of the
  same launch need no halo and run at once.  Buffers must come from
  :meth:`BandOperator.empty` (IPC-mappable) and be registered with
  :meth:`BandOperator.attach`;
* ``"p2p"`` -- torch.distributed batched isend/irecv on the device tensors
  (NCCL over NVLink/NVSwitch; also gloo for CPU tensors);
* ``"host"`` -- rows staged through host memory and exchanged with gloo
  (test transport: lets several ranks share one GPU).
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
        if transport not in ("p2p", "host", "fused"):
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
                            nrows=layout.nrows, jlo=layout.jlo, jhi=layout.jhi, row_chunk=row_chunk,
                            bottom=op_host.bottom_nodal)
        self.global_alpha = op_host.rusanov.mode == "global" and op_host.rusanov.alpha is None
        if self.global_alpha:
            _lib.check(self.ctx.lib.dgswe_set_external_alpha(self.ctx.h, 1), "set_external_alpha")
        if transport == "fused" and self.global_alpha:
            raise ValueError("transport 'fused' supports local / pinned alpha only")
        # the fused transport still exchanges u's halos once per step batch
        # (begin), over NCCL -- or the host when the group is gloo
        hx = "p2p" if transport == "fused" else transport
        if hx == "p2p" and dist.is_initialized() and dist.get_backend(group) == "gloo":
            hx = "host"                # gloo moves host memory only
        self.halo = HaloExchange(layout, hx, group)
        self._owned_mem = []       # (ptr, keep-alive) of library allocations
        self._opened = []          # peer mappings to close
        self._peer_rows = {}       # data_ptr of our buffer -> (south row ptr, north row ptr)

    def empty(self, device=None):
        if self.transport != "fused":
            return torch.zeros(self.shape, dtype=torch.float64,
                               device=device or torch.device("cuda", torch.cuda.current_device()))
        # IPC-mappable, zero-filled library allocation viewed as a tensor
        lib = self.ctx.lib
        nbytes = int(np.prod(self.shape)) * 8
        ptr = ctypes.c_void_p()
        _lib.check(lib.dgswe_dev_alloc(nbytes, ctypes.byref(ptr)), "dgswe_dev_alloc")
        shape = self.shape

        class _Mem:
            __cuda_array_interface__ = {"shape": shape, "typestr": "<f8", "data": (ptr.value, False),
                                        "version": 3}
        t = torch.as_tensor(_Mem(), device="cuda")
        self._owned_mem.append((ptr.value, t))
        return t

    def attach(self, *buffers):
        """Fused transport: exchange CUDA IPC handles of this rank's state
        buffers (their order is their role, identical on every rank) and of
        the receive counters, and register the peer mappings."""
        if self.transport != "fused":
            return
        lib, L = self.ctx.lib, self.layout
        ctrl = self.empty_ctrl()
        ptrs = [b.data_ptr() for b in buffers] + [ctrl]
        handles = []
        for ptr in ptrs:
            buf = ctypes.create_string_buffer(64)
            _lib.check(lib.dgswe_ipc_handle(ctypes.c_void_p(ptr), buf), "dgswe_ipc_handle")
            handles.append(buf.raw)
        mine = {"rank": L.rank, "nrows": L.nrows, "handles": handles}
        allinfo = [None] * L.world
        dist.all_gather_object(allinfo, mine, group=self.group)
        rstride = int(np.prod(self.shape[2:]))                  # doubles per buffer row
        peers = {}
        for side, nb in ((0, L.south), (1, L.north)):
            if nb is None:
                continue
            info = allinfo[nb]
            opened = []
            for h in info["handles"]:
                p = ctypes.c_void_p()
                _lib.check(lib.dgswe_ipc_open(h, ctypes.byref(p)), "dgswe_ipc_open")
                opened.append(p.value)
                self._opened.append(p.value)
            peers[side] = (info["nrows"], opened)
        # our edge row goes to the south neighbour's NORTH halo (its last row)
        # and to the north neighbour's SOUTH halo (its row 0)
        for k, b in enumerate(buffers):
            rows = []
            for side in (0, 1):
                if side not in peers:
                    rows.append(None)
                    continue
                nrows, opened = peers[side]
                row = nrows - 1 if side == 0 else 0
                rows.append(opened[k] + row * rstride * 8)
            self._peer_rows[b.data_ptr()] = rows
        cnt = [None, None]
        zs = [0, 0]
        for side in (0, 1):
            if side in peers:
                nrows, opened = peers[side]
                # the neighbour's counter of deliveries from OUR side of it
                cnt[side] = opened[-1] + (8 if side == 0 else 0)
                zs[side] = nrows * rstride
        _lib.check(lib.dgswe_set_exchange(self.ctx.h, zs[0], ctypes.c_void_p(cnt[0] or 0), zs[1],
                                          ctypes.c_void_p(cnt[1] or 0), ctypes.c_void_p(ctrl),
                                          ctypes.c_void_p(ctrl + 16)), "dgswe_set_exchange")
        torch.cuda.synchronize()
        dist.barrier(group=self.group)          # every rank mapped before any delivery

    def empty_ctrl(self):
        """recv_count[2] (south, north deliveries) + stage_ctr[2], zeroed."""
        ptr = ctypes.c_void_p()
        _lib.check(self.ctx.lib.dgswe_dev_alloc(32, ctypes.byref(ptr)), "dgswe_dev_alloc")
        self._owned_mem.append((ptr.value, None))
        return ptr.value

    def close(self):
        lib = self.ctx.lib
        for p in self._opened:
            lib.dgswe_ipc_close(ctypes.c_void_p(p))
        self._opened = []
        for p, _ in self._owned_mem:
            lib.dgswe_dev_free(ctypes.c_void_p(p))
        self._owned_mem = []

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

    def _stage_fused(self, a, U, b, X, g, Y, tag):
        """The whole band in one launch (dgswe_stage_band): edge rows first,
        stored into the neighbours' halos over peer memory; interior rows
        need no halo and run at once."""
        c = self.ctx
        rows = self._peer_rows.get(Y.data_ptr())
        if rows is None:
            raise ValueError("fused transport: Y was not registered with attach()")
        _lib.check(c.lib.dgswe_stage_band(
            c.h, float(a), ctypes.c_void_p(U.data_ptr() if U is not None else 0), float(b),
            ctypes.c_void_p(X.data_ptr()), float(g), ctypes.c_void_p(Y.data_ptr()), int(tag),
            ctypes.c_void_p(rows[0] or 0), ctypes.c_void_p(rows[1] or 0), c.stream()), "dgswe_stage_band")

    def stage(self, a, U, b, X, g, Y, tag=0):
        """Halo exchange of X, then Y = a U + b X + g RHS(X) on owned rows."""
        L = self.layout
        if self.transport == "fused":
            return self._stage_fused(a, U, b, X, g, Y, tag)
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

    # Step batches run on nodal values (include/dgswe_b200.h, "State basis"):
    # begin() converts the owned rows of u in place and refreshes its halo
    # rows from the neighbours' converted rows, the stages then exchange
    # nodal rows, end() converts the owned rows back.  Between begin() and
    # end(), stage() / _launch*() take nodal states.
    def begin(self, u):
        L = self.layout
        self.ctx.convert(u, True, L.jlo, L.jhi)
        self.ctx.set_basis(True)
        if L.world > 1:
            self.halo.start(u)
            self.halo.finish()

    def end(self, u):
        L = self.layout
        self.ctx.convert(u, False, L.jlo, L.jhi)
        self.ctx.set_basis(False)

    def nodal_steps(self, u, w1, w2, dt, k, tag=0):
        """k SSPRK3 steps on a nodal u (between begin and end; capturable
        in a CUDA graph for the fused transport)."""
        for i in range(k):
            t = tag + i
            self.stage(0.0, None, 1.0, u, dt, w1, t)
            self.stage(0.75, u, 0.25, w1, 0.25 * dt, w2, t)
            self.stage(1.0 / 3.0, u, 2.0 / 3.0, w2, (2.0 / 3.0) * dt, u, t)

    def ssprk3_steps(self, u, w1, w2, dt, k, tag=0):
        """k SSPRK3 steps of the band's modal state u (one conversion each way)."""
        self.begin(u)
        self.nodal_steps(u, w1, w2, dt, k, tag)
        self.end(u)

    def ssprk3_step(self, u, w1, w2, dt, tag=0):
        self.ssprk3_steps(u, w1, w2, dt, 1, tag)

    def status(self, reset=True):
        return self.ctx.status(reset)

    def launch_count(self):
        return self.ctx.launches()
