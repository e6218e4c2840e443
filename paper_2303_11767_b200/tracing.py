"""Operation recorder: the counterpart of the reference's
``fields.set_op_recorder`` (/root/reference/pkg/src/dgswe/fields.py:66-76,
295-298), which its benchmark harness uses to collect analytic flop / byte
counts of every engine operation.

The reference records one entry per numpy/numba engine call (``kind``,
``op``, execution region, flops, bytes).  Here the path is a few fused
kernels, so one entry is recorded per device launch issued through
``SpatialOperator``: ``kind`` = "stage" | "rhs" | "axpy" | "rk_steps",
``op`` = the entry point, ``rgn`` = a :class:`LaunchRegion` (elements x
rows x levels and the degree), ``flops`` = an analytic estimate of the
fused operator's FP64 flops (:func:`stage_flops_per_dof`), ``nbytes`` = the
algorithmic HBM bytes (states read and written once: 16 B per DOF for a
stage without u^n, 24 with it).
"""

from __future__ import annotations

from dataclasses import dataclass

_RECORDER = None


def set_op_recorder(recorder) -> None:
    """Install (or clear, with None) the global operation recorder: an
    object with ``record(kind, op, rgn, flops, nbytes)``."""
    global _RECORDER
    _RECORDER = recorder


def get_op_recorder():
    return _RECORDER


@dataclass(frozen=True)
class LaunchRegion:
    """The work of one launch: ``domain`` = (nx, rows, nz) elements, degree
    p, ``nvars`` variables (3 for shallow water, 1 for linear advection)."""

    domain: tuple
    p: int
    nvars: int = 3

    @property
    def dofs(self) -> int:
        nx, rows, nz = self.domain
        return nx * rows * nz * self.nvars * (self.p + 1) ** 2


def stage_flops_per_dof(p: int) -> float:
    """Analytic FP64 flops per DOF-update of one fused stage (nodal form,
    n = p+1 nodes per direction; an FMA counts 2): element traces
    4 n (2n-1) / n^2 per DOF, the two weak derivatives 4n, pointwise physics
    ~10 (momentum equations: one reciprocal, velocities, fluxes, source),
    the two faces per element ~30 flops per face node and variable spread
    over n DOFs, the four face lifts 8, mass and stage combination 4."""
    n = p + 1
    return 4.0 * (2 * n - 1) / n + 4.0 * n + 10.0 + 20.0 / n + 8.0 + 4.0


def adv_stage_flops_per_dof(p: int) -> float:
    """Analytic FP64 flops per DOF-update of one linear-advection stage
    (dgswe_adv.cuh, n = p+1, FMA = 2): modal <-> nodal conversions 8n, the
    two weak derivatives 4n, traces of the element and its neighbours from
    the modes ~16 over n^2 nodes per face pair, fluxes and lifts ~12,
    mass and stage combination 4."""
    n = p + 1
    return 12.0 * n + 16.0 / n + 16.0


def record(kind: str, op: str, rgn: LaunchRegion, bytes_per_dof: float, flops_per_dof: float) -> None:
    if _RECORDER is not None:
        d = rgn.dofs
        _RECORDER.record(kind, op, rgn, int(round(flops_per_dof * d)), int(round(bytes_per_dof * d)))
