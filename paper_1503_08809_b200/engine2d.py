"""Drop-in for the reference's μ-quadrature engine (engine2d.py:62-211) on the GPU.

    build_ptable(tables, grid, rule, legendre, budget_bytes=2 GiB) -> PTable
    gamma2d_matrix(tables, mapping, grid, rule, legendre, integrator="trap", workers=1,
                   ptable=None, *, device=0) -> GammaMatrix

Same arguments, errors (MemoryError above the P-table budget, engine2d.py:75-79; ValueError
for a short Legendre table, :80-81) and meta keys ("modal2d", n_mu, workers).  The P table
is built on the device with the reference's Kahan order and is bit-identical to it; the cell
sums (permanent, μ rule, radial rule) agree to rounding.  This engine is the paper's
"separable, unstable" Modal2D; it is kept as the reference keeps it: the cross-check of
the direct engine (acceptance criterion 1, test_acceptance.py:50-57).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .engine3d import _FP_POOL, _meta_dict
from .gamma import GammaMatrix
from .quadrature import default_mu_points, gauss_legendre, legendre_table, x_weights

__all__ = ["PTable", "build_ptable", "gamma2d_matrix", "default_mu_points", "gauss_legendre",
           "legendre_table", "DEFAULT_PTABLE_BUDGET", "last_kernel_ms"]

DEFAULT_PTABLE_BUDGET = 2 << 30


@dataclass(frozen=True)
class PTable:
    """values[a, b, x, m]: late index a, primordial index b, radial point x, μ node m."""

    values: np.ndarray

    @property
    def p_max(self) -> int:
        return self.values.shape[0]


def last_kernel_ms() -> tuple:
    """(P-table kernel ms, cell-sum kernels ms) of this thread's last build_ptable /
    gamma2d_matrix call, from CUDA events around the launches (mg_gamma2d_timings)."""
    import ctypes
    a, b = ctypes.c_double(0.0), ctypes.c_double(0.0)
    nat.check(nat.lib().mg_gamma2d_timings(ctypes.byref(a), ctypes.byref(b)))
    return a.value, b.value


def _inputs(tables, legendre):
    if legendre.shape[0] < tables.l_max + 1:
        raise ValueError("legendre table does not reach l_max")
    ells = np.arange(tables.l_min, tables.l_max + 1).astype(np.float64)
    lw = (2.0 * ells + 1.0) / (tables.v * np.sqrt(tables.C))        # engine2d.py:44-47
    leg = np.ascontiguousarray(legendre[tables.l_min:tables.l_max + 1], np.float64)
    q = np.ascontiguousarray(tables.q, np.float64)
    qt = np.ascontiguousarray(tables.q_tilde, np.float64)
    return q, qt, np.ascontiguousarray(lw), leg


def build_ptable(tables, grid, rule, legendre, budget_bytes: int = DEFAULT_PTABLE_BUDGET,
                 *, device: int = 0) -> PTable:
    p, nr, nmu = tables.p_max, tables.n_radial, rule.n
    need = p * p * nr * nmu * 8
    if need > budget_bytes:
        raise MemoryError(f"P table needs {need} bytes but the budget allows {budget_bytes}")
    q, qt, lw, leg = _inputs(tables, legendre)
    if np.size(grid.r) != nr:
        raise ValueError(f"radial grid has {np.size(grid.r)} points but q_tilde has {nr}")
    out = np.empty((p, p, nr, nmu))      # every element is written by the device copy
    nat.check(nat.lib().mg_ptable(nat.ptr(q), nat.ptr(qt), nat.ptr(lw), nat.ptr(leg), p, nr,
                                  lw.size, nmu, int(device), nat.ptr(out)))
    return PTable(out)


def gamma2d_matrix(tables, mapping, grid, rule, legendre, integrator: str = "trap",
                   workers: int = 1, ptable: PTable | None = None, *,
                   device: int = 0) -> GammaMatrix:
    p, nr, nmu = tables.p_max, tables.n_radial, rule.n
    e = np.ascontiguousarray(mapping.entries, np.int64)
    n = e.shape[0]
    wr2 = np.ascontiguousarray(x_weights(grid.r, integrator))
    if wr2.size != nr:
        raise ValueError(f"radial grid has {wr2.size} points but q_tilde has {nr} (n_radial)")
    muw = np.ascontiguousarray(rule.weights, np.float64)
    out = np.zeros((n, n))
    fp = _FP_POOL.submit(lambda: (tables.fingerprint(), grid.fingerprint(),
                                  mapping.fingerprint()))   # overlaps the GPU call
    if ptable is not None:
        pv = np.ascontiguousarray(ptable.values, np.float64)
        if pv.shape != (p, p, nr, nmu):
            raise ValueError("P table shape does not match the inputs")
        nat.check(nat.lib().mg_gamma2d(None, None, None, None, nat.ptr(pv), nat.ptr(muw),
                                       nat.ptr(wr2), nat.ptr(e), p, nr, 0, nmu, n,
                                       int(device), nat.ptr(out)))
    else:
        need = p * p * nr * nmu * 8
        if need > DEFAULT_PTABLE_BUDGET:
            raise MemoryError(f"P table needs {need} bytes but the budget allows "
                              f"{DEFAULT_PTABLE_BUDGET}")
        q, qt, lw, leg = _inputs(tables, legendre)
        nat.check(nat.lib().mg_gamma2d(nat.ptr(q), nat.ptr(qt), nat.ptr(lw), nat.ptr(leg),
                                       None, nat.ptr(muw), nat.ptr(wr2), nat.ptr(e), p, nr,
                                       lw.size, nmu, n, int(device), nat.ptr(out)))
    meta = _meta_dict(tables, grid, mapping, integrator, "n/a", 1, workers, *fp.result())
    meta.pop("h2_mode"), meta.pop("block")
    meta.update({"engine": "modal2d", "n_mu": nmu, "workers": workers})
    return GammaMatrix(out, meta)
