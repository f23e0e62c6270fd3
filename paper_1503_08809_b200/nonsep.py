"""Non-separable direct Γ path on a sparse l-grid (BASELINE config 3).

No reference counterpart exists; the call is written in the style of `gamma3d_matrix`
(engine3d.py:156-186) and its loop structure follows `gamma3d_naive` (engine3d.py:189-215):
per triple, the primordial bispectrum B(t,x) = Σ_n' α_n' Σ_6perms q̃q̃q̃ is evaluated
pointwise (not factored through Γ), integrated over x with wr2, weighted by zm_t and the
sparse-grid volume weight W_t, and projected onto the late-time modes:

    b[m] = Σ_t W_t zm_t P[m,t] Σ_x wr2_x B(t,x)        -> GammaMatrix of shape [n, 1]
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .engine3d import _FP_POOL, _meta_dict, check_shapes
from .gamma import GammaMatrix
from .quadrature import x_weights

__all__ = ["SparseDomain", "gamma_nonsep"]


@dataclass
class SparseDomain:
    """Ordered triples l1 <= l2 <= l3 of a sparse l-grid with volume weights W."""

    l1: np.ndarray
    l2: np.ndarray
    l3: np.ndarray
    weight: np.ndarray

    def __post_init__(self):
        self.l1 = np.asarray(self.l1, np.int64)
        self.l2 = np.asarray(self.l2, np.int64)
        self.l3 = np.asarray(self.l3, np.int64)
        self.weight = np.asarray(self.weight, np.float64)
        if not (self.l1.shape == self.l2.shape == self.l3.shape == self.weight.shape):
            raise ValueError("sparse domain arrays must have equal length")

    @property
    def count(self) -> int:
        return int(self.l1.size)

    @classmethod
    def from_grid(cls, grid, w1d):
        from .configs import sparse_domain
        return cls(*sparse_domain(grid, w1d))


def gamma_nonsep(tables, mapping, grid, alpha, domain: SparseDomain, h2_mode: str = "gosper",
                 integrator: str = "trap", *, device: int = 0) -> GammaMatrix:
    if h2_mode not in nat.MG_H2:
        raise ValueError(f"unknown h2_mode {h2_mode!r}")
    q = np.ascontiguousarray(tables.q, np.float64)
    qt = np.ascontiguousarray(tables.q_tilde, np.float64)
    C = np.ascontiguousarray(tables.C, np.float64)
    v = np.ascontiguousarray(tables.v, np.float64)
    entries = np.ascontiguousarray(mapping.entries, np.int64)
    alpha = np.ascontiguousarray(alpha, np.float64)
    if alpha.shape != (entries.shape[0],):
        raise ValueError("alpha must have one coefficient per primordial mode")
    wr2 = np.ascontiguousarray(x_weights(grid.r, integrator), np.float64)
    check_shapes(q, qt, C, v, wr2, int(tables.l_min), int(tables.l_max))
    l1 = np.ascontiguousarray(domain.l1, np.int32)
    l2 = np.ascontiguousarray(domain.l2, np.int32)
    l3 = np.ascontiguousarray(domain.l3, np.int32)
    W = np.ascontiguousarray(domain.weight, np.float64)
    n = entries.shape[0]
    b = np.zeros(n)
    fp = _FP_POOL.submit(lambda: (tables.fingerprint(), grid.fingerprint(),
                                  mapping.fingerprint()))   # overlaps the GPU call
    nat.check(nat.lib().mg_gamma_nonsep(
        nat.ptr(q), nat.ptr(qt), nat.ptr(C), nat.ptr(v), nat.ptr(wr2), nat.ptr(entries),
        q.shape[0], qt.shape[1], n, int(tables.l_min), int(tables.l_max), nat.MG_H2[h2_mode],
        nat.ptr(alpha), nat.ptr(l1), nat.ptr(l2), nat.ptr(l3), nat.ptr(W), int(l1.size),
        int(device), nat.ptr(b)))
    meta = _meta_dict(tables, grid, mapping, integrator, h2_mode, 1, 1, *fp.result())
    meta["engine"] = "modal3d-nonsep"
    meta["triples"] = int(l1.size)
    return GammaMatrix(b.reshape(n, 1), meta)
