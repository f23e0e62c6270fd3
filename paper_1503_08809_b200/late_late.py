"""Late-late inner product ⟨Q,Q⟩ and the full estimator Γ = ⟨Q,Q⟩⁻¹⟨Q,Q̃'⟩.

PAPER.md:705-722 (out of scope for the reference):
    ⟨A,B⟩ = Σ_{l1l2l3} (h/(v1v2v3))² A B,   Q_n = (1/6) Σ_6perms q_i q_j q_k,
so over the ordered domain with multiplicities
    ⟨Q_n,Q_m⟩ = Σ_t mult_t h²_t / (36 (v1v2v3)²) P[n,t] P[m,t].
That is the separable Γ' engine with q̃ -> q (one "x" point of weight 1) and C_l -> v_l²
(the Gosper or exact h² weights are unchanged), so it runs on the same kernels.
"""

from __future__ import annotations

import numpy as np

from . import _native as nat
from .engine3d import _meta_dict, gamma3d_matrix
from .gamma import GammaMatrix

__all__ = ["gamma_late_late", "gamma_estimator"]


def gamma_late_late(tables, mapping, h2_mode: str = "gosper", *,
                    device: int = 0, _fingerprints=None) -> GammaMatrix:
    """⟨Q_n, Q_m⟩ on the tetrahedral domain, [n, n] symmetric.  `_fingerprints` = (tables,
    mapping) digests already computed by the caller (gamma_estimator hashes the tables once)."""
    if h2_mode not in nat.MG_H2:
        raise ValueError(f"unknown h2_mode {h2_mode!r}")
    q = np.ascontiguousarray(tables.q, np.float64)
    v = np.ascontiguousarray(tables.v, np.float64)
    qt = np.ascontiguousarray(q[:, None, :])          # [p, 1, L]
    C = np.ascontiguousarray(v * v)                   # sqrt(C1C2C3) -> v1v2v3
    wr2 = np.ones(1)
    e = np.ascontiguousarray(mapping.entries, np.int64)
    n = e.shape[0]
    out = np.zeros((n, n))
    devs = np.array([device], np.int32)
    nat.check(nat.lib().mg_gamma_sep(
        nat.ptr(q), nat.ptr(qt), nat.ptr(C), nat.ptr(v), nat.ptr(wr2), nat.ptr(e), q.shape[0],
        1, n, int(tables.l_min), int(tables.l_max), nat.MG_H2[h2_mode], 0, -1, 1,
        nat.ptr(devs), nat.ptr(out)))
    ft, fm = _fingerprints or (tables.fingerprint(), mapping.fingerprint())
    meta = {"engine": "modal3d-QQ", "l_min": tables.l_min, "l_max": tables.l_max,
            "p_max": tables.p_max, "n_max": n, "h2_mode": h2_mode, "tables": ft, "mapping": fm}
    return GammaMatrix(out, meta)


def gamma_estimator(tables, mapping, grid, h2_mode: str = "gosper",
                    integrator: str = "trap", *, device: int = 0):
    """(Γ, ⟨Q,Q⟩, Γ') with Γ = ⟨Q,Q⟩⁻¹ Γ'; Γ' = gamma3d_matrix."""
    gp = gamma3d_matrix(tables, mapping, grid, h2_mode=h2_mode, integrator=integrator,
                        device=device)
    ft, fg, fm = gp.meta["tables"], gp.meta["grid"], gp.meta["mapping"]
    qq = gamma_late_late(tables, mapping, h2_mode, device=device, _fingerprints=(ft, fm))
    full = np.linalg.solve(qq.values, gp.values)
    meta = _meta_dict(tables, grid, mapping, integrator, h2_mode, 1, 1, ft, fg, fm)
    meta["engine"] = "modal3d-estimator"
    return GammaMatrix(full, meta), qq, gp
