"""CPU ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Non-separable direct path (BASELINE config 3) restated in the loop structure of
gamma3d_naive (engine3d.py:189-215) with radial_integral_x (engine3d.py:56-70) and
late_product_y (engine3d.py:73-83):

    b[m] = Σ_t W_t zm_t P[m,t] Σ_x wr2_x Σ_n' α_n' Σ_6perms q̃q̃q̃(x; t)

No reference implementation exists — parity unpinned; anchored by the known answer
b == Γ α on a step-1 grid (W = 1, exact parity), where Γ is the reference Γ.
"""

from __future__ import annotations

from itertools import permutations

import numpy as np

from .ref import triple_zm

_PERMS = tuple(permutations((0, 1, 2)))


def nonsep(q, qt, C, v, wr2, entries, alpha, l_min, l1, l2, l3, W, h2_mode="gosper",
           block=256):
    n = entries.shape[0]
    b = np.zeros(n)
    cols = (entries[:, 0], entries[:, 1], entries[:, 2])
    for s in range(0, l1.size, block):
        a1, a2, a3 = l1[s:s + block], l2[s:s + block], l3[s:s + block]
        i1, i2, i3 = a1 - l_min, a2 - l_min, a3 - l_min
        zm = triple_zm(l_min, a1, a2, a3, C, v, h2_mode)
        t1, t2, t3 = qt[:, :, i1], qt[:, :, i2], qt[:, :, i3]          # [p, Nx, B]
        f = np.zeros((n, qt.shape[1], a1.size))
        for a, bb, c in _PERMS:
            f += t1[cols[a]] * t2[cols[bb]] * t3[cols[c]]
        B = np.einsum("n,nxb->xb", alpha, f)                           # pointwise bispectrum
        X = wr2 @ B                                                    # [B]
        q1, q2, q3 = q[:, i1], q[:, i2], q[:, i3]
        P = np.zeros((n, a1.size))
        for a, bb, c in _PERMS:
            P += q1[cols[a]] * q2[cols[bb]] * q3[cols[c]]
        b += P @ (W[s:s + block] * zm * X)
    return b


_SHARED = {}


def _nonsep_job(args):
    lo, hi, h2_mode, block = args
    d = _SHARED
    return nonsep(d["q"], d["qt"], d["C"], d["v"], d["wr2"], d["entries"], d["alpha"],
                  d["l_min"], d["l1"][lo:hi], d["l2"][lo:hi], d["l3"][lo:hi], d["W"][lo:hi],
                  h2_mode, block)


def nonsep_parallel(q, qt, C, v, wr2, entries, alpha, l_min, l1, l2, l3, W, h2_mode="gosper",
                    workers=None, block=256):
    """`nonsep` over a fork pool: contiguous chunks, partials summed in worker order (the
    reference's worker split, engine3d.py:175-186).  Inputs reach the workers through fork."""
    import os
    from multiprocessing import get_context

    workers = workers or os.cpu_count() or 1
    l1, l2, l3 = (np.asarray(a, np.int64) for a in (l1, l2, l3))
    _SHARED.update(q=q, qt=qt, C=C, v=v, wr2=wr2, entries=entries, alpha=alpha, l_min=l_min,
                   l1=l1, l2=l2, l3=l3, W=np.asarray(W, np.float64))
    try:
        bounds = np.linspace(0, l1.size, workers + 1).astype(np.int64)
        jobs = [(int(a), int(b), h2_mode, block) for a, b in zip(bounds[:-1], bounds[1:]) if b > a]
        if len(jobs) <= 1:
            parts = [_nonsep_job(j) for j in jobs]
        else:
            with get_context("fork").Pool(len(jobs)) as pool:
                parts = pool.map(_nonsep_job, jobs)
    finally:
        _SHARED.clear()
    out = np.zeros(entries.shape[0])
    for p_ in parts:
        out += p_
    return out
