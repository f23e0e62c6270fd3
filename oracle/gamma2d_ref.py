"""CPU ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

μ-quadrature ("separable", Modal2D) engine restated in NumPy:

    ptable   engine2d.py:62-95    P[a,b,x,m] = Σ_l lw_l q_a(l) q̃_b(x,l) P_l(μ_m), ascending l,
                                  Kahan-compensated, lw_l = (2l+1)/(v_l sqrt C_l) (:44-47)
    gamma2d  engine2d.py:101-129  per cell: permanent of the 3 x 3 block P[rows(n), cols(n')],
                                  μ rule first, then Σ_x w_x r_x² (·) / (48π)

Pinned by tests/test_oracle_golden.py::TestGamma2DPin against tables and matrices written by
the unmodified reference (tests/golden/io2d.npz): the P table bit for bit, Γ2d to rounding.
"""

from __future__ import annotations

import numpy as np


def l_weight(C, v, l_min, l_max):
    ells = np.arange(l_min, l_max + 1).astype(np.float64)
    return (2.0 * ells + 1.0) / (v * np.sqrt(C))


def ptable(q, qt, C, v, l_min, l_max, legendre):
    """legendre[l, m] for l = 0..l_max (rows below l_min unused)."""
    lw = l_weight(C, v, l_min, l_max)
    p, nx, L = qt.shape
    nmu = legendre.shape[1]
    acc = np.zeros((p, p, nx, nmu))
    comp = np.zeros_like(acc)
    for li in range(L):
        a = (lw[li] * q[:, li])[:, None, None] * qt[None, :, :, li]        # [a, b, x]
        term = a[..., None] * legendre[l_min + li][None, None, None, :]
        y = term - comp
        t = acc + y
        comp = (t - acc) - y
        acc = t
    return acc


def gamma2d(P, entries, mu_w, wr2):
    """wr2[x] = w_x r_x² (the radial rule's weights times r²)."""
    n = entries.shape[0]
    out = np.zeros((n, n))
    e = np.asarray(entries)
    for i in range(n):
        r = e[i]
        # m[a][b]: [n', x, μ] blocks of the rows this mode selects
        m = [[P[r[a], e[:, b]] for b in range(3)] for a in range(3)]
        per = (m[0][0] * m[1][1] * m[2][2] + m[0][0] * m[1][2] * m[2][1]
               + m[0][1] * m[1][0] * m[2][2] + m[0][1] * m[1][2] * m[2][0]
               + m[0][2] * m[1][0] * m[2][1] + m[0][2] * m[1][1] * m[2][0])
        out[i] = (per @ mu_w) @ wr2 / (48.0 * np.pi)
    return out
