"""CPU ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Stage 1 (absent from the reference: SPEC.md:14,224 put transfer functions and Bessel
functions out of scope) restated from PAPER.md:700 and BASELINE.json config 0:

    Δ_l(k)   = j_l(14000 k) exp(-(k/0.1)^2) (1 + 0.01 ε_{l,k})
    C_l      = Σ_k wk Δ_l(k)^2 / k
    q̃_p(x,l) = Σ_k wk k^2 q_p(k) Δ_l(k) j_l(k x)

The Bessel oracle is scipy.special.spherical_jn (third-party, scipy 1.18.1 in this image;
the reference pins only scipy>=1.9, pyproject.toml:12): upward recurrence for l < z and
AMOS J_{l+1/2} for l >= z.  No reference test pins this stage — parity unpinned.
"""

from __future__ import annotations

import numpy as np
from scipy.special import spherical_jn

X_DELTA = 14000.0
K_DAMP = 0.1
EPS_AMP = 0.01


def delta_table(k, eps, l_min, l_max):
    """Δ[l-l_min, k]."""
    ells = np.arange(l_min, l_max + 1)
    J = spherical_jn(ells[:, None], X_DELTA * k[None, :])
    return J * np.exp(-(k / K_DAMP) ** 2)[None, :] * (1.0 + EPS_AMP * eps)


def c_ell(delta, k, wk):
    """C[l-l_min] = Σ_k wk Δ^2 / k."""
    return (delta ** 2) @ (wk / k)


def qtilde(k, wk, x, qk, delta, l_min, l_max, ells=None):
    """q̃[p, x, l-l_min] (all l, or only the listed `ells`, others left 0)."""
    p = qk.shape[0]
    out = np.zeros((p, x.size, l_max - l_min + 1))
    b = qk * (wk * k * k)[None, :]                      # [p, Nk]
    kx = np.outer(k, x)                                 # [Nk, Nx]
    todo = range(l_min, l_max + 1) if ells is None else ells
    for l in todo:
        J = spherical_jn(int(l), kx)                    # [Nk, Nx]
        out[:, :, l - l_min] = (b * delta[l - l_min][None, :]) @ J
    return out


def build(hi, ells=None):
    """(C, q̃, Δ) for a paper_1503_08809_b200.configs.HostInputs."""
    d = delta_table(hi.k, hi.eps, hi.l_min, hi.l_max)
    C = c_ell(d, hi.k, hi.wk)
    qt = qtilde(hi.k, hi.wk, hi.x, hi.qk, d, hi.l_min, hi.l_max, ells)
    return C, qt, d
