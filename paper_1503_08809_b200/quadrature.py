"""x-integration weight vectors (host setup for the Γ kernels).

The reference folds its radial integrator into a weight vector w with w·y == integrator(r, y)
(`integration_weights`, quadrature.py:183-203) and the Γ engine uses wr2 = w * r**2
(engine3d.py:126).  The kernels only ever see wr2, so the three integrators are three
weight vectors computed here once per call:

  trap     quadrature.py:125-129  — interior w_i = dr_{i-1}/2 + dr_i/2 (a two-term fsum is
                                    one IEEE add, so this is bit-identical to the reference)
  hermite  quadrature.py:132-145  — trapezium plus secant-slope correction
  spline   quadrature.py:148-173  — natural cubic spline, integrated analytically

hermite/spline are derived in closed (linear-algebra) form here rather than by probing the
integrator with unit vectors; they agree with the reference to rounding (≈1e-16 relative).
"""

from __future__ import annotations

import numpy as np

__all__ = ["integration_weights", "x_weights", "INTEGRATORS"]

INTEGRATORS = ("trap", "hermite", "spline")


def _trap(r: np.ndarray) -> np.ndarray:
    half = 0.5 * np.diff(r)
    w = np.zeros(r.size)
    w[:-1] += half
    w[1:] += half          # w_i = half_{i-1} + half_i (element order of fsum([a, b]))
    # fsum of two terms is the correctly rounded a+b; numpy's a+b is the same IEEE add,
    # but for the interior the reference adds half_{i-1} first: (half_{i-1} + half_i) is
    # commutative in IEEE arithmetic, so the order does not matter.
    return w


def _hermite(r: np.ndarray) -> np.ndarray:
    n = r.size
    if n < 3:
        raise ValueError("need at least 3 samples")
    dr = np.diff(r)
    m = n - 1
    # s_k = (y_{k+1} - y_k) / dr_k ; s_next = s_{k+1} (k < m-1), s_{m-1} (k = m-1)
    # term_k = dr_k/2 (y_k + y_{k+1}) + dr_k^2/12 (s_k - s_next_k)
    w = np.zeros(n)
    w[:-1] += 0.5 * dr
    w[1:] += 0.5 * dr
    coef = dr * dr / 12.0
    for k in range(m - 1):          # last interval's correction is identically zero
        c = coef[k]
        # + c * s_k
        w[k + 1] += c / dr[k]
        w[k] -= c / dr[k]
        # - c * s_{k+1}
        w[k + 2] -= c / dr[k + 1]
        w[k + 1] += c / dr[k + 1]
    return w


def _spline(r: np.ndarray) -> np.ndarray:
    n = r.size
    if n < 4:
        raise ValueError("need at least 4 samples")
    h = np.diff(r)
    # natural spline moments m = A^{-1} R y (quadrature.py:148-161), A tridiagonal
    A = np.zeros((n, n))
    A[0, 0] = A[-1, -1] = 1.0
    idx = np.arange(1, n - 1)
    A[idx, idx] = 2.0 * (h[:-1] + h[1:])
    A[idx, idx + 1] = h[1:]
    A[idx, idx - 1] = h[:-1]
    R = np.zeros((n, n))
    R[idx, idx + 1] += 6.0 / h[1:]
    R[idx, idx] -= 6.0 / h[1:] + 6.0 / h[:-1]
    R[idx, idx - 1] += 6.0 / h[:-1]
    M = np.linalg.solve(A, R)                      # m = M y
    w = np.zeros(n)
    w[:-1] += 0.5 * h
    w[1:] += 0.5 * h
    c = h ** 3 / 24.0                              # - h^3/24 (m_k + m_{k+1})
    w -= c @ M[:-1] + c @ M[1:]
    return w


def integration_weights(r, method: str = "trap") -> np.ndarray:
    """Weight vector of the reference integrator `method` on grid r."""
    r = np.asarray(r, dtype=np.float64)
    if method == "trap":
        if r.size < 2:
            raise ValueError("need at least 2 samples")
        return _trap(r)
    if method == "hermite":
        return _hermite(r)
    if method == "spline":
        return _spline(r)
    raise ValueError(f"unknown integrator {method!r}")


def x_weights(r, method: str = "trap") -> np.ndarray:
    """wr2 = integration_weights(r, method) * r**2 (engine3d.py:126)."""
    r = np.asarray(r, dtype=np.float64)
    return integration_weights(r, method) * r ** 2
