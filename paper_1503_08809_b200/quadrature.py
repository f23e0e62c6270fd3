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


# ------------------------------------------------------------------------------------------
# Gauss-Legendre rule and Legendre table for the 2D (mu-quadrature) engine
# (quadrature.py:38-112 of the reference; restated with the same Newton scheme so the nodes
#  and weights agree with the reference to the last bit or so)
# ------------------------------------------------------------------------------------------

class QuadratureRule:
    """Gauss-Legendre nodes and weights on [-1, 1]."""

    def __init__(self, nodes, weights):
        self.nodes = np.asarray(nodes, dtype=np.float64)
        self.weights = np.asarray(weights, dtype=np.float64)

    @property
    def n(self) -> int:
        return int(self.nodes.size)


def _legendre_pd(n: int, x: np.ndarray):
    p0, p1 = np.ones_like(x), x.copy()
    if n == 0:
        return p0, np.zeros_like(x)
    for k in range(1, n):
        p0, p1 = p1, ((2 * k + 1) * x * p1 - k * p0) / (k + 1)
    return p1, n * (x * p1 - p0) / (x * x - 1.0)


def gauss_legendre(n: int) -> QuadratureRule:
    """n-node rule: Newton on P_n from Chebyshev-angle guesses, one clean-up step, exact
    symmetry enforced (reference quadrature.py:68-98)."""
    if n < 1:
        raise ValueError("n must be >= 1")
    if n == 1:
        return QuadratureRule(np.zeros(1), np.full(1, 2.0))
    b = np.arange(n, dtype=np.float64)
    x = np.cos(np.pi * (4 * b + 3) / (4 * n + 2))
    for _ in range(100):
        p, dp = _legendre_pd(n, x)
        dx = p / dp
        x = x - dx
        if np.max(np.abs(dx)) < 1e-15:
            p, dp = _legendre_pd(n, x)
            x = x - p / dp
            break
    else:
        raise RuntimeError(f"Gauss-Legendre Newton iteration failed at n={n}")
    x = np.sort(x)
    x = 0.5 * (x - x[::-1])
    _, dp = _legendre_pd(n, x)
    w = 2.0 / ((1.0 - x * x) * dp * dp)
    return QuadratureRule(x, 0.5 * (w + w[::-1]))


def legendre_table(l_max: int, rule) -> np.ndarray:
    """P_l at every node, [l_max+1, n], upward recurrence (reference quadrature.py:101-112)."""
    if l_max < 0:
        raise ValueError("l_max must be >= 0")
    x = np.asarray(rule.nodes, dtype=np.float64)
    t = np.empty((l_max + 1, x.size))
    t[0] = 1.0
    if l_max >= 1:
        t[1] = x
    for l in range(1, l_max):
        t[l + 1] = ((2 * l + 1) * x * t[l] - l * t[l - 1]) / (l + 1)
    return t


def default_mu_points(l_max: int) -> int:
    """Exact for the degree-3 l_max integrand (reference engine2d.py:40-41)."""
    return -(-(3 * l_max + 1) // 2) + 2
