"""The five BASELINE.json workloads as seeded synthetic inputs.

Host-side, deterministic setup only: grids, quadrature weights, the seeded ε (and α for
config 3), Legendre bases and the mode mapping.  The Bessel-dependent inputs — Δ_l(k), C_l
and q̃ — are built on the GPU by `qtilde.build_qtilde` (stage 1).

Frozen choices (BASELINE.json leaves them open; recorded in DESIGN.md §5):
  x  = linspace(x0, x1, Nx), wr2 = trap weights(x) * x^2           (engine3d.py:126)
  k  = linspace(kmin, kmax, Nk), wk = trap weights(k)               (quadrature.py:183-203)
  ε  = default_rng(seed).standard_normal((L, Nk)), rows l = l_min..l_max ascending
  α  = (config 3 only) next draw of the same generator: standard_normal(n)/(1+i+j+k)
  Δ_l(k) = j_l(14000 k) exp(-(k/0.1)^2) (1 + 0.01 ε_{l,k});  C_l = Σ_k wk Δ_l(k)^2 / k
  v  = (2l+1)^(1/6)                                                  (basis.py:293)
  q(l) = shifted Legendre on [l_min, l_max]                          (basis.py:265-276)
  q_p(k) = P_p(2(k-kmin)/(kmax-kmin) - 1), same recurrence
  mapping = default_mode_mapping(p)                                  (basis.py:97-106)
  config 3 l-grid: every l <= 50, then every 10th l up to 2000; volume weights = trapezium
  weights of the l-grid plus 1/2 at both ends (Euler-Maclaurin sum weights, exactly 1 on a
  step-1 grid); all-unit-weight triples keep exact parity, the others enter with factor 1/2
  and no parity cut.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .basis import default_mode_mapping, legendre_on_interval, shifted_legendre
from .quadrature import integration_weights

__all__ = ["ConfigSpec", "CONFIGS", "HostInputs", "host_inputs", "sparse_grid",
           "sparse_domain"]

X_DELTA = 14000.0
K_DAMP = 0.1
EPS_AMP = 0.01
L_MIN = 2


@dataclass(frozen=True)
class ConfigSpec:
    name: str
    l_max: int
    p: int
    n_k: int
    k_range: tuple
    n_x: int
    x_range: tuple
    seed: int
    sparse: bool = False


CONFIGS = {
    "c0": ConfigSpec("c0", 200, 6, 800, (1e-4, 0.2), 100, (13600.0, 14400.0), 0),
    "c1": ConfigSpec("c1", 2000, 15, 3000, (1e-4, 0.3), 500, (13500.0, 14500.0), 1),
    "c2": ConfigSpec("c2", 2500, 22, 4000, (1e-4, 0.2), 1000, (13600.0, 14400.0), 2),
    "c3": ConfigSpec("c3", 2000, 8, 2000, (1e-4, 0.2), 300, (13600.0, 14400.0), 3, True),
    "c4": ConfigSpec("c4", 3000, 30, 5000, (1e-4, 0.4), 2000, (13000.0, 15000.0), 4),
}


@dataclass
class HostInputs:
    spec: ConfigSpec
    l_min: int
    l_max: int
    k: np.ndarray        # [Nk]
    wk: np.ndarray       # [Nk]
    x: np.ndarray        # [Nx]
    wr2: np.ndarray      # [Nx]
    eps: np.ndarray      # [L, Nk]
    q: np.ndarray        # [p, L]
    qk: np.ndarray       # [p, Nk]
    v: np.ndarray        # [L]
    entries: np.ndarray  # [n, 3]
    alpha: np.ndarray | None = None


def host_inputs(spec: ConfigSpec | str, l_max: int | None = None) -> HostInputs:
    """Seeded host inputs of a config (optionally with a smaller l_max for tests)."""
    if isinstance(spec, str):
        spec = CONFIGS[spec]
    lmax = spec.l_max if l_max is None else l_max
    n_l = lmax - L_MIN + 1
    k = np.linspace(spec.k_range[0], spec.k_range[1], spec.n_k)
    wk = integration_weights(k, "trap")
    x = np.linspace(spec.x_range[0], spec.x_range[1], spec.n_x)
    wr2 = integration_weights(x, "trap") * x ** 2
    rng = np.random.default_rng(spec.seed)
    eps = rng.standard_normal((n_l, spec.n_k))
    mapping = default_mode_mapping(spec.p)
    alpha = None
    if spec.sparse:
        e = mapping.entries
        alpha = rng.standard_normal(e.shape[0]) / (1.0 + e.sum(axis=1))
    q = shifted_legendre(spec.p, L_MIN, lmax)
    qk = legendre_on_interval(spec.p, k, spec.k_range[0], spec.k_range[1] - spec.k_range[0])
    ells = np.arange(L_MIN, lmax + 1, dtype=np.float64)
    v = (2.0 * ells + 1.0) ** (1.0 / 6.0)
    return HostInputs(spec, L_MIN, lmax, k, wk, x, wr2, eps, q, qk, v, mapping.entries, alpha)


def sparse_grid(l_max: int = 2000, dense_to: int = 50, step: int = 10, l_min: int = L_MIN):
    """Config-3 l-grid and its 1D sum weights (see module docstring)."""
    dense = np.arange(l_min, min(dense_to, l_max) + 1)
    coarse = np.arange(dense_to + step, l_max + 1, step) if l_max > dense_to else []
    grid = np.concatenate([dense, np.asarray(coarse, dtype=np.int64)]).astype(np.int64)
    if grid[-1] != l_max:
        grid = np.append(grid, l_max)
    w = integration_weights(grid.astype(np.float64), "trap") if grid.size > 1 else np.ones(1)
    w = w.copy()
    w[0] += 0.5
    w[-1] += 0.5
    return grid, w


def sparse_domain(grid: np.ndarray, w1d: np.ndarray):
    """Ordered triples of grid points closing a triangle, with volume weights W.

    Triples whose three 1D weights are all exactly 1 lie in the step-1 region: they keep the
    exact even-parity cut and W = 1.  Every other triple represents a cell of dense triples of
    which half have even l1+l2+l3: it enters regardless of its own parity with
    W = w1 w2 w3 / 2.  On a step-1 grid this reduces to the reference's domain with W = 1.
    """
    g = np.asarray(grid, np.int64)
    unit = w1d == 1.0
    out1, out2, out3, ow = [], [], [], []
    n = g.size
    for a in range(n):
        for b in range(a, n):
            cmax = g[a] + g[b]
            c = np.arange(b, n)
            c = c[g[c] <= cmax]
            if c.size == 0:
                continue
            l3 = g[c]
            dense = unit[a] & unit[b] & unit[c]
            even = ((g[a] + g[b] + l3) % 2) == 0
            keep = np.where(dense, even, True)
            W = np.where(dense, 1.0, 0.5 * w1d[a] * w1d[b] * w1d[c])
            out1.append(np.full(keep.sum(), g[a]))
            out2.append(np.full(keep.sum(), g[b]))
            out3.append(l3[keep])
            ow.append(W[keep])
    return (np.concatenate(out1), np.concatenate(out2), np.concatenate(out3),
            np.concatenate(ow))
