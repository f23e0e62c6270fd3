"""Input types of the Γ projection — host-side mirror of the reference's `cmbproj.basis`.

These carry the same attribute names and validation as the reference so that the drop-in
`gamma3d_matrix` accepts either the reference's objects or these (duck typing on
`.q/.q_tilde/.C/.v/.l_min/.l_max`, `.entries/.n_max`, `.r`, `.fingerprint()`).

Reference interfaces mirrored (file:line under /root/reference/pkg/src/cmbproj/):
  ModeMapping           basis.py:57-94   (validation :64-74, fingerprint :93-94)
  default_mode_mapping  basis.py:97-106  (k-major order: k, then j<=k, then i<=j)
  RadialGrid            basis.py:173-190
  BasisTables           basis.py:219-262
  _shifted_legendre     basis.py:265-276 (the CMB-side q_i(l) of every BASELINE config)
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass

import numpy as np

__all__ = [
    "ModeMapping",
    "RadialGrid",
    "BasisTables",
    "default_mode_mapping",
    "shifted_legendre",
    "legendre_on_interval",
]


def _digest(*parts) -> str:
    """16-hex-digit sha256 over the concatenated byte strings (basis.py:50-54).  Arrays are
    hashed through a memoryview of their C-order buffer: the same bytes as `.tobytes()`
    without the copy (120 MB of q̃ at config 1)."""
    h = hashlib.sha256()
    for part in parts:
        if isinstance(part, np.ndarray):
            part = memoryview(np.ascontiguousarray(part)).cast("B")
        h.update(part)
    return h.hexdigest()[:16]


@dataclass(frozen=True)
class ModeMapping:
    """Flat mode index n -> ordered 1D-basis triple (i, j, k), i <= j <= k < p_max."""

    entries: np.ndarray
    p_max: int

    def __post_init__(self):
        e = np.asarray(self.entries, dtype=np.int64).reshape(-1, 3)
        object.__setattr__(self, "entries", e)
        if e.shape[0] == 0:
            raise ValueError("mode mapping must contain at least one entry")
        if (e < 0).any() or (e >= self.p_max).any():
            raise ValueError("mapping indices must lie in [0, p_max)")
        if (e[:, 0] > e[:, 1]).any() or (e[:, 1] > e[:, 2]).any():
            raise ValueError("mapping triples must satisfy i <= j <= k")
        if np.unique(e, axis=0).shape[0] != e.shape[0]:
            raise ValueError("mapping contains duplicate triples")

    @property
    def n_max(self) -> int:
        return int(self.entries.shape[0])

    def triple(self, n: int) -> tuple[int, int, int]:
        a, b, c = (int(t) for t in self.entries[n])
        return a, b, c

    def index_of(self, triple) -> int:
        hit = np.flatnonzero((self.entries == np.asarray(triple, dtype=np.int64)).all(1))
        if hit.size == 0:
            raise KeyError(f"triple {tuple(triple)!r} not in mapping")
        return int(hit[0])

    def fingerprint(self) -> str:
        return _digest(np.int64(self.p_max).tobytes(), self.entries)


def default_mode_mapping(p_max: int) -> ModeMapping:
    """Every i <= j <= k < p_max, k slowest, i fastest; n_max = C(p_max + 2, 3)."""
    if p_max < 1:
        raise ValueError("p_max must be >= 1")
    rows = [(i, j, k) for k in range(p_max) for j in range(k + 1) for i in range(j + 1)]
    return ModeMapping(np.asarray(rows, dtype=np.int64), p_max)


@dataclass(frozen=True)
class RadialGrid:
    """Strictly increasing, non-negative radial (x) samples."""

    r: np.ndarray
    zone_bounds: tuple = (0.0, 0.0)

    def __post_init__(self):
        r = np.asarray(self.r, dtype=np.float64)
        object.__setattr__(self, "r", r)
        if r.ndim != 1 or r.size == 0:
            raise ValueError("radial samples must be a non-empty 1D array")
        if r[0] < 0 or (np.diff(r) <= 0).any():
            raise ValueError("radial samples must be >= 0 and increasing")

    def __len__(self) -> int:
        return int(self.r.size)

    def fingerprint(self) -> str:
        return _digest(self.r)


@dataclass(frozen=True)
class BasisTables:
    """q[i, l-l_min], q_tilde[i, x, l-l_min], C[l-l_min], v[l-l_min] (all float64)."""

    q: np.ndarray
    q_tilde: np.ndarray
    C: np.ndarray
    v: np.ndarray
    l_min: int
    l_max: int

    def __post_init__(self):
        for name in ("q", "q_tilde", "C", "v"):
            arr = np.asarray(getattr(self, name), dtype=np.float64)
            object.__setattr__(self, name, arr)
            if not np.isfinite(arr).all():
                raise ValueError(f"table {name} contains non-finite values")
        n_l = self.l_max - self.l_min + 1
        ok = (self.q.ndim == 2 and self.q.shape[1] == n_l and self.q_tilde.ndim == 3
              and self.q_tilde.shape[2] == n_l and self.q_tilde.shape[0] == self.q.shape[0]
              and self.C.shape == (n_l,) and self.v.shape == (n_l,))
        if not ok:
            raise ValueError("table shapes inconsistent with l range")
        if (self.C <= 0).any():
            raise ValueError("power spectrum C_l must be strictly positive")

    @property
    def p_max(self) -> int:
        return int(self.q.shape[0])

    @property
    def n_radial(self) -> int:
        return int(self.q_tilde.shape[1])

    def ells(self) -> np.ndarray:
        return np.arange(self.l_min, self.l_max + 1)

    def fingerprint(self) -> str:
        return _digest(self.q, self.q_tilde, self.C,
                       self.v.tobytes(), np.int64([self.l_min, self.l_max]).tobytes())


def legendre_on_interval(p_max: int, t: np.ndarray, lo: float, span: float) -> np.ndarray:
    """P_0..P_{p_max-1} at u = 2 (t - lo) / span - 1, by the Bonnet recurrence in the
    operation order of basis.py:267-276 (so the result is bit-identical to the reference's
    `_shifted_legendre` when t is the integer l grid and span = max(l_max - l_min, 1))."""
    t = np.asarray(t, dtype=np.float64)
    u = 2.0 * (t - lo) / span - 1.0
    out = np.empty((p_max, t.size))
    out[0] = 1.0
    if p_max > 1:
        out[1] = u
    for i in range(1, p_max - 1):
        out[i + 1] = ((2 * i + 1) * u * out[i] - i * out[i - 1]) / (i + 1)
    return out


def shifted_legendre(p_max: int, l_min: int, l_max: int) -> np.ndarray:
    """CMB-side basis q_i(l), l = l_min..l_max (basis.py:265-276)."""
    ells = np.arange(l_min, l_max + 1, dtype=np.float64)
    return legendre_on_interval(p_max, ells, l_min, max(l_max - l_min, 1))
