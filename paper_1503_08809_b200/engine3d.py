"""Drop-in replacement for `cmbproj.gamma3d_matrix` (engine3d.py:156-186).

    gamma3d_matrix(tables, mapping, grid, h2_mode="gosper", integrator="trap", block=64,
                   workers=1, domain=None, *, device=None) -> GammaMatrix

Same signature, argument meaning, errors and `meta` keys as the reference; a user switches
by rebinding the name (harness.py:21 imports it at module level, which is how the
reference's own tests swap engines, test_harness.py:278-279) — see INTEGRATION.md.

Differences that do not change results:
  * `block` and `workers` are validated and recorded in `meta` like the reference does, but
    the device path has its own tiling; `workers` CPU processes become one GPU (or the
    ranks of `paper_1503_08809_b200.dist`).
  * `domain` may be the reference's TriangularDomain (or any object with l1/l2/l3/count), a
    `DomainRange` (a contiguous flat range, never materialised), or None (whole domain).
    A domain that is a contiguous flat range of the full enumeration runs through the
    range path; any other triple list runs through the explicit-triple path.
"""

from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import _native as nat
from .gamma import GammaMatrix
from .quadrature import x_weights

__all__ = ["gamma3d_matrix", "DomainRange", "DEFAULT_BLOCK", "domain_count",
           "domain_triples", "triple_weights"]

DEFAULT_BLOCK = 64
_FP_POOL = ThreadPoolExecutor(max_workers=1, thread_name_prefix="mg-fingerprint")


class DomainRange:
    """Contiguous flat range [begin, end) of the reference enumeration (geometry.py:161-171),
    without materialising the triples."""

    def __init__(self, l_min: int, l_max: int, begin: int = 0, end: int | None = None):
        total = domain_count(l_min, l_max)
        self.l_min, self.l_max = int(l_min), int(l_max)
        self.begin = int(begin)
        self.end = total if end is None else int(end)
        if not 0 <= self.begin <= self.end <= total:
            raise ValueError("invalid flat range")
        self.count = self.end - self.begin

    def __len__(self) -> int:
        return self.count

    def arrays(self, device: int = 0):
        return domain_triples(self.l_min, self.l_max, self.begin, self.end, device)

    @property
    def l1(self):
        return self.arrays()[0]

    @property
    def l2(self):
        return self.arrays()[1]

    @property
    def l3(self):
        return self.arrays()[2]


def domain_count(l_min: int, l_max: int) -> int:
    """Number of ordered valid triples (host arithmetic, geometry.py:161-171)."""
    c = np.zeros(1, np.int64)
    nat.check(nat.lib().mg_domain_count(int(l_min), int(l_max), nat.ptr(c), None))
    return int(c[0])


def domain_triples(l_min: int, l_max: int, begin: int = 0, end: int | None = None,
                   device: int = 0):
    """(l1, l2, l3) int64 arrays of flat indices [begin, end), enumerated on the GPU."""
    if end is None:
        end = domain_count(l_min, l_max)
    n = max(int(end) - int(begin), 0)
    out = [np.zeros(n, np.int32) for _ in range(3)]
    if n:
        nat.check(nat.lib().mg_domain_triples(int(l_min), int(l_max), int(begin), int(end),
                                              *(nat.ptr(a) for a in out), int(device)))
    return tuple(a.astype(np.int64) for a in out)


def triple_weights(C, v, l_min: int, l_max: int, begin: int = 0, end: int | None = None,
                   h2_mode: str = "gosper", device: int = 0) -> np.ndarray:
    """zm = _triple_z * permutation_multiplicity for flat [begin, end) on the GPU
    (engine3d.py:41-53,133-134); bit-identical to NumPy for h2_mode="gosper"."""
    if h2_mode not in nat.MG_H2:
        raise ValueError(f"unknown h2_mode {h2_mode!r}")
    if end is None:
        end = domain_count(l_min, l_max)
    C = np.ascontiguousarray(C, np.float64)
    v = np.ascontiguousarray(v, np.float64)
    out = np.zeros(max(int(end) - int(begin), 0))
    if out.size:
        nat.check(nat.lib().mg_weights(int(l_min), int(l_max), nat.ptr(C), nat.ptr(v),
                                       nat.MG_H2[h2_mode], int(begin), int(end), nat.ptr(out),
                                       int(device)))
    return out


def _base_meta(tables, grid, mapping, integrator, h2_mode, block, workers):
    """Provenance keys of engine3d.py:139-153,172-174."""
    return _meta_dict(tables, grid, mapping, integrator, h2_mode, block, workers,
                      tables.fingerprint(), grid.fingerprint(), mapping.fingerprint())


def _meta_dict(tables, grid, mapping, integrator, h2_mode, block, workers, ft, fg, fm):
    return {
        "engine": "modal3d",
        "l_min": tables.l_min,
        "l_max": tables.l_max,
        "p_max": tables.p_max,
        "n_max": mapping.n_max,
        "integrator": integrator,
        "tables": ft,
        "grid": fg,
        "mapping": fm,
        "h2_mode": h2_mode,
        "block": block,
        "workers": workers,
    }


def _as_range(domain, l_min, l_max):
    """(begin, end) if `domain` is a contiguous flat range of the full enumeration."""
    if domain is None:
        return 0, domain_count(l_min, l_max)
    if isinstance(domain, DomainRange):
        if (domain.l_min, domain.l_max) != (l_min, l_max):
            return None
        return domain.begin, domain.end
    return None


def _flat_index_of_first(l1, l2, l3, l_min, l_max):
    """Flat index of triple (l1,l2,l3) in the reference order (for range detection)."""
    n = 0
    for a in range(l_min, l1):
        for b in range(a, l_max + 1):
            start = b if a % 2 == 0 else b + 1
            stop = min(a + b, l_max)
            n += 0 if start > stop else (stop - start) // 2 + 1
    for b in range(l1, l2):
        start = b if l1 % 2 == 0 else b + 1
        stop = min(l1 + b, l_max)
        n += 0 if start > stop else (stop - start) // 2 + 1
    start = l2 if l1 % 2 == 0 else l2 + 1
    return n + (l3 - start) // 2


def gamma3d_matrix(tables, mapping, grid, h2_mode: str = "gosper", integrator: str = "trap",
                   block: int = DEFAULT_BLOCK, workers: int = 1, domain=None, *,
                   device: int | None = None) -> GammaMatrix:
    """Γ[n, n'] = Σ_t zm_t P[n,t] X[n',t] on the GPU (see module docstring)."""
    if block < 1:                                              # engine3d.py:168-169
        raise ValueError("block must be >= 1")
    if h2_mode not in nat.MG_H2:                               # engine3d.py:53
        raise ValueError(f"unknown h2_mode {h2_mode!r}")
    if device is None:
        device = 0
    q = np.ascontiguousarray(tables.q, np.float64)
    qt = np.ascontiguousarray(tables.q_tilde, np.float64)
    C = np.ascontiguousarray(tables.C, np.float64)
    v = np.ascontiguousarray(tables.v, np.float64)
    if np.any(C <= 0):
        raise ValueError("power spectrum C_l must be strictly positive")
    entries = np.ascontiguousarray(mapping.entries, np.int64)
    wr2 = np.ascontiguousarray(x_weights(grid.r, integrator), np.float64)
    p, nx, n = q.shape[0], qt.shape[1], entries.shape[0]
    l_min, l_max = int(tables.l_min), int(tables.l_max)
    # The sha256 fingerprints of the inputs (meta, engine3d.py:139-153) cost ~0.25 s for a
    # config-1 q̃; hashlib and the ctypes call both release the GIL, so they overlap.
    fp = _FP_POOL.submit(lambda: (tables.fingerprint(), grid.fingerprint(),
                                  mapping.fingerprint()))

    def meta():
        return _meta_dict(tables, grid, mapping, integrator, h2_mode, block, workers,
                          *fp.result())

    out = np.zeros((n, n))
    lib = nat.lib()
    common = (nat.ptr(q), nat.ptr(qt), nat.ptr(C), nat.ptr(v), nat.ptr(wr2), nat.ptr(entries),
              p, nx, n, l_min, l_max, nat.MG_H2[h2_mode])
    rng = _as_range(domain, l_min, l_max)
    if rng is None:
        l1 = np.ascontiguousarray(np.asarray(domain.l1), np.int32)
        l2 = np.ascontiguousarray(np.asarray(domain.l2), np.int32)
        l3 = np.ascontiguousarray(np.asarray(domain.l3), np.int32)
        rng = _detect_contiguous(l1, l2, l3, l_min, l_max)
        if rng is None:
            nat.check(lib.mg_gamma_sep_triples(*common, nat.ptr(l1), nat.ptr(l2), nat.ptr(l3),
                                               int(l1.size), int(device), nat.ptr(out)))
            return GammaMatrix(out, meta())
    begin, end = rng
    if end > begin:
        nat.check(lib.mg_gamma_sep(*common, int(begin), int(end), int(device), nat.ptr(out)))
    return GammaMatrix(out, meta())


def _detect_contiguous(l1, l2, l3, l_min, l_max):
    """If the triple arrays are exactly flat range [b, e) of the enumeration, return it."""
    n = l1.size
    if n == 0:
        return (0, 0)
    b = _flat_index_of_first(int(l1[0]), int(l2[0]), int(l3[0]), l_min, l_max)
    total = domain_count(l_min, l_max)
    if b + n > total:
        return None
    r1, r2, r3 = domain_triples(l_min, l_max, b, b + n)
    if np.array_equal(r1, l1) and np.array_equal(r2, l2) and np.array_equal(r3, l3):
        return (b, b + n)
    return None
