"""Drop-in replacement for `cmbproj.gamma3d_matrix` (engine3d.py:156-186).

    gamma3d_matrix(tables, mapping, grid, h2_mode="gosper", integrator="trap", block=64,
                   workers=1, domain=None, *, device=None, devices=None) -> GammaMatrix

Same signature, argument meaning, errors and `meta` keys as the reference; a user switches
by rebinding the name (harness.py:21 imports it at module level, which is how the
reference's own tests swap engines, test_harness.py:278-279) — see INTEGRATION.md.

Differences that do not change results:
  * `block` and `workers` are validated and recorded in `meta` like the reference does, but
    the device path has its own tiling; the reference's `workers` fork pool becomes the
    visible GPUs (`devices`, one l2-slab shard per GPU, partials merged in order), or the
    ranks of `paper_1503_08809_b200.dist` under torchrun.
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

__all__ = ["gamma3d_matrix", "resolve_devices", "DomainRange", "DEFAULT_BLOCK", "domain_count",
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


def check_shapes(q, qt, C, v, wr2, l_min: int, l_max: int) -> None:
    """Shape agreement of the host arrays handed to the C-ABI (which reads p*L, p*Nx*L, L and
    Nx doubles through raw pointers).  The reference fails the same inputs with a ValueError
    from its einsum (engine3d.py:117) or its BasisTables validation (basis.py:232-246)."""
    L = int(l_max) - int(l_min) + 1
    if q.ndim != 2 or q.shape[1] != L:
        raise ValueError(f"q must have shape (p, {L}), got {q.shape}")
    if qt.ndim != 3 or qt.shape[0] != q.shape[0] or qt.shape[2] != L:
        raise ValueError(f"q_tilde must have shape ({q.shape[0]}, Nx, {L}), got {qt.shape}")
    if C.shape != (L,) or v.shape != (L,):
        raise ValueError(f"C and v must have shape ({L},)")
    if wr2.shape != (qt.shape[1],):
        raise ValueError(f"radial grid has {wr2.size} points but q_tilde has "
                         f"{qt.shape[1]} (n_radial)")


def _meta_dict(tables, grid, mapping, integrator, h2_mode, block, workers, ft, fg, fm):
    """Provenance keys of engine3d.py:139-153,172-174; ft/fg/fm = the tables / grid / mapping
    fingerprints (hashed on the `_FP_POOL` thread beside the GPU call by every drop-in)."""
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


def resolve_devices(device=None, devices=None) -> list[int]:
    """Devices a one-shot call shards over, in order of precedence:
    `devices` (sequence) > `device` (int) > env MG_DEVICES ("0,1,2,3") > under torchrun
    (WORLD_SIZE > 1) the rank's own LOCAL_RANK > every visible device.  Entries may repeat
    (two shards on one GPU run one after the other)."""
    import os
    if devices is not None:
        out = [int(d) for d in devices]
    elif device is not None:
        out = [int(device)]
    elif os.environ.get("MG_DEVICES"):
        out = [int(d) for d in os.environ["MG_DEVICES"].split(",") if d.strip()]
    elif int(os.environ.get("WORLD_SIZE", "1")) > 1:
        out = [int(os.environ.get("LOCAL_RANK", "0"))]
    else:
        out = list(range(max(1, nat.lib().mg_device_count())))
    if not out or len(out) > 64:
        raise ValueError("need between 1 and 64 devices")
    return out


def gamma3d_matrix(tables, mapping, grid, h2_mode: str = "gosper", integrator: str = "trap",
                   block: int = DEFAULT_BLOCK, workers: int = 1, domain=None, *,
                   device: int | None = None, devices=None) -> GammaMatrix:
    """Γ[n, n'] = Σ_t zm_t P[n,t] X[n',t] on the GPU (see module docstring).

    `device` / `devices` choose the GPU(s) (see `resolve_devices`; default: every visible
    GPU).  With several devices the domain is cut into l2 slabs of equal modelled cost, one
    per device, and the partial Γ's are summed in slab order — the reference's fork pool +
    merge_partials (engine3d.py:175-186) with GPUs for workers, inside the unchanged call.
    `meta["devices"]` records the list."""
    if block < 1:                                              # engine3d.py:168-169
        raise ValueError("block must be >= 1")
    if h2_mode not in nat.MG_H2:                               # engine3d.py:53
        raise ValueError(f"unknown h2_mode {h2_mode!r}")
    devs = np.ascontiguousarray(resolve_devices(device, devices), np.int32)
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
    check_shapes(q, qt, C, v, wr2, l_min, l_max)
    # The sha256 fingerprints of the inputs (meta, engine3d.py:139-153) cost ~0.25 s for a
    # config-1 q̃; hashlib and the ctypes call both release the GIL, so they overlap.
    fp = _FP_POOL.submit(lambda: (tables.fingerprint(), grid.fingerprint(),
                                  mapping.fingerprint()))

    def meta():
        m = _meta_dict(tables, grid, mapping, integrator, h2_mode, block, workers, *fp.result())
        m["devices"] = devs.tolist()
        return m

    out = np.zeros((n, n))
    lib = nat.lib()
    common = (nat.ptr(q), nat.ptr(qt), nat.ptr(C), nat.ptr(v), nat.ptr(wr2), nat.ptr(entries),
              p, nx, n, l_min, l_max, nat.MG_H2[h2_mode])
    shards = (int(devs.size), nat.ptr(devs))
    rng = _as_range(domain, l_min, l_max)
    if rng is None:
        l1 = np.ascontiguousarray(np.asarray(domain.l1), np.int32)
        l2 = np.ascontiguousarray(np.asarray(domain.l2), np.int32)
        l3 = np.ascontiguousarray(np.asarray(domain.l3), np.int32)
        rng = _detect_contiguous(l1, l2, l3, l_min, l_max)
        if rng is None:
            nat.check(lib.mg_gamma_sep_triples(*common, nat.ptr(l1), nat.ptr(l2), nat.ptr(l3),
                                               int(l1.size), *shards, nat.ptr(out)))
            return GammaMatrix(out, meta())
    begin, end = rng
    if end > begin:
        nat.check(lib.mg_gamma_sep(*common, int(begin), int(end), *shards, nat.ptr(out)))
    return GammaMatrix(out, meta())


def _detect_contiguous(l1, l2, l3, l_min, l_max):
    """(b, e) if the int32 triple arrays are exactly flat range [b, e) of the enumeration
    (one host-side O(n) walk in the C library, no device enumeration), else None."""
    b = np.zeros(1, np.int64)
    nat.check(nat.lib().mg_domain_match_range(int(l_min), int(l_max), nat.ptr(l1), nat.ptr(l2),
                                              nat.ptr(l3), int(l1.size), nat.ptr(b)))
    return None if b[0] < 0 else (int(b[0]), int(b[0]) + int(l1.size))
