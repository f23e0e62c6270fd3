"""CPU ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

NumPy restatement of the reference's direct Γ engine and of its weights, used as the
parity checker of the CUDA path and as the CPU baseline timed by bench.py.  Every function
names the reference lines it restates (paths under /root/reference/pkg/src/cmbproj/).
"""

from __future__ import annotations

import ctypes
import math
import os
from itertools import permutations
from multiprocessing import get_context

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_PERMS = tuple(permutations((0, 1, 2)))


# ----------------------------------------------------------------------------------------
# bit-exact C restatement of enumeration + Gosper weights (oracle/domain_ref.c)
# ----------------------------------------------------------------------------------------

def _clib():
    path = os.path.join(_HERE, "_build", "liboracle_domain.so")
    if not os.path.exists(path):
        import subprocess
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    lib = ctypes.CDLL(path)
    i64, i32p, f64p = ctypes.c_int64, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_double)
    lib.or_domain_count.restype = i64
    lib.or_domain_count.argtypes = [ctypes.c_int, ctypes.c_int]
    lib.or_domain_triples.restype = i64
    lib.or_domain_triples.argtypes = [ctypes.c_int, ctypes.c_int, i64, i64, i32p, i32p, i32p]
    lib.or_weights.restype = None
    lib.or_weights.argtypes = [ctypes.c_int, ctypes.c_int, i32p, i32p, i32p, f64p, f64p, f64p]
    lib.or_h2_gosper.restype = ctypes.c_double
    lib.or_h2_gosper.argtypes = [ctypes.c_int] * 3
    return lib


_LIB = None


def clib():
    global _LIB
    if _LIB is None:
        _LIB = _clib()
    return _LIB


def _p(a, t):
    return a.ctypes.data_as(ctypes.POINTER(t))


def domain_count(l_min: int, l_max: int) -> int:
    """len(enumerate_domain(l_min, l_max)) (geometry.py:153-180)."""
    return int(clib().or_domain_count(l_min, l_max))


def domain_triples(l_min: int, l_max: int, begin: int = 0, end: int | None = None):
    """(l1, l2, l3) int64 arrays of flat indices [begin, end) (geometry.py:161-171)."""
    if end is None:
        end = domain_count(l_min, l_max)
    n = max(end - begin, 0)
    a = np.zeros(n, np.int32)
    b = np.zeros(n, np.int32)
    c = np.zeros(n, np.int32)
    got = clib().or_domain_triples(l_min, l_max, begin, end, _p(a, ctypes.c_int32),
                                   _p(b, ctypes.c_int32), _p(c, ctypes.c_int32))
    assert got == n
    return a.astype(np.int64), b.astype(np.int64), c.astype(np.int64)


def zm_c(l_min, l1, l2, l3, C, v) -> np.ndarray:
    """z * multiplicity per triple via the C restatement (engine3d.py:133-134)."""
    l1 = np.ascontiguousarray(l1, np.int32)
    l2 = np.ascontiguousarray(l2, np.int32)
    l3 = np.ascontiguousarray(l3, np.int32)
    C = np.ascontiguousarray(C, np.float64)
    v = np.ascontiguousarray(v, np.float64)
    out = np.empty(l1.size)
    clib().or_weights(l_min, l1.size, _p(l1, ctypes.c_int32), _p(l2, ctypes.c_int32),
                      _p(l3, ctypes.c_int32), _p(C, ctypes.c_double), _p(v, ctypes.c_double),
                      _p(out, ctypes.c_double))
    return out


# ----------------------------------------------------------------------------------------
# NumPy restatement of the weights (same arithmetic as the reference, used by the port)
# ----------------------------------------------------------------------------------------

def multiplicity(l1, l2, l3) -> np.ndarray:
    """permutation_multiplicity (geometry.py:114-123)."""
    l1, l2, l3 = (np.asarray(a, np.int64) for a in (l1, l2, l3))
    return np.where(l1 == l3, 1, np.where((l1 == l2) | (l2 == l3), 3, 6))


def h2_gosper(l1, l2, l3) -> np.ndarray:
    """geometry.py:97-110."""
    a, b, c = (np.asarray(x, np.float64) for x in (l1, l2, l3))
    L = a + b + c
    La, Lb, Lc = L - 2 * a, L - 2 * b, L - 2 * c
    main = ((2 * a + 1) * (2 * b + 1) * (2 * c + 1) * (L + 1.0 / 3.0)
            / ((L + 1) * (La + 1.0 / 3.0) * (Lb + 1.0 / 3.0) * (Lc + 1.0 / 3.0)))
    root = np.sqrt((La + 1.0 / 6.0) * (Lb + 1.0 / 6.0) * (Lc + 1.0 / 6.0) / (L + 1.0 / 6.0))
    return main * root / (2.0 * np.pi ** 2)


_LF = np.zeros(1)


def _log_fact(n: int) -> np.ndarray:
    """log-factorial table grown like geometry.py:32-40."""
    global _LF
    if len(_LF) <= n:
        size = max(n + 1, 2 * len(_LF))
        t = np.zeros(size)
        t[1:] = np.cumsum(np.log(np.arange(1, size)))
        _LF = t
    return _LF


def h2_exact(l1, l2, l3) -> np.ndarray:
    """Racah closed form in the log-factorial domain (geometry.py:56-86); exactly 0 where
    the triangle or even-parity condition fails (theta_indicator gate, geometry.py:44-54,
    67-71)."""
    a, b, c = np.broadcast_arrays(*(np.atleast_1d(np.asarray(x, np.int64))
                                    for x in (l1, l2, l3)))
    L = a + b + c
    ok = (L % 2 == 0) & (c <= a + b) & (b <= a + c) & (a <= b + c)
    out = np.zeros(a.shape)
    if np.any(ok):
        a, b, c, L = a[ok], b[ok], c[ok], L[ok]
        g = L // 2
        lf = _log_fact(int(L.max()) + 1)
        log3j2 = (lf[L - 2 * a] + lf[L - 2 * b] + lf[L - 2 * c] - lf[L + 1]
                  + 2.0 * (lf[g] - lf[g - a] - lf[g - b] - lf[g - c]))
        pref = (2 * a + 1) * (2 * b + 1) * (2 * c + 1) / (4.0 * np.pi)
        out[ok] = pref * np.exp(log3j2)
    return out


def triple_zm(l_min, l1, l2, l3, C, v, h2_mode="gosper") -> np.ndarray:
    """_triple_z(...) * permutation_multiplicity(...) (engine3d.py:41-53,133-134;
    geometry.py:126-142)."""
    i1 = np.asarray(l1) - l_min
    i2 = np.asarray(l2) - l_min
    i3 = np.asarray(l3) - l_min
    denom = 36.0 * v[i1] * v[i2] * v[i3] * np.sqrt(C[i1] * C[i2] * C[i3])
    if h2_mode == "gosper":
        h2 = h2_gosper(l1, l2, l3)
    elif h2_mode == "exact":
        h2 = h2_exact(l1, l2, l3)
    else:
        raise ValueError(f"unknown h2_mode {h2_mode!r}")
    return (h2 / denom) * multiplicity(l1, l2, l3)


# ----------------------------------------------------------------------------------------
# Γ port: _block_accumulate / _sweep_chunk / gamma3d_matrix (engine3d.py:86-186)
# ----------------------------------------------------------------------------------------

def block_accumulate(gamma, q, qt, entries, wr2, i1, i2, i3, zm, cols=None):
    """engine3d.py:86-120 — gamma += P X^T for one block of triples.  `cols` (test speed-up
    at the largest configs) restricts X to a subset of the primordial modes: gamma is then
    [n, len(cols)] and equals the full Γ[:, cols] (column n' of Γ only needs X[n'])."""
    rows = (entries[:, 0], entries[:, 1], entries[:, 2])
    xe = entries if cols is None else entries[np.asarray(cols)]
    xcols = (xe[:, 0], xe[:, 1], xe[:, 2])
    q1, q2, q3 = q[:, i1], q[:, i2], q[:, i3]
    p_blk = np.zeros((entries.shape[0], i1.size))
    for a, b, c in _PERMS:
        p_blk += q1[rows[a]] * q2[rows[b]] * q3[rows[c]]
    t1, t2, t3 = qt[:, :, i1], qt[:, :, i2], qt[:, :, i3]
    f = np.zeros((xe.shape[0], qt.shape[1], i1.size))
    for a, b, c in _PERMS:
        f += t1[xcols[a]] * t2[xcols[b]] * t3[xcols[c]]
    x_blk = np.einsum("r,nrb->nb", wr2, f)
    x_blk *= zm
    gamma += p_blk @ x_blk.T


def sweep_triples(q, qt, C, v, wr2, entries, l_min, l1, l2, l3, block=64,
                  h2_mode="gosper", cols=None):
    """engine3d.py:123-136 over an explicit triple list."""
    n = entries.shape[0]
    gamma = np.zeros((n, n if cols is None else len(cols)))
    for b0 in range(0, l1.size, block):
        b1 = min(b0 + block, l1.size)
        a, b, c = l1[b0:b1], l2[b0:b1], l3[b0:b1]
        zm = triple_zm(l_min, a, b, c, C, v, h2_mode)
        block_accumulate(gamma, q, qt, entries, wr2, a - l_min, b - l_min, c - l_min, zm, cols)
    return gamma


_SHARED = {}


def _triples_job(args):
    lo, hi, block, h2_mode, cols = args
    d = _SHARED
    return sweep_triples(d["q"], d["qt"], d["C"], d["v"], d["wr2"], d["entries"], d["l_min"],
                         d["l1"][lo:hi], d["l2"][lo:hi], d["l3"][lo:hi], block, h2_mode, cols)


def sweep_triples_parallel(q, qt, C, v, wr2, entries, l_min, l1, l2, l3, workers=None,
                           block=64, h2_mode="gosper", cols=None):
    """sweep_triples over a fork pool (the reference's worker split, engine3d.py:175-186:
    contiguous chunks, partials summed in worker order).  The inputs are shared with the
    workers through fork, not pickled."""
    workers = workers or os.cpu_count() or 1
    l1, l2, l3 = (np.asarray(a, np.int64) for a in (l1, l2, l3))
    _SHARED.update(q=q, qt=qt, C=C, v=v, wr2=wr2, entries=entries, l_min=l_min, l1=l1, l2=l2,
                   l3=l3)
    try:
        bounds = np.linspace(0, l1.size, workers + 1).astype(np.int64)
        jobs = [(int(a), int(b), block, h2_mode, cols) for a, b in zip(bounds[:-1], bounds[1:])
                if b > a]
        if len(jobs) <= 1:
            parts = [_triples_job(j) for j in jobs]
        else:
            with get_context("fork").Pool(len(jobs)) as pool:
                parts = pool.map(_triples_job, jobs)
    finally:
        _SHARED.clear()
    if not parts:
        return np.zeros((entries.shape[0], entries.shape[0] if cols is None else len(cols)))
    out = parts[0].copy()
    for p_ in parts[1:]:
        out += p_
    return out


def slab_triples(l_min, l_max, l2_begin, l2_end):
    """Every ordered valid triple whose l2 lies in [l2_begin, l2_end) (geometry.py:161-171
    restricted to an l2 slab), ordered (l2, l3, l1).  Built directly, without enumerating the
    domain: for each (l2, l3) row, l1 runs over max(l_min, l3 - l2) .. l2 with l1+l2+l3 even."""
    out = [[], [], []]
    for l2 in range(max(l2_begin, l_min), min(l2_end, l_max + 1)):
        for l3 in range(l2, min(2 * l2, l_max) + 1):
            lo = max(l_min, l3 - l2)
            lo += (lo + l2 + l3) & 1
            if lo > l2:
                continue
            l1 = np.arange(lo, l2 + 1, 2, dtype=np.int64)
            out[0].append(l1)
            out[1].append(np.full(l1.size, l2, np.int64))
            out[2].append(np.full(l1.size, l3, np.int64))
    if not out[0]:
        return tuple(np.zeros(0, np.int64) for _ in range(3))
    return tuple(np.concatenate(o) for o in out)


def _sweep_job(args):
    begin, end, l_min, l_max, block, h2_mode = args
    d = _SHARED
    l1, l2, l3 = domain_triples(l_min, l_max, begin, end)
    return sweep_triples(d["q"], d["qt"], d["C"], d["v"], d["wr2"], d["entries"], l_min, l1, l2,
                         l3, block, h2_mode)


def gamma3d(q, qt, C, v, wr2, entries, l_min, l_max, begin=0, end=None, workers=1,
            block=64, h2_mode="gosper") -> np.ndarray:
    """gamma3d_matrix (engine3d.py:156-186): make_plan over [begin, end), fork pool of
    _sweep_chunk, merge in worker order (scheduler.py:32-66).  Same split, same order as the
    reference; the tables reach the workers through fork instead of being pickled per job
    (the reference pickles them once per Γ, which is noise at its run times but would
    dominate the bounded samples timed here)."""
    if end is None:
        end = domain_count(l_min, l_max)
    total = end - begin
    base, extra = divmod(total, workers)
    jobs, s = [], begin
    for w in range(workers):
        size = base + (1 if w < extra else 0)
        jobs.append((s, s + size, l_min, l_max, block, h2_mode))
        s += size
    _SHARED.update(q=q, qt=qt, C=C, v=v, wr2=wr2, entries=entries)
    try:
        if workers == 1:
            parts = [_sweep_job(jobs[0])]
        else:
            with get_context("fork").Pool(workers) as pool:
                parts = pool.map(_sweep_job, jobs)
    finally:
        _SHARED.clear()
    out = parts[0].copy()
    for p in parts[1:]:
        out += p
    return out


def radial_integral_x(l1, l2, l3, np_, qt, entries, wr2, l_min):
    """engine3d.py:56-70 with the trap rule folded into wr2."""
    ip, jp, kp = entries[np_]
    idx = (ip, jp, kp)
    f = np.zeros(qt.shape[1])
    for a, b, c in _PERMS:
        f += qt[idx[a], :, l1 - l_min] * qt[idx[b], :, l2 - l_min] * qt[idx[c], :, l3 - l_min]
    return float(math.fsum(wr2 * f))


def late_product_y(l1, l2, l3, n, q, entries, l_min):
    """engine3d.py:73-83."""
    idx = tuple(entries[n])
    return float(sum(q[idx[a], l1 - l_min] * q[idx[b], l2 - l_min] * q[idx[c], l3 - l_min]
                     for a, b, c in _PERMS))
