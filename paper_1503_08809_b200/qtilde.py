"""Stage 1 on the GPU: Δ_l(k), C_l and q̃_p(x, l) (absent from the reference,
SPEC.md:14,224 — its stand-in is synthesize_basis, basis.py:279-297).

    build_qtilde(inputs) -> (C [L], q_tilde [p, Nx, L])           host arrays
    build_qtilde_device(inputs, device) -> (C_dev, qt_dev)         torch tensors on the GPU

`inputs` is a `configs.HostInputs` (or anything with k, wk, x, eps, qk, l_min, l_max).
"""

from __future__ import annotations

import numpy as np

from . import _native as nat
from .configs import EPS_AMP, K_DAMP, X_DELTA

__all__ = ["build_qtilde", "build_qtilde_device", "bessel_table"]


def _args(hi):
    k = np.ascontiguousarray(hi.k, np.float64)
    wk = np.ascontiguousarray(hi.wk, np.float64)
    x = np.ascontiguousarray(hi.x, np.float64)
    eps = np.ascontiguousarray(hi.eps, np.float64)
    qk = np.ascontiguousarray(hi.qk, np.float64)
    L = hi.l_max - hi.l_min + 1
    if eps.shape != (L, k.size) or qk.shape[1] != k.size:
        raise ValueError("inconsistent stage-1 input shapes")
    return k, wk, x, eps, qk


def build_qtilde(hi, device: int = 0, with_delta: bool = False):
    """(C, q̃[, Δ]) as host float64 arrays, computed on `device`."""
    k, wk, x, eps, qk = _args(hi)
    p, L = qk.shape[0], hi.l_max - hi.l_min + 1
    C = np.zeros(L)
    qt = np.zeros((p, x.size, L))
    delta = np.zeros((L, k.size)) if with_delta else None
    nat.check(nat.lib().mg_build_qtilde(
        nat.ptr(k), nat.ptr(wk), k.size, nat.ptr(x), x.size, nat.ptr(eps), nat.ptr(qk), p,
        hi.l_min, hi.l_max, X_DELTA, K_DAMP, EPS_AMP, int(device), nat.ptr(C), nat.ptr(qt),
        nat.ptr(delta)))
    return (C, qt, delta) if with_delta else (C, qt)


def build_qtilde_device(hi, device: int = 0, stream=None):
    """(C, q̃) left in device memory as torch float64 tensors (for the resident plan)."""
    import torch

    k, wk, x, eps, qk = _args(hi)
    p, L = qk.shape[0], hi.l_max - hi.l_min + 1
    dev = torch.device("cuda", device)
    C = torch.zeros(L, dtype=torch.float64, device=dev)
    qt = torch.zeros((p, x.size, L), dtype=torch.float64, device=dev)
    s = None if stream is None else stream.cuda_stream
    nat.check(nat.lib().mg_build_qtilde_dev(
        nat.ptr(k), nat.ptr(wk), k.size, nat.ptr(x), x.size, nat.ptr(eps), nat.ptr(qk), p,
        hi.l_min, hi.l_max, X_DELTA, K_DAMP, EPS_AMP, int(device), C.data_ptr(), qt.data_ptr(),
        s))
    return C, qt


def bessel_table(z, l_max: int, device: int = 0) -> np.ndarray:
    """j_l(z) for l = 0..l_max from the on-device recurrence, shape [len(z), l_max+1]."""
    z = np.ascontiguousarray(np.atleast_1d(z), np.float64)
    out = np.zeros((z.size, l_max + 1))
    nat.check(nat.lib().mg_bessel_table(nat.ptr(z), z.size, int(l_max), int(device),
                                        nat.ptr(out)))
    return out
