"""ctypes binding of the C-ABI library `libmodal_b200.so` (include/modal_b200.h).

The library is built in-tree (`python -m paper_1503_08809_b200.build` or
`__graft_entry__.build()`).  Importing this module never falls back to anything: if the
library is missing, `lib()` raises; if no B200 is visible, every compute entry point
returns MG_ECUDA and `check()` raises RuntimeError.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

__all__ = ["lib", "check", "LIB_PATH", "ptr", "MG_H2", "NativeError"]

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MG_LIB_PATH") or os.path.join(HERE, "_native", "libmodal_b200.so")
MG_H2 = {"gosper": 0, "exact": 1}

_i = ctypes.c_int
_i64 = ctypes.c_int64
_d = ctypes.c_double
_vp = ctypes.c_void_p
_I64P = ctypes.POINTER(ctypes.c_int64)

_SIGS = {
    "mg_version": (_i, []),
    "mg_last_error": (ctypes.c_char_p, []),
    "mg_device_count": (_i, []),
    "mg_debug_checks": (_i, [_vp, _i, _i, _vp, _i]),
    "mg_domain_count": (_i, [_i, _i, _vp, _vp]),
    "mg_domain_triples": (_i, [_i, _i, _i64, _i64, _vp, _vp, _vp, _i]),
    "mg_domain_match_range": (_i, [_i, _i, _vp, _vp, _vp, _i64, _vp]),
    "mg_weights": (_i, [_i, _i, _vp, _vp, _i, _i64, _i64, _vp, _i]),
    "mg_gamma_sep": (_i, [_vp, _vp, _vp, _vp, _vp, _vp, _i, _i, _i, _i, _i, _i, _i64, _i64, _i,
                          _vp, _vp]),
    "mg_gamma_sep_slab": (_i, [_vp, _vp, _vp, _vp, _vp, _vp, _i, _i, _i, _i, _i, _i, _i, _i, _i,
                               _vp]),
    "mg_gamma_sep_triples": (_i, [_vp, _vp, _vp, _vp, _vp, _vp, _i, _i, _i, _i, _i, _i, _vp, _vp,
                                  _vp, _i64, _i, _vp, _vp]),
    "mg_slab_plan": (_i, [_i, _i, _i, _i, _i, _vp]),
    "mg_plan_create": (_i, [_vp, _vp, _vp, _vp, _vp, _vp, _i, _i, _i, _i, _i, _i, _i, _vp]),
    "mg_plan_create_dev": (_i, [_vp, _vp, _vp, _vp, _vp, _vp, _i, _i, _i, _i, _i, _i, _i, _vp]),
    "mg_plan_execute": (_i, [_vp, _i, _i, _vp, _vp]),
    "mg_plan_fetch": (_i, [_vp, _vp, _vp]),
    "mg_plan_stats": (_i, [_vp, _vp, _vp, _vp, _vp]),
    "mg_plan_set_profile": (_i, [_vp, _i]),
    "mg_plan_kernel_ms": (_i, [_vp, _vp]),
    "mg_plan_destroy": (None, [_vp]),
    "mg_plan_set_sparse_domain": (_i, [_vp, _vp, _vp, _vp, _vp, _i64]),
    "mg_plan_nonsep": (_i, [_vp, _vp, _vp, _vp, _vp]),
    "mg_build_qtilde": (_i, [_vp, _vp, _i, _vp, _i, _vp, _vp, _i, _i, _i, _d, _d, _d, _i, _vp,
                             _vp, _vp]),
    "mg_build_qtilde_dev": (_i, [_vp, _vp, _i, _vp, _i, _vp, _vp, _i, _i, _i, _d, _d, _d, _i,
                                 _vp, _vp, _vp]),
    "mg_bessel_table": (_i, [_vp, _i, _i, _i, _vp]),
    "mg_ptable": (_i, [_vp, _vp, _vp, _vp, _i, _i, _i, _i, _i, _vp]),
    "mg_gamma2d_timings": (_i, [_vp, _vp]),
    "mg_gamma2d": (_i, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i, _i, _i, _i, _i, _i, _vp]),
    "mg_gamma_nonsep": (_i, [_vp, _vp, _vp, _vp, _vp, _vp, _i, _i, _i, _i, _i, _i, _vp, _vp, _vp,
                             _vp, _vp, _i64, _i, _vp]),
}

_LIB = None


class NativeError(RuntimeError):
    pass


def lib():
    """Load the in-tree CUDA library (raises if it has not been built)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_1503_08809_b200.build` "
                "(there is no CPU fallback)")
        handle = ctypes.CDLL(LIB_PATH)
        variant = "MG_LIB_PATH" in os.environ   # tuning variants may predate newer symbols
        for name, (res, args) in _SIGS.items():
            if variant and not hasattr(handle, name):
                continue
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = handle
    return _LIB


def check(rc: int) -> None:
    """Map MG_* return codes onto the reference's exception classes (cli.py:139-148)."""
    if rc == 0:
        return
    msg = lib().mg_last_error().decode("utf-8", "replace")
    if rc == 1:
        raise ValueError(msg)
    if rc == 2:
        raise MemoryError(msg)
    raise NativeError(msg)


CHECK_SITES = ("panel write", "K1 panel source", "K1 WQB source", "K1 H write",
               "pair-product S write", "K2 S source", "K2 H source", "K2 G write",
               "gather R/Sq write", "K3 Sq source", "K3 R source", "K3 Z write",
               "non-separable QTS source", "non-separable Q1W read", "non-separable triple l-range")


def debug_checks(reset: bool = False, device: int = 0):
    """(checked_build, {site: violations}) from a library built with -DMG_CHECKED=1."""
    counts = np.zeros(16, np.uint32)
    flag = np.zeros(1, np.int32)
    check(lib().mg_debug_checks(ptr(counts), 16, int(reset), ptr(flag), int(device)))
    return bool(flag[0]), {s: int(c) for s, c in zip(CHECK_SITES, counts)}


def ptr(a: np.ndarray | None):
    if a is None:
        return None
    return ctypes.c_void_p(a.ctypes.data)
