"""Device-resident Γ plan: tables uploaded once, any number of Γ's / l2-slab shards.

Wraps mg_plan_* (include/modal_b200.h).  Used by bench.py (inputs resident in HBM) and by
the multi-GPU ranks (`dist.py`), each of which executes one l2 slab.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as nat
from .quadrature import x_weights

__all__ = ["GammaPlan"]


class GammaPlan:
    def __init__(self, q, q_tilde, C, v, wr2, entries, l_min, l_max, h2_mode="gosper",
                 device: int = 0):
        """`q_tilde` may be a host ndarray [p, Nx, L] or a CUDA torch tensor of that shape."""
        self.q = np.ascontiguousarray(q, np.float64)
        self.C = np.ascontiguousarray(C, np.float64)
        self.v = np.ascontiguousarray(v, np.float64)
        self.wr2 = np.ascontiguousarray(wr2, np.float64)
        self.entries = np.ascontiguousarray(entries, np.int64)
        self.l_min, self.l_max = int(l_min), int(l_max)
        self.device = int(device)
        self.p = self.q.shape[0]
        self.n = self.entries.shape[0]
        self.nx = self.wr2.size
        self._h = ctypes.c_void_p()
        L = self.l_max - self.l_min + 1
        if tuple(q_tilde.shape) != (self.p, self.nx, L):
            raise ValueError(f"q_tilde must have shape ({self.p}, {self.nx}, {L}) to match q "
                             f"and wr2, got {tuple(q_tilde.shape)}")
        if self.q.shape != (self.p, L) or self.C.shape != (L,) or self.v.shape != (L,):
            raise ValueError("q, C, v do not match [l_min, l_max]")
        lib = nat.lib()
        args = (nat.ptr(self.q), None, nat.ptr(self.C), nat.ptr(self.v), nat.ptr(self.wr2),
                nat.ptr(self.entries), self.p, self.nx, self.n, self.l_min, self.l_max,
                nat.MG_H2[h2_mode], self.device, ctypes.byref(self._h))
        if isinstance(q_tilde, np.ndarray):
            qt = np.ascontiguousarray(q_tilde, np.float64)
            args = args[:1] + (nat.ptr(qt),) + args[2:]
            nat.check(lib.mg_plan_create(*args))
        else:
            args = args[:1] + (ctypes.c_void_p(q_tilde.data_ptr()),) + args[2:]
            nat.check(lib.mg_plan_create_dev(*args))

    @classmethod
    def from_tables(cls, tables, mapping, grid, h2_mode="gosper", integrator="trap", device=0):
        return cls(tables.q, tables.q_tilde, tables.C, tables.v, x_weights(grid.r, integrator),
                   mapping.entries, tables.l_min, tables.l_max, h2_mode, device)

    def execute(self, l2_begin: int | None = None, l2_end: int | None = None, out=None,
                stream=None):
        """Run the l2 slab [l2_begin, l2_end) (default: everything).  `out` may be a CUDA
        torch tensor [n, n] receiving Γ; `stream` a torch.cuda.Stream."""
        b = self.l_min if l2_begin is None else int(l2_begin)
        e = -1 if l2_end is None else int(l2_end)
        s = None if stream is None else ctypes.c_void_p(stream.cuda_stream)
        o = None if out is None else ctypes.c_void_p(out.data_ptr())
        nat.check(nat.lib().mg_plan_execute(self._h, b, e, o, s))

    def fetch(self, stream=None) -> np.ndarray:
        out = np.zeros((self.n, self.n))
        s = None if stream is None else ctypes.c_void_p(stream.cuda_stream)
        nat.check(nat.lib().mg_plan_fetch(self._h, nat.ptr(out), s))
        return out

    def stats(self) -> dict:
        f = [ctypes.c_double() for _ in range(3)]
        n = ctypes.c_int64()
        nat.check(nat.lib().mg_plan_stats(self._h, *(ctypes.byref(x) for x in f),
                                          ctypes.byref(n)))
        return {"flops_run": f[0].value, "flops_x": f[1].value, "flops_pair": f[2].value,
                "launches": n.value}

    def set_profile(self, on: bool = True):
        nat.check(nat.lib().mg_plan_set_profile(self._h, int(bool(on))))

    def kernel_ms(self) -> dict:
        ms = np.zeros(8)
        nat.check(nat.lib().mg_plan_kernel_ms(self._h, nat.ptr(ms)))
        return dict(zip(("operands", "run", "x", "gather", "pair", "final", "operands_side",
                         "nonsep"), ms.tolist()))

    # ---- non-separable path on a resident sparse domain (BASELINE config 3) ----
    def set_sparse_domain(self, domain):
        """Upload a `SparseDomain` (l1, l2, l3, weight) once for repeated `nonsep` calls."""
        self._ns = tuple(np.ascontiguousarray(a, np.int32) for a in (domain.l1, domain.l2,
                                                                      domain.l3))
        W = np.ascontiguousarray(domain.weight, np.float64)
        nat.check(nat.lib().mg_plan_set_sparse_domain(self._h, *(nat.ptr(a) for a in self._ns),
                                                      nat.ptr(W), int(W.size)))

    def nonsep(self, alpha, out=None, stream=None) -> np.ndarray | None:
        """b = Σ_t W_t zm_t P[:,t] Σ_x wr2_x B(t,x) for primordial coefficients `alpha` [n].
        With `out` (CUDA torch tensor [n]) the result stays on the device (asynchronous);
        otherwise it is returned as a host array."""
        a = np.ascontiguousarray(alpha, np.float64)
        if a.shape != (self.n,):
            raise ValueError("alpha must have one coefficient per primordial mode")
        s = None if stream is None else ctypes.c_void_p(stream.cuda_stream)
        if out is not None:
            nat.check(nat.lib().mg_plan_nonsep(self._h, nat.ptr(a),
                                               ctypes.c_void_p(out.data_ptr()), None, s))
            return None
        b = np.zeros(self.n)
        nat.check(nat.lib().mg_plan_nonsep(self._h, nat.ptr(a), None, nat.ptr(b), s))
        return b

    def close(self):
        if self._h:
            nat.lib().mg_plan_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
