"""Latency of the drop-in call at the reference's own CPU-runnable sizes (host buffers in,
Γ out): desk (l_max 16, p 3), acceptance (l_max 32, p 4, Nx 216) and config 0."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1503_08809_b200 import (BasisTables, ModeMapping, RadialGrid,  # noqa: E402
                                   build_qtilde, gamma3d_matrix)
from paper_1503_08809_b200.configs import host_inputs  # noqa: E402

g = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "desk.npz"))
cases = []
for tag in ("desk", "desk32"):
    lmin, lmax = (int(x) for x in g[f"{tag}_lrange"])
    t = BasisTables(g[f"{tag}_q"], g[f"{tag}_qt"], g[f"{tag}_C"], g[f"{tag}_v"], lmin, lmax)
    cases.append((tag, t, ModeMapping(g[f"{tag}_entries"], t.p_max), RadialGrid(g[f"{tag}_r"])))
hi = host_inputs("c0")
C, qt = build_qtilde(hi, device=0)
cases.append(("c0", BasisTables(hi.q, qt, C, hi.v, hi.l_min, hi.l_max),
              ModeMapping(hi.entries, hi.spec.p), RadialGrid(hi.x)))
for tag, t, m, r in cases:
    ts = []
    for i in range(8):
        t0 = time.perf_counter()
        gamma3d_matrix(t, m, r)
        ts.append(time.perf_counter() - t0)
    print(f"{tag:7s} l_max={t.l_max:4d} p={t.p_max} Nx={t.n_radial:4d}: first {ts[0]*1e3:8.2f} ms, "
          f"median of next 7 {np.median(ts[1:])*1e3:8.2f} ms, min {min(ts)*1e3:8.2f} ms")
