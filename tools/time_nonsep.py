"""Break down the config-3 call: setup (plan, uploads) vs the pointwise kernel."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1503_08809_b200 import (BasisTables, ModeMapping, RadialGrid, SparseDomain,  # noqa: E402
                                   build_qtilde, gamma_nonsep)
from paper_1503_08809_b200.configs import host_inputs, sparse_domain, sparse_grid  # noqa: E402

hi = host_inputs("c3")
C, qt = build_qtilde(hi)
t = BasisTables(hi.q, qt, C, hi.v, 2, hi.l_max)
m = ModeMapping(hi.entries, 8)
g = RadialGrid(hi.x)
dom = SparseDomain(*sparse_domain(*sparse_grid()))
for n in (1000, 100000, dom.count):
    d = SparseDomain(dom.l1[:n], dom.l2[:n], dom.l3[:n], dom.weight[:n])
    gamma_nonsep(t, m, g, hi.alpha, d)
    t0 = time.perf_counter()
    gamma_nonsep(t, m, g, hi.alpha, d)
    print(n, f"{time.perf_counter() - t0:.4f} s")
