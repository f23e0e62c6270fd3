"""Small end-to-end case for compute-sanitizer (racecheck / synccheck / memcheck).

Runs every kernel family once on a problem small enough for instrumented execution:
stage 1 (Bessel + q̃ build), the separable Γ pipeline (panels, pair products, the three
persistent DMMA/TMA contractions with multi-k-tile windows, gather, final) through the
one-shot call with two shards, the explicit-triple path, and the non-separable DMMA kernel
on a sparse grid — each checked against the CPU oracle, so a silent corruption fails too.

    compute-sanitizer --tool racecheck python tools/sanitize_case.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from oracle import nonsep_ref, ref  # noqa: E402
from paper_1503_08809_b200 import (BasisTables, ModeMapping, RadialGrid, SparseDomain,  # noqa: E402
                                   build_qtilde, gamma3d_matrix, gamma_nonsep)
from paper_1503_08809_b200.configs import host_inputs, sparse_domain, sparse_grid  # noqa: E402

L_MAX = int(os.environ.get("SAN_LMAX", "90"))


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


hi = host_inputs("c0", l_max=L_MAX)
C, qt = build_qtilde(hi)
t = BasisTables(hi.q, qt, C, hi.v, 2, L_MAX)
m, r = ModeMapping(hi.entries, hi.spec.p), RadialGrid(hi.x)
want = ref.gamma3d(hi.q, qt, C, hi.v, hi.wr2, hi.entries, 2, L_MAX)
got = gamma3d_matrix(t, m, r, devices=[0, 0]).values
e1 = rel(got, want)

l1, l2, l3 = ref.domain_triples(2, L_MAX)
keep = (np.arange(l1.size) % 4) != 1


class Dom:
    pass


d = Dom()
d.l1, d.l2, d.l3, d.count = l1[keep], l2[keep], l3[keep], int(keep.sum())
got2 = gamma3d_matrix(t, m, r, domain=d, devices=[0]).values
want2 = ref.sweep_triples(hi.q, qt, C, hi.v, hi.wr2, hi.entries, 2, d.l1, d.l2, d.l3)
e2 = rel(got2, want2)

hi3 = host_inputs("c3", l_max=L_MAX)
C3, qt3 = build_qtilde(hi3)
t3 = BasisTables(hi3.q, qt3, C3, hi3.v, 2, L_MAX)
g, w = sparse_grid(l_max=L_MAX, dense_to=30, step=6)
dom = SparseDomain(*sparse_domain(g, w))
b = gamma_nonsep(t3, ModeMapping(hi3.entries, 8), RadialGrid(hi3.x), hi3.alpha, dom).values[:, 0]
bw = nonsep_ref.nonsep(hi3.q, qt3, C3, hi3.v, hi3.wr2, hi3.entries, hi3.alpha, 2, dom.l1,
                       dom.l2, dom.l3, dom.weight)
e3 = rel(b, bw)
print(f"sanitize case l_max={L_MAX}: separable {e1:.2e}, triples {e2:.2e}, non-separable {e3:.2e}")
assert e1 < 1e-10 and e2 < 1e-10 and e3 < 1e-8
