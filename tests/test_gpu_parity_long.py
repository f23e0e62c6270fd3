"""GPU parity in the benchmarked regime: long l1-windows at p >= 15, rows with holes, several
batches, and the full config-3 non-separable projection.

Round 1 checked c1/c2/c4 only on short flat ranges (every (l2,l3) row then holds a 1-triple
l1 window).  Here the oracle runs on exactly the triples of narrow TOP-l2 slabs, whose rows
carry l1 windows of ~1000-1500 triples, so the multi-k-tile persistent run contraction, the
nested-window union of packed tiles (rows with different l1 lower bounds l3 - l2 share a
128-slot tile) and the x/pair contractions at p = 15, 22, 30 are all compared with the
reference algorithm (oracle/ref.py = engine3d._sweep_chunk over an explicit triple list,
engine3d.py:123-136, pinned bit-for-bit to the reference on config 0).

Tolerance: relative Frobenius <= 1e-10 (north_star); non-separable <= 1e-8.
"""

import os

import numpy as np
import pytest

from conftest import frob_rel, golden
from oracle import nonsep_ref, ref
from paper_1503_08809_b200 import (BasisTables, GammaPlan, ModeMapping, RadialGrid,
                                   SparseDomain, build_qtilde, gamma3d_matrix, gamma_nonsep,
                                   x_weights)
from paper_1503_08809_b200.configs import host_inputs, sparse_domain, sparse_grid

pytestmark = pytest.mark.gpu

WORKERS = min(os.cpu_count() or 1, 16)


@pytest.fixture(scope="module")
def stage1():
    cache = {}

    def get(cfg):
        if cfg not in cache:
            hi = host_inputs(cfg)
            C, qt = build_qtilde(hi)
            cache.clear()                      # one config's q̃ at a time (c4 q̃ is 1.4 GB)
            cache[cfg] = (hi, C, qt)
        return cache[cfg]
    return get


def col_subset(n, k, seed):
    """k primordial modes (columns of Γ) incl. the first and last, seeded."""
    rng = np.random.default_rng(seed)
    return np.unique(np.concatenate([[0, n - 1], rng.choice(n, k, replace=False)]))


@pytest.mark.parametrize("cfg,l2a,l2b,ncols", [
    ("c1", 1998, 2001, None),      # p=15: 6 rows, 5994 triples, windows ~1000
    ("c2", 2500, 2501, None),      # p=22: 1 row, 1250 triples, 40 k-tiles
    ("c4", 2999, 3001, 248),       # p=30: 3 rows, 4498 triples; 250 of 4960 columns
])
def test_top_l2_slab_vs_oracle(stage1, cfg, l2a, l2b, ncols):
    hi, C, qt = stage1(cfg)
    l1, l2, l3 = ref.slab_triples(2, hi.l_max, l2a, l2b)
    plan = GammaPlan(hi.q, qt, C, hi.v, hi.wr2, hi.entries, 2, hi.l_max)
    plan.execute(l2a, l2b)
    got = plan.fetch()
    plan.close()
    n = hi.entries.shape[0]
    cols = None if ncols is None else col_subset(n, ncols, 7)
    want = ref.sweep_triples_parallel(hi.q, qt, C, hi.v, hi.wr2, hi.entries, 2, l1, l2, l3,
                                      workers=WORKERS, block=16 if cfg == "c4" else 64,
                                      cols=cols)
    if cols is not None:
        got = got[:, cols]
    assert frob_rel(got, want) <= 1e-10


def test_rows_with_holes_two_batches(stage1):
    """Explicit triple list (mg_gamma_sep_triples) at config 1: every (l2,l3) row of the
    l2 slab [1000, 1009) keeps only the first and last l1 of its window (a hole in between),
    ~9000 rows > the 8288-row batch of the run/x contractions, triples shuffled."""
    hi, C, qt = stage1("c1")
    l1, l2, l3 = ref.slab_triples(2, hi.l_max, 1000, 1009)
    key = l2 * 4096 + l3
    first = np.r_[True, key[1:] != key[:-1]]
    last = np.r_[key[1:] != key[:-1], True]
    keep = first | last
    a, b, c = l1[keep], l2[keep], l3[keep]
    assert np.unique(key).size > 8288
    perm = np.random.default_rng(5).permutation(a.size)
    a, b, c = a[perm], b[perm], c[perm]

    class Dom:
        pass

    d = Dom()
    d.l1, d.l2, d.l3, d.count = a, b, c, a.size
    t = BasisTables(hi.q, qt, C, hi.v, 2, hi.l_max)
    got = gamma3d_matrix(t, ModeMapping(hi.entries, hi.spec.p), RadialGrid(hi.x), domain=d).values
    cols = col_subset(hi.entries.shape[0], 168, 11)
    want = ref.sweep_triples_parallel(hi.q, qt, C, hi.v, hi.wr2, hi.entries, 2, a, b, c,
                                      workers=WORKERS, cols=cols)
    assert frob_rel(got[:, cols], want) <= 1e-10


class TestConfig3Full:
    """All 724,930 sparse triples of config 3 (l_max 2000, 120 modes, Nx 300) against the
    restatement run in full when the golden was written (tests/golden/make_c3_golden.py),
    itself pinned to the reference's per-triple functions on a sample (test_oracle_golden)."""

    @pytest.fixture(scope="class")
    def c3(self):
        g = golden("c3.npz")
        hi = host_inputs("c3")
        l1, l2, l3, W = sparse_domain(*sparse_grid(l_max=hi.l_max))
        assert l1.size == int(g["count"])
        return hi, g, SparseDomain(l1, l2, l3, W)

    @pytest.mark.parametrize("mode", ["gosper", "exact"])
    def test_same_inputs(self, c3, mode):
        """Identical inputs (the golden's scipy q̃ at the grid multipoles, zeros elsewhere)."""
        hi, g, dom = c3
        qt = np.zeros((hi.spec.p, hi.x.size, hi.l_max - 1))
        qt[:, :, g["grid"] - 2] = g["qt_grid"]
        t = BasisTables(hi.q, qt, g["C"], hi.v, 2, hi.l_max)
        b = gamma_nonsep(t, ModeMapping(hi.entries, hi.spec.p), RadialGrid(hi.x), hi.alpha,
                         dom, h2_mode=mode).values[:, 0]
        assert frob_rel(b, g[f"b_{mode}"]) <= 1e-12

    def test_end_to_end_gpu_stage1(self, c3):
        """q̃ and C built on the GPU (all l), then the GPU projection, vs the golden b."""
        hi, g, dom = c3
        C, qt = build_qtilde(hi)
        t = BasisTables(hi.q, qt, C, hi.v, 2, hi.l_max)
        b = gamma_nonsep(t, ModeMapping(hi.entries, hi.spec.p), RadialGrid(hi.x), hi.alpha,
                         dom).values[:, 0]
        assert frob_rel(b, g["b_gosper"]) <= 1e-8

    def test_odd_parity_cells_exact_mode(self, c3):
        """h2_mode="exact" on odd-parity cells: weight exactly 0 (theta gate), so the exact-
        mode b over the odd cells alone vanishes and the even cells reproduce the golden."""
        hi, g, dom = c3
        qt = np.zeros((hi.spec.p, hi.x.size, hi.l_max - 1))
        qt[:, :, g["grid"] - 2] = g["qt_grid"]
        t = BasisTables(hi.q, qt, g["C"], hi.v, 2, hi.l_max)
        odd = (dom.l1 + dom.l2 + dom.l3) % 2 == 1
        assert odd.any()
        m, r = ModeMapping(hi.entries, hi.spec.p), RadialGrid(hi.x)
        sub = SparseDomain(dom.l1[odd], dom.l2[odd], dom.l3[odd], dom.weight[odd])
        b_odd = gamma_nonsep(t, m, r, hi.alpha, sub, h2_mode="exact").values[:, 0]
        assert not np.any(b_odd)
        ev = ~odd
        sub = SparseDomain(dom.l1[ev], dom.l2[ev], dom.l3[ev], dom.weight[ev])
        b_ev = gamma_nonsep(t, m, r, hi.alpha, sub, h2_mode="exact").values[:, 0]
        assert frob_rel(b_ev, g["b_exact"]) <= 1e-12


def test_config3_resident_plan_matches_oneshot():
    """The resident plan (bench value path) equals the one-shot call on a c3 sub-grid."""
    hi = host_inputs("c3", l_max=400)
    C, qt = build_qtilde(hi)
    g, w = sparse_grid(l_max=400)
    dom = SparseDomain(*sparse_domain(g, w))
    t = BasisTables(hi.q, qt, C, hi.v, 2, 400)
    m, r = ModeMapping(hi.entries, hi.spec.p), RadialGrid(hi.x)
    b1 = gamma_nonsep(t, m, r, hi.alpha, dom).values[:, 0]
    plan = GammaPlan(hi.q, qt, C, hi.v, x_weights(hi.x), hi.entries, 2, 400)
    plan.set_sparse_domain(dom)
    b2 = plan.nonsep(hi.alpha)
    plan.close()
    assert np.array_equal(b1, b2)
    want = nonsep_ref.nonsep_parallel(hi.q, qt, C, hi.v, hi.wr2, hi.entries, hi.alpha, 2,
                                      dom.l1, dom.l2, dom.l3, dom.weight, workers=WORKERS)
    assert frob_rel(b1, want) <= 1e-8
