"""GPU parity of stage 1 (Bessel generator, Δ, C_l, q̃) and of the non-separable path.

Stage 1 and the non-separable path have no reference implementation:
the oracle is the scipy restatement (oracle/qtilde_ref.py) and the gamma3d_naive-shaped
restatement (oracle/nonsep_ref.py) — "parity unpinned".  The non-separable
path is additionally anchored on the reference's own Γ: on a step-1 grid b == Γ·α.
Tolerances: q̃ per-l relative Frobenius <= 1e-11; non-separable relative <= 1e-8.
"""

import numpy as np
import pytest
from scipy.special import spherical_jn

from conftest import frob_rel
from oracle import nonsep_ref, qtilde_ref
from paper_1503_08809_b200 import (BasisTables, ModeMapping, RadialGrid, SparseDomain,
                                   bessel_table, build_qtilde, gamma3d_matrix, gamma_nonsep)
from paper_1503_08809_b200.configs import host_inputs, sparse_domain, sparse_grid

pytestmark = pytest.mark.gpu


class TestBessel:
    def test_against_scipy(self):
        rng = np.random.default_rng(3)
        z = np.concatenate([rng.uniform(0.5, 6000, 64), np.arange(1.0, 3100, 97),
                            [1.3, 1.4, 2.0, 2000.0, 2000.5, 5600.0]])
        got = bessel_table(z, 3000)
        want = spherical_jn(np.arange(3001)[None, :], z[:, None])
        scale = np.abs(want).max(1, keepdims=True)
        assert np.max(np.abs(got - want) / scale) < 1e-12
        # relative accuracy away from zero crossings (CUDA and glibc sin/cos differ by an ulp,
        # which the recurrence carries; near a zero of j_l only the absolute error is meaningful)
        sig = np.abs(want) > 1e-3 * scale
        assert np.max(np.abs(got - want)[sig] / np.abs(want)[sig]) < 1e-11
        tail = (np.arange(3001)[None, :] > z[:, None]) & (np.abs(want) > 1e-200)
        assert np.max(np.abs(got - want)[tail] / np.abs(want)[tail]) < 2e-12

    def test_zero_argument(self):
        got = bessel_table(np.array([0.0]), 5)
        assert np.array_equal(got[0], [1, 0, 0, 0, 0, 0])


class TestStage1:
    def test_c0_against_scipy(self, g_c0):
        hi = host_inputs("c0")
        C, qt, delta = build_qtilde(hi, with_delta=True)
        assert np.max(np.abs(delta[[0, 50, 198]] - g_c0["delta_rows"])) \
            < 1e-13 * np.abs(g_c0["delta_rows"]).max()
        assert np.max(np.abs(C / g_c0["C"] - 1)) < 1e-11
        ref = g_c0["qt"]
        num = np.linalg.norm(qt - ref, axis=(0, 1))
        den = np.linalg.norm(ref, axis=(0, 1))
        assert np.max(num / den) < 1e-11                      # per-l relative Frobenius

    def test_c1_sampled_l(self):
        hi = host_inputs("c1")
        C, qt = build_qtilde(hi)
        ells = [2, 3, 500, 1499, 1998, 2000]
        d = qtilde_ref.delta_table(hi.k, hi.eps, 2, hi.l_max)
        Cr = qtilde_ref.c_ell(d, hi.k, hi.wk)
        assert np.max(np.abs(C / Cr - 1)) < 1e-11
        ref = qtilde_ref.qtilde(hi.k, hi.wk, hi.x, hi.qk, d, 2, hi.l_max, ells)
        for l in ells:
            a, b = qt[:, :, l - 2], ref[:, :, l - 2]
            assert np.linalg.norm(a - b) <= 1e-11 * np.linalg.norm(b), l

    def test_gamma_end_to_end_c0(self, g_c0):
        """GPU-built q̃ -> GPU Γ vs the reference Γ on scipy-built q̃."""
        hi = host_inputs("c0")
        C, qt = build_qtilde(hi)
        t = BasisTables(hi.q, qt, C, hi.v, 2, 200)
        got = gamma3d_matrix(t, ModeMapping(hi.entries, 6), RadialGrid(hi.x)).values
        assert frob_rel(got, g_c0["gamma"]) < 1e-10


class TestNonSeparable:
    def test_step1_grid_equals_gamma_alpha(self, g_c0):
        """Known answer: W = 1 and exact parity on a step-1 grid -> b = Γ α."""
        hi = host_inputs("c0")
        t = BasisTables(hi.q, g_c0["qt"], g_c0["C"], hi.v, 2, 200)
        m = ModeMapping(hi.entries, 6)
        grid, w = sparse_grid(l_max=200, dense_to=200)
        assert np.all(w == 1.0)
        dom = SparseDomain(*sparse_domain(grid, w))
        alpha = np.random.default_rng(5).standard_normal(m.n_max)
        b = gamma_nonsep(t, m, RadialGrid(hi.x), alpha, dom).values[:, 0]
        want = g_c0["gamma"] @ alpha
        assert np.linalg.norm(b - want) <= 1e-12 * np.linalg.norm(want)

    def test_config3_against_restatement(self):
        hi = host_inputs("c3", l_max=400)
        C, qt = build_qtilde(hi)
        t = BasisTables(hi.q, qt, C, hi.v, 2, hi.l_max)
        m = ModeMapping(hi.entries, 8)
        grid, w = sparse_grid(l_max=hi.l_max)
        l1, l2, l3, W = sparse_domain(grid, w)
        b = gamma_nonsep(t, m, RadialGrid(hi.x), hi.alpha, SparseDomain(l1, l2, l3, W))
        want = nonsep_ref.nonsep(hi.q, qt, C, hi.v, hi.wr2, hi.entries, hi.alpha, 2, l1, l2,
                                 l3, W)
        assert b.shape == (120, 1)
        assert np.linalg.norm(b.values[:, 0] - want) <= 1e-8 * np.linalg.norm(want)
