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

    @pytest.mark.parametrize("cfg,ells", [("c1", [2, 3, 500, 1499, 1998, 2000]),
                                          ("c2", [2, 1251, 2499, 2500]),
                                          ("c4", [2, 1501, 2999, 3000])])
    def test_sampled_l(self, cfg, ells):
        """Sampled multipoles at p = 15 / 22 / 30, Nk 3000 / 4000 / 5000, kx up to 6000."""
        hi = host_inputs(cfg)
        C, qt = build_qtilde(hi)
        d = qtilde_ref.delta_table(hi.k, hi.eps, 2, hi.l_max)
        Cr = qtilde_ref.c_ell(d, hi.k, hi.wk)
        assert np.max(np.abs(C / Cr - 1)) < 1e-11
        # the scipy oracle costs ~2 µs per (l, k, x): compare on ~125 evenly spaced x (both ends
        # included) so the whole GPU suite stays well inside the driver's 20-minute limit
        xi = np.unique(np.linspace(0, hi.x.size - 1, 125).round().astype(int))
        ref = qtilde_ref.qtilde(hi.k, hi.wk, hi.x[xi], hi.qk, d, 2, hi.l_max, ells)
        for l in ells:
            a, b = qt[:, xi, l - 2], ref[:, :, l - 2]
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

    @staticmethod
    def _small(p, l_max=120, seed=11, nx=40):
        """Random tables of basis size p on a small sparse grid (kernel-shape coverage)."""
        from paper_1503_08809_b200.basis import default_mode_mapping
        rng = np.random.default_rng(seed)
        L = l_max - 1
        q = rng.standard_normal((p, L))
        qt = rng.standard_normal((p, nx, L)) * 1e-3
        C = rng.uniform(0.5, 2.0, L)
        v = (2.0 * np.arange(2, l_max + 1) + 1.0) ** (1.0 / 6.0)
        x = np.linspace(13600.0, 14400.0, nx)
        entries = default_mode_mapping(p).entries
        grid, w = sparse_grid(l_max=l_max, dense_to=30, step=7)
        dom = SparseDomain(*sparse_domain(grid, w))
        alpha = rng.standard_normal(entries.shape[0])
        return q, qt, C, v, x, entries, dom, alpha

    @pytest.mark.parametrize("p", [1, 3, 5, 8, 12, 16, 18])
    def test_basis_sizes_against_restatement(self, p):
        """Every compile-time kernel instance (p <= 16) and the generic kernel (p > 16)."""
        from paper_1503_08809_b200.quadrature import x_weights
        q, qt, C, v, x, entries, dom, alpha = self._small(p, nx=37 if p % 2 else 40)
        t = BasisTables(q, qt, C, v, 2, q.shape[1] + 1)
        m = ModeMapping(entries, p)
        b = gamma_nonsep(t, m, RadialGrid(x), alpha, dom).values[:, 0]
        want = nonsep_ref.nonsep(q, qt, C, v, x_weights(x, "trap"), entries, alpha, 2,
                                 dom.l1, dom.l2, dom.l3, dom.weight)
        assert np.linalg.norm(b - want) <= 1e-8 * np.linalg.norm(want)

    def test_mode_subset(self):
        """A mapping with a subset of the ordered triples (Ã built only from its modes)."""
        from paper_1503_08809_b200.quadrature import x_weights
        q, qt, C, v, x, entries, dom, alpha = self._small(6)
        keep = np.arange(0, entries.shape[0], 3)
        ent, al = entries[keep], alpha[keep]
        t = BasisTables(q, qt, C, v, 2, q.shape[1] + 1)
        b = gamma_nonsep(t, ModeMapping(ent, 6), RadialGrid(x), al, dom).values[:, 0]
        want = nonsep_ref.nonsep(q, qt, C, v, x_weights(x, "trap"), ent, al, 2, dom.l1, dom.l2,
                                 dom.l3, dom.weight)
        assert b.shape == (keep.size,)
        assert np.linalg.norm(b - want) <= 1e-8 * np.linalg.norm(want)

    def test_resident_plan(self):
        """GammaPlan.set_sparse_domain/nonsep: same b as the one-shot call, bitwise stable
        across calls, linear in α, device output, empty domain -> zeros."""
        import torch
        from paper_1503_08809_b200 import GammaPlan
        from paper_1503_08809_b200.quadrature import x_weights
        q, qt, C, v, x, entries, dom, alpha = self._small(8)
        lmax = q.shape[1] + 1
        t = BasisTables(q, qt, C, v, 2, lmax)
        one = gamma_nonsep(t, ModeMapping(entries, 8), RadialGrid(x), alpha, dom).values[:, 0]
        plan = GammaPlan(q, qt, C, v, x_weights(x, "trap"), entries, 2, lmax)
        plan.set_sparse_domain(dom)
        b1 = plan.nonsep(alpha)
        b2 = plan.nonsep(alpha)
        assert np.array_equal(b1, b2)
        assert np.array_equal(b1, one)
        b3 = plan.nonsep(2.0 * alpha - 0.5 * alpha)   # linear in α
        assert np.linalg.norm(b3 - 1.5 * b1) <= 1e-13 * np.linalg.norm(b1)
        out = torch.zeros(entries.shape[0], dtype=torch.float64, device="cuda")
        plan.nonsep(alpha, out=out)
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy(), b1)
        plan.set_sparse_domain(SparseDomain([], [], [], []))
        assert not plan.nonsep(alpha).any()
        with pytest.raises(ValueError):
            plan.nonsep(alpha[:-1])
        with pytest.raises(ValueError):
            plan.set_sparse_domain(SparseDomain([5], [3], [4], [1.0]))
        plan.close()
