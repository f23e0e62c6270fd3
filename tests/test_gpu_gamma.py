"""GPU parity of the separable Γ path against the oracle and the reference's golden vectors.

Mirrors the reference's hot-path tests (pkg/tests/test_engine3d.py, test_geometry.py,
test_acceptance.py criteria 3, 4, 7) but runs the CUDA library through the drop-in API.
Tolerances: weights and enumeration bit-exact; Γ relative Frobenius <= 1e-10 (north_star);
the reference's own 1e-12 relative_gap is also asserted where it applies.
"""

import numpy as np
import pytest

from conftest import frob_rel, gap_rel
from oracle import ref
from paper_1503_08809_b200 import (BasisTables, DomainRange, GammaPlan, ModeMapping,
                                   RadialGrid, domain_count, domain_triples, gamma3d_matrix,
                                   triple_weights, x_weights)
from paper_1503_08809_b200.configs import host_inputs

pytestmark = pytest.mark.gpu


def desk_problem(g, tag):
    lmin, lmax = (int(x) for x in g[f"{tag}_lrange"])
    t = BasisTables(g[f"{tag}_q"], g[f"{tag}_qt"], g[f"{tag}_C"], g[f"{tag}_v"], lmin, lmax)
    m = ModeMapping(g[f"{tag}_entries"], t.p_max)
    r = RadialGrid(g[f"{tag}_r"])
    return t, m, r


class TestDomainAndWeights:
    def test_counts(self, g_domain):
        for m, c in zip(g_domain["count_lmax"], g_domain["count"]):
            assert domain_count(2, int(m)) == int(c)

    def test_enumeration_golden(self, g_domain):
        got = np.stack(domain_triples(2, 4), 1)
        assert np.array_equal(got, g_domain["triples_2_4"])
        a, b, c = domain_triples(3, 40)
        assert np.array_equal(a, g_domain["l1_3_40"])
        assert np.array_equal(b, g_domain["l2_3_40"])
        assert np.array_equal(c, g_domain["l3_3_40"])

    @pytest.mark.parametrize("lmax,begin,end", [(200, 0, None), (2000, 0, 200000),
                                                 (2000, 167_000_000, 167_250_000),
                                                 (3000, 1_128_000_000, None)])
    def test_enumeration_vs_oracle(self, lmax, begin, end):
        end = domain_count(2, lmax) if end is None else end
        got = domain_triples(2, lmax, begin, end)
        want = ref.domain_triples(2, lmax, begin, end)
        for x, y in zip(got, want):
            assert np.array_equal(x, y)

    def test_weights_bit_exact_golden(self, g_domain):
        zm = triple_weights(g_domain["zm64_C"], g_domain["zm64_v"], 2, 64)
        assert np.array_equal(zm, g_domain["zm64"])          # bitwise, NumPy order

    def test_weights_exact_mode(self, g_domain):
        zm = triple_weights(g_domain["zm64_C"], g_domain["zm64_v"], 2, 64, h2_mode="exact")
        assert np.max(np.abs(zm / g_domain["zm64_exact"] - 1)) < 1e-13

    @pytest.mark.parametrize("lmax,begin,end", [(200, 0, None), (2000, 250_000_000, 250_400_000)])
    def test_weights_bit_exact_large(self, lmax, begin, end):
        rng = np.random.default_rng(11)
        C = rng.uniform(1e-6, 1e-1, lmax - 1)
        v = (2.0 * np.arange(2, lmax + 1) + 1.0) ** (1.0 / 6.0)
        end = domain_count(2, lmax) if end is None else end
        zm = triple_weights(C, v, 2, lmax, begin, end)
        l1, l2, l3 = ref.domain_triples(2, lmax, begin, end)
        assert np.array_equal(zm, ref.zm_c(2, l1, l2, l3, C, v))
        assert np.array_equal(zm, ref.triple_zm(2, l1, l2, l3, C, v))

    def test_zm_222_unit(self, g_domain):
        zm = triple_weights(np.ones(1), np.ones(1), 2, 2)
        assert zm[0] == g_domain["z222_unit"]                 # mult(2,2,2) = 1
        assert abs(zm[0] - 0.016088) < 2e-6                   # test_geometry.py:175-179

    def test_rejects_nonpositive_spectrum(self):
        with pytest.raises(ValueError):
            triple_weights(np.zeros(1), np.ones(1), 2, 2)


class TestGammaDesk:
    """test_engine3d.py TestBlockedVsNaive / TestOrderedEnumeration on the GPU."""

    @pytest.mark.parametrize("tag", ["desk", "desk32", "small12"])
    def test_matches_reference(self, g_desk, tag):
        t, m, r = desk_problem(g_desk, tag)
        got = gamma3d_matrix(t, m, r).values
        assert gap_rel(got, g_desk[f"{tag}_gamma"]) < 1e-12
        assert frob_rel(got, g_desk[f"{tag}_gamma"]) < 1e-12

    def test_matches_naive(self, g_desk):
        t, m, r = desk_problem(g_desk, "desk")
        assert gap_rel(gamma3d_matrix(t, m, r).values, g_desk["desk_naive"]) < 1e-12

    def test_ordered_equals_unordered(self, g_desk):
        t, m, r = desk_problem(g_desk, "small12")
        assert gap_rel(gamma3d_matrix(t, m, r).values, g_desk["small12_unordered"]) < 1e-12

    @pytest.mark.parametrize("integrator", ["hermite", "spline"])
    def test_other_integrators(self, g_desk, integrator):
        t, m, r = desk_problem(g_desk, "desk")
        got = gamma3d_matrix(t, m, r, integrator=integrator).values
        assert gap_rel(got, g_desk[f"desk_{integrator}"]) < 1e-12

    def test_exact_mode(self, g_desk):
        t, m, r = desk_problem(g_desk, "desk")
        got = gamma3d_matrix(t, m, r, h2_mode="exact").values
        assert gap_rel(got, g_desk["desk_exact"]) < 1e-12

    def test_block_and_workers_are_metadata(self, g_desk):
        t, m, r = desk_problem(g_desk, "desk32")
        a = gamma3d_matrix(t, m, r, block=7, workers=4)
        assert gap_rel(a.values, g_desk["desk32_w4"]) < 1e-12
        assert a.meta["block"] == 7 and a.meta["workers"] == 4
        assert a.meta["engine"] == "modal3d" and a.meta["tables"] == t.fingerprint()

    def test_bitwise_reproducible(self, g_desk):
        t, m, r = desk_problem(g_desk, "desk32")
        a = gamma3d_matrix(t, m, r).values
        b = gamma3d_matrix(t, m, r).values
        assert np.array_equal(a, b)

    def test_errors(self, g_desk):
        t, m, r = desk_problem(g_desk, "desk")
        with pytest.raises(ValueError):
            gamma3d_matrix(t, m, r, h2_mode="asymptotic")
        with pytest.raises(ValueError):
            gamma3d_matrix(t, m, r, block=0)

    def test_explicit_noncontiguous_domain(self, g_desk):
        t, m, r = desk_problem(g_desk, "desk32")
        l1, l2, l3 = ref.domain_triples(2, 32)
        keep = (np.arange(l1.size) % 3) != 1

        class Dom:
            pass

        d = Dom()
        d.l1, d.l2, d.l3 = l1[keep], l2[keep], l3[keep]
        d.count = int(keep.sum())
        got = gamma3d_matrix(t, m, r, domain=d).values
        want = ref.sweep_triples(t.q, t.q_tilde, t.C, t.v, x_weights(r.r), m.entries, 2,
                                 d.l1, d.l2, d.l3)
        assert frob_rel(got, want) < 1e-12

    def test_empty_range(self, g_desk):
        t, m, r = desk_problem(g_desk, "desk")
        got = gamma3d_matrix(t, m, r, domain=DomainRange(2, 16, 5, 5)).values
        assert not got.any()


class TestGammaC0:
    def tables(self, g_c0):
        hi = host_inputs("c0")
        t = BasisTables(hi.q, g_c0["qt"], g_c0["C"], hi.v, 2, 200)
        return t, ModeMapping(hi.entries, hi.spec.p), RadialGrid(hi.x)

    def test_full_gamma(self, g_c0):
        t, m, r = self.tables(g_c0)
        got = gamma3d_matrix(t, m, r).values
        assert frob_rel(got, g_c0["gamma"]) < 1e-10
        assert gap_rel(got, g_c0["gamma"]) < 1e-12

    @pytest.mark.parametrize("a,b", [(0, 1000), (1000, 20000), (200000, 348151)])
    def test_flat_range_partials(self, g_c0, a, b):
        t, m, r = self.tables(g_c0)
        got = gamma3d_matrix(t, m, r, domain=DomainRange(2, 200, a, b)).values
        assert frob_rel(got, g_c0[f"partial_{a}_{b}"]) < 1e-10

    def test_exact_mode(self, g_c0):
        t, m, r = self.tables(g_c0)
        got = gamma3d_matrix(t, m, r, h2_mode="exact").values
        assert frob_rel(got, g_c0["gamma_exact"]) < 1e-10

    def test_slabs_add_up(self, g_c0):
        t, m, r = self.tables(g_c0)
        plan = GammaPlan.from_tables(t, m, r)
        total = np.zeros((56, 56))
        for a, b in ((2, 60), (60, 131), (131, 201)):
            plan.execute(a, b)
            total += plan.fetch()
        assert frob_rel(total, g_c0["gamma"]) < 1e-12


@pytest.fixture(scope="module")
def c1():
    from paper_1503_08809_b200 import build_qtilde
    hi = host_inputs("c1")
    C, qt = build_qtilde(hi)
    return hi, C, qt


class TestGammaLarge:
    """Config-1 scale: flat-range partials vs the oracle on the same (GPU-built) q̃."""

    @pytest.mark.parametrize("frac", [0.1, 0.5, 0.9])
    def test_partial_vs_oracle(self, c1, frac):
        hi, C, qt = c1
        total = domain_count(2, hi.l_max)
        a = int(frac * total)
        b = a + 1500                  # the long-window regime is tests/test_gpu_parity_long.py
        t = BasisTables(hi.q, qt, C, hi.v, 2, hi.l_max)
        m = ModeMapping(hi.entries, hi.spec.p)
        got = gamma3d_matrix(t, m, RadialGrid(hi.x), domain=DomainRange(2, hi.l_max, a, b)).values
        want = ref.gamma3d(hi.q, qt, C, hi.v, hi.wr2, hi.entries, 2, hi.l_max, a, b, workers=8)
        assert frob_rel(got, want) < 1e-10

    def test_slab_partition_is_exact(self, c1):
        """Size-independent property at full c1 size: l2 slabs sum to the full Γ."""
        hi, C, qt = c1
        plan = GammaPlan(hi.q, qt, C, hi.v, hi.wr2, hi.entries, 2, hi.l_max)
        plan.execute()
        full = plan.fetch()
        bounds = [2, 700, 1300, hi.l_max + 1]
        parts = []
        for a, b in zip(bounds[:-1], bounds[1:]):
            plan.execute(a, b)
            parts.append(plan.fetch())
        assert frob_rel(sum(parts), full) < 1e-12
        plan.execute()
        assert np.array_equal(plan.fetch(), full)              # bitwise reproducible

    def test_async_executes_into_device_buffers(self, c1):
        """mg_plan_execute is asynchronous: back-to-back executes into device tensors on a
        side stream, no host sync in between, match the synchronous per-slab results."""
        import torch
        hi, C, qt = c1
        plan = GammaPlan(hi.q, qt, C, hi.v, hi.wr2, hi.entries, 2, hi.l_max)
        n = hi.entries.shape[0]
        bounds = [(2, 400), (400, 800), (800, 1000)]
        want = []
        for a, b in bounds:
            plan.execute(a, b)
            want.append(plan.fetch())
        s = torch.cuda.Stream()
        outs = [torch.empty((n, n), dtype=torch.float64, device="cuda") for _ in bounds]
        with torch.cuda.stream(s):
            for (a, b), o in zip(bounds, outs):
                plan.execute(a, b, out=o, stream=s)
        s.synchronize()
        for o, w in zip(outs, want):
            assert np.array_equal(o.cpu().numpy(), w)
        plan.set_profile(True)
        plan.execute(2, 400, stream=s)
        ms = plan.kernel_ms()                                  # resolves the pending events
        assert ms["run"] > 0 and ms["x"] > 0


@pytest.mark.parametrize("cfg,ntri", [("c2", 750), ("c4", 80)])
def test_large_config_partials(cfg, ntri):
    """Configs 2 and 4 (p = 22, 30: several M-tiles in the x/pair contractions, packed
    slots spanning rows): flat-range partials at 30 % and 80 % of the index vs the oracle on
    the same GPU-built q̃."""
    from paper_1503_08809_b200 import build_qtilde
    hi = host_inputs(cfg)
    C, qt = build_qtilde(hi)
    t = BasisTables(hi.q, qt, C, hi.v, 2, hi.l_max)
    m = ModeMapping(hi.entries, hi.spec.p)
    total = domain_count(2, hi.l_max)
    for frac in (0.3, 0.8):
        a = int(frac * total)
        got = gamma3d_matrix(t, m, RadialGrid(hi.x),
                             domain=DomainRange(2, hi.l_max, a, a + ntri)).values
        want = ref.gamma3d(hi.q, qt, C, hi.v, hi.wr2, hi.entries, 2, hi.l_max, a, a + ntri,
                           workers=8, block=8)
        assert frob_rel(got, want) < 1e-10


class TestLateLate:
    """⟨Q,Q⟩ = the Γ' engine with q̃ -> q, one x point, C -> v²."""

    def oracle(self, t, m, h2_mode="gosper"):
        qt = t.q[:, None, :]
        return ref.gamma3d(t.q, qt, t.v * t.v, t.v, np.ones(1), m.entries, t.l_min, t.l_max,
                           h2_mode=h2_mode)

    @pytest.mark.parametrize("tag", ["desk", "desk32"])
    def test_against_oracle(self, g_desk, tag):
        from paper_1503_08809_b200 import gamma_late_late
        t, m, r = desk_problem(g_desk, tag)
        got = gamma_late_late(t, m).values
        want = self.oracle(t, m)
        assert frob_rel(got, want) < 1e-12
        assert np.allclose(got, got.T, rtol=1e-12, atol=0)       # symmetric inner product

    def test_c0_and_estimator(self, g_c0):
        from paper_1503_08809_b200 import gamma_estimator
        hi = host_inputs("c0")
        t = BasisTables(hi.q, g_c0["qt"], g_c0["C"], hi.v, 2, 200)
        m = ModeMapping(hi.entries, 6)
        full, qq, gp = gamma_estimator(t, m, RadialGrid(hi.x))
        assert frob_rel(qq.values, self.oracle(t, m)) < 1e-12
        assert frob_rel(gp.values, g_c0["gamma"]) < 1e-10
        assert frob_rel(qq.values @ full.values, g_c0["gamma"]) < 1e-9
        assert np.all(np.linalg.eigvalsh(qq.values) > 0)           # positive definite


class TestGamma2D:
    """μ-quadrature engine vs the reference's engine2d (golden io2d.npz) and the
    2D ≡ 3D-exact identity (acceptance criterion 1, test_acceptance.py:50-57)."""

    def setup(self, g_desk, g2, tag, nmu):
        from paper_1503_08809_b200 import gauss_legendre, legendre_table
        t, m, r = desk_problem(g_desk, tag)
        rule = gauss_legendre(nmu)
        assert np.array_equal(rule.nodes, g2[f"{tag}_mu_nodes"])
        return t, m, r, rule, legendre_table(t.l_max, rule)

    @pytest.mark.parametrize("tag,nmu", [("desk", 27), ("desk32", 50)])
    def test_ptable_bit_exact(self, g_desk, tag, nmu):
        from conftest import golden
        from paper_1503_08809_b200 import build_ptable
        g2 = golden("io2d.npz")
        t, m, r, rule, leg = self.setup(g_desk, g2, tag, nmu)
        assert np.array_equal(build_ptable(t, r, rule, leg).values, g2[f"{tag}_ptable"])

    @pytest.mark.parametrize("tag,nmu", [("desk", 27), ("desk32", 50)])
    def test_gamma2d(self, g_desk, tag, nmu):
        from conftest import golden
        from paper_1503_08809_b200 import build_ptable, gamma2d_matrix
        g2 = golden("io2d.npz")
        t, m, r, rule, leg = self.setup(g_desk, g2, tag, nmu)
        got = gamma2d_matrix(t, m, r, rule, leg)
        assert gap_rel(got.values, g2[f"{tag}_gamma2d"]) < 1e-12
        assert got.meta["engine"] == "modal2d" and got.meta["n_mu"] == nmu
        pt = build_ptable(t, r, rule, leg)
        again = gamma2d_matrix(t, m, r, rule, leg, ptable=pt).values
        assert np.array_equal(again, got.values)
        # criterion 1: separable (2D) == direct with exact weights (3D-exact)
        g3 = gamma3d_matrix(t, m, r, h2_mode="exact").values
        assert gap_rel(got.values, g3) < 1e-10

    @pytest.mark.parametrize("lds", [False, True])
    @pytest.mark.parametrize("lmin,lmax,p,nx,nmu", [(2, 70, 5, 37, 107),    # 3 l chunks, 2 μ tiles
                                                     (3, 34, 7, 19, 65),     # 33 = 32 + 1 rows of l
                                                     (2, 150, 3, 130, 228),  # 19 row tiles
                                                     (2, 30, 8, 23, 50),     # p = 8: 8 m-fragments
                                                     (2, 24, 9, 11, 40),     # p > 8: 2 M tiles
                                                     (2, 20, 12, 7, 30),     # 3 M tiles, 64-sample chunks
                                                     (2, 18, 15, 5, 24),     # 4 M tiles, 32-sample chunks
                                                     (2, 14, 20, 3, 20),     # 7 M tiles, 16-sample chunks
                                                     (2, 12, 25, 2, 12),     # beyond the DMMA form
                                                     (2, 12, 1, 5, 20),      # one mode
                                                     (2, 40, 2, 9, 64)])
    def test_tiled_kernels_vs_oracle(self, lmin, lmax, p, nx, nmu, lds, monkeypatch):
        """Sizes that cross every tile edge of the P-table kernel (64 x 64 x 32: partial row,
        column and l tiles) and of both cell kernels — the DMMA form (p <= 8: partial
        m-fragments, partial n-fragments, idle warps, split-K with a short last chunk,
        several M tiles for p > 8) and the per-cell form (MG_G2D_LDS=1 or p > 24: x chunks per CTA, μ chunks of 64, partial 16 x 16
        cell tiles) — against oracle/gamma2d_ref.py (pinned to the reference's tables)."""
        from oracle import gamma2d_ref
        if lds:
            monkeypatch.setenv("MG_G2D_LDS", "1")
        else:
            monkeypatch.delenv("MG_G2D_LDS", raising=False)
        from paper_1503_08809_b200 import (build_ptable, default_mode_mapping, gamma2d_matrix,
                                           gauss_legendre, legendre_table)
        t, r = TestEdgeCases().random_tables(lmin, lmax, p, nx, seed=11)
        m = default_mode_mapping(p)
        rule = gauss_legendre(nmu)
        leg = legendre_table(lmax, rule)
        want_p = gamma2d_ref.ptable(t.q, t.q_tilde, t.C, t.v, lmin, lmax, leg)
        pt = build_ptable(t, r, rule, leg)
        assert np.array_equal(pt.values, want_p)
        want = gamma2d_ref.gamma2d(want_p, m.entries, rule.weights, x_weights(r.r))
        got = gamma2d_matrix(t, m, r, rule, leg).values
        assert gap_rel(got, want) < 1e-12
        assert np.array_equal(gamma2d_matrix(t, m, r, rule, leg, ptable=pt).values, got)

    @pytest.mark.parametrize("lds", [False, True])
    def test_custom_mode_subset(self, lds, monkeypatch):
        """A mapping that is not the default k-major list (repeated indices, gaps, arbitrary
        order) through both cell kernels."""
        from oracle import gamma2d_ref
        from paper_1503_08809_b200 import gamma2d_matrix, gauss_legendre, legendre_table
        if lds:
            monkeypatch.setenv("MG_G2D_LDS", "1")
        else:
            monkeypatch.delenv("MG_G2D_LDS", raising=False)
        t, r = TestEdgeCases().random_tables(2, 28, 6, 17, seed=5)
        entries = np.array([[5, 5, 5], [0, 0, 0], [0, 2, 4], [1, 1, 3], [0, 1, 2], [2, 3, 5],
                            [3, 3, 4]])
        m = ModeMapping(entries, 6)
        rule = gauss_legendre(45)
        leg = legendre_table(28, rule)
        P = gamma2d_ref.ptable(t.q, t.q_tilde, t.C, t.v, 2, 28, leg)
        want = gamma2d_ref.gamma2d(P, entries, rule.weights, x_weights(r.r))
        got = gamma2d_matrix(t, m, r, rule, leg).values
        assert got.shape == (7, 7)
        assert gap_rel(got, want) < 1e-12

    def test_kernel_timings_hook(self, g_desk):
        from paper_1503_08809_b200 import build_ptable, gamma2d_matrix, gauss_legendre, legendre_table
        from paper_1503_08809_b200.engine2d import last_kernel_ms
        t, m, r = desk_problem(g_desk, "desk")
        rule = gauss_legendre(27)
        leg = legendre_table(t.l_max, rule)
        gamma2d_matrix(t, m, r, rule, leg)
        a, b = last_kernel_ms()
        assert a > 0 and b > 0
        pt = build_ptable(t, r, rule, leg)
        a, b = last_kernel_ms()
        assert a > 0 and b == 0
        gamma2d_matrix(t, m, r, rule, leg, ptable=pt)
        a, b = last_kernel_ms()
        assert a == 0 and b > 0

    def test_budget_and_errors(self, g_desk):
        from paper_1503_08809_b200 import build_ptable, gauss_legendre, legendre_table
        t, m, r = desk_problem(g_desk, "desk")
        rule = gauss_legendre(27)
        with pytest.raises(MemoryError):
            build_ptable(t, r, rule, legendre_table(16, rule), budget_bytes=1000)
        with pytest.raises(ValueError):
            build_ptable(t, r, rule, legendre_table(10, rule))


class TestEdgeCases:
    """Shapes the configs do not exercise: l_min > 2, odd Nx on a non-uniform grid (the
    padded-x paths), a custom mode subset, p = 1, the single-triple domain (l_min = l_max)."""

    def random_tables(self, lmin, lmax, p, nx, seed=0):
        from paper_1503_08809_b200 import shifted_legendre
        rng = np.random.default_rng(seed)
        L = lmax - lmin + 1
        q = shifted_legendre(p, lmin, lmax)
        qt = rng.standard_normal((p, nx, L)) * 1e-3
        C = rng.uniform(0.5, 2.0, L) * 1e-3
        ells = np.arange(lmin, lmax + 1, dtype=np.float64)
        v = (2.0 * ells + 1.0) ** (1.0 / 6.0)
        r = np.cumsum(rng.uniform(0.5, 1.5, nx)) + 100.0
        return BasisTables(q, qt, C, v, lmin, lmax), RadialGrid(r)

    @pytest.mark.parametrize("lmin,lmax,p,nx,integ", [(3, 20, 4, 37, "spline"),
                                                      (5, 41, 3, 33, "trap"),
                                                      (2, 9, 1, 7, "hermite"),
                                                      (2, 2, 2, 5, "trap"),
                                                      (4, 4, 3, 9, "trap")])
    def test_against_oracle(self, lmin, lmax, p, nx, integ):
        from paper_1503_08809_b200 import default_mode_mapping
        t, r = self.random_tables(lmin, lmax, p, nx)
        m = default_mode_mapping(p)
        got = gamma3d_matrix(t, m, r, integrator=integ).values
        want = ref.gamma3d(t.q, t.q_tilde, t.C, t.v, x_weights(r.r, integ), m.entries, lmin,
                           lmax)
        if not np.any(want):
            assert not np.any(got)
        else:
            assert frob_rel(got, want) < 1e-12

    def test_custom_mode_subset(self):
        t, r = self.random_tables(2, 30, 5, 41, seed=3)
        entries = np.array([[0, 0, 0], [0, 2, 4], [1, 1, 3], [4, 4, 4], [0, 1, 2], [2, 3, 4]])
        m = ModeMapping(entries, 5)
        got = gamma3d_matrix(t, m, r).values
        want = ref.gamma3d(t.q, t.q_tilde, t.C, t.v, x_weights(r.r), entries, 2, 30)
        assert got.shape == (6, 6)
        assert frob_rel(got, want) < 1e-12

    def test_lmin_odd_flat_ranges(self):
        from paper_1503_08809_b200 import default_mode_mapping
        t, r = self.random_tables(3, 25, 3, 16, seed=5)
        m = default_mode_mapping(3)
        total = domain_count(3, 25)
        for a, b in ((0, 1), (7, 93), (total - 5, total)):
            got = gamma3d_matrix(t, m, r, domain=DomainRange(3, 25, a, b)).values
            want = ref.gamma3d(t.q, t.q_tilde, t.C, t.v, x_weights(r.r), m.entries, 3, 25, a, b)
            assert frob_rel(got, want) < 1e-12


class TestMultiDevice:
    """gamma3d_matrix over several devices inside the unchanged call (engine3d.py:175-186's
    fork pool with GPUs for workers).  One GPU here, so the shards are `devices=[0, 0]`: the
    host threads, the per-shard plans, the l2-slab split and the ordered merge all run; the
    shards serialise on the device's execute lock."""

    def test_full_domain_two_shards_c0(self, g_c0):
        from paper_1503_08809_b200 import slab_plan
        hi = host_inputs("c0")
        t = BasisTables(hi.q, g_c0["qt"], g_c0["C"], hi.v, 2, 200)
        m, r = ModeMapping(hi.entries, 6), RadialGrid(hi.x)
        one = gamma3d_matrix(t, m, r, devices=[0])
        two = gamma3d_matrix(t, m, r, devices=[0, 0])
        assert two.meta["devices"] == [0, 0] and one.meta["devices"] == [0]
        b = slab_plan(2, 200, 6, hi.x.size, 2)
        plan = GammaPlan.from_tables(t, m, r)
        parts = []
        for a, e in zip(b[:-1], b[1:]):
            plan.execute(a, e)
            parts.append(plan.fetch())
        want = parts[0].copy()
        want += parts[1]
        assert np.array_equal(two.values, want)             # = the two-slab sum, bitwise
        assert frob_rel(two.values, one.values) < 1e-12
        assert frob_rel(two.values, g_c0["gamma"]) < 1e-10

    def test_full_domain_four_shards_c1(self, c1):
        hi, C, qt = c1
        t = BasisTables(hi.q, qt, C, hi.v, 2, hi.l_max)
        m, r = ModeMapping(hi.entries, hi.spec.p), RadialGrid(hi.x)
        one = gamma3d_matrix(t, m, r, devices=[0]).values
        four = gamma3d_matrix(t, m, r, devices=[0, 0, 0, 0]).values
        assert frob_rel(four, one) < 1e-12
        again = gamma3d_matrix(t, m, r, devices=[0, 0, 0, 0]).values
        assert np.array_equal(four, again)                   # reproducible per device list

    def test_subrange_and_triples_sharded(self, g_c0):
        hi = host_inputs("c0")
        t = BasisTables(hi.q, g_c0["qt"], g_c0["C"], hi.v, 2, 200)
        m, r = ModeMapping(hi.entries, 6), RadialGrid(hi.x)
        d = DomainRange(2, 200, 1000, 20000)
        got = gamma3d_matrix(t, m, r, domain=d, devices=[0, 0, 0]).values
        assert frob_rel(got, g_c0["partial_1000_20000"]) < 1e-10
        l1, l2, l3 = ref.domain_triples(2, 200)
        keep = (np.arange(l1.size) % 5) != 2

        class Dom:
            pass

        dd = Dom()
        dd.l1, dd.l2, dd.l3 = l1[keep], l2[keep], l3[keep]
        dd.count = int(keep.sum())
        a = gamma3d_matrix(t, m, r, domain=dd, devices=[0]).values
        b = gamma3d_matrix(t, m, r, domain=dd, devices=[0, 0]).values
        assert frob_rel(b, a) < 1e-12


def test_large_basis_beyond_32():
    """p_max = 40 (> 32: the reference accepts any p_max, basis.py:57-94): stage 1 in
    component blocks vs scipy, and the separable Γ on a 160-mode subset mapping vs the
    oracle (P2 = 820 pairs, p^2 = 1600 (c,c') columns, several M/N tiles per row)."""
    from dataclasses import replace
    from oracle import qtilde_ref
    from paper_1503_08809_b200 import build_qtilde, default_mode_mapping
    from paper_1503_08809_b200.basis import legendre_on_interval, shifted_legendre
    p = 40
    hi = host_inputs("c0", l_max=48)
    qk = legendre_on_interval(p, hi.k, hi.spec.k_range[0],
                              hi.spec.k_range[1] - hi.spec.k_range[0])
    hi = replace(hi, qk=qk, q=shifted_legendre(p, 2, 48))
    C, qt = build_qtilde(hi)
    d = qtilde_ref.delta_table(hi.k, hi.eps, 2, 48)
    ells = [2, 25, 48]
    want = qtilde_ref.qtilde(hi.k, hi.wk, hi.x, hi.qk, d, 2, 48, ells)
    for l in ells:
        a, b = qt[:, :, l - 2], want[:, :, l - 2]
        assert np.linalg.norm(a - b) <= 1e-11 * np.linalg.norm(b), l
    full = default_mode_mapping(p).entries
    rng = np.random.default_rng(4)
    sub = full[np.unique(np.concatenate([[0, full.shape[0] - 1],
                                         rng.choice(full.shape[0], 158, replace=False)]))]
    t = BasisTables(hi.q, qt, C, hi.v, 2, 48)
    m = ModeMapping(sub, p)
    got = gamma3d_matrix(t, m, RadialGrid(hi.x)).values
    ref_g = ref.gamma3d(hi.q, qt, C, hi.v, hi.wr2, sub, 2, 48, workers=8, block=32)
    assert got.shape == (sub.shape[0], sub.shape[0])
    assert frob_rel(got, ref_g) < 1e-12


@pytest.mark.parametrize("p", [15, 22, 30])
def test_every_x_contraction_tile(p, monkeypatch):
    """Every x-contraction tile (MG_XTILE = 0..7, incl. the N-split forms whose partial last
    N tile is dealt over the warp columns; a forced N-split tile that does not fit the basis
    falls back to the automatic choice) against the oracle at the benchmark basis sizes, on a
    small domain with Nx = 100 (the last k-tile is partial) and a mode subset that keeps the
    first and last modes."""
    from dataclasses import replace
    from paper_1503_08809_b200 import build_qtilde, default_mode_mapping
    from paper_1503_08809_b200.basis import legendre_on_interval, shifted_legendre
    lmax = 30
    hi = host_inputs("c0", l_max=lmax)
    qk = legendre_on_interval(p, hi.k, hi.spec.k_range[0],
                              hi.spec.k_range[1] - hi.spec.k_range[0])
    hi = replace(hi, qk=qk, q=shifted_legendre(p, 2, lmax))
    C, qt = build_qtilde(hi)
    full = default_mode_mapping(p).entries
    rng = np.random.default_rng(p)
    sub = full[np.unique(np.concatenate([[0, full.shape[0] - 1],
                                         rng.choice(full.shape[0], 118, replace=False)]))]
    t = BasisTables(hi.q, qt, C, hi.v, 2, lmax)
    m = ModeMapping(sub, p)
    want = ref.gamma3d(hi.q, qt, C, hi.v, hi.wr2, sub, 2, lmax, workers=8, block=32)
    auto = gamma3d_matrix(t, m, RadialGrid(hi.x)).values
    assert frob_rel(auto, want) < 1e-12
    for tile in range(8):
        monkeypatch.setenv("MG_XTILE", str(tile))
        got = gamma3d_matrix(t, m, RadialGrid(hi.x)).values
        assert frob_rel(got, want) < 1e-12, tile


@pytest.mark.parametrize("p", [7, 10, 13, 16, 18, 19, 21, 24, 27, 32])
def test_basis_sizes_automatic_tile(p):
    """Basis sizes between the benchmark ones: whatever x-contraction tile choose_xtile picks
    (plain or N-split, partial M and N tiles, 1 to 3 n-fragments dealt per warp column) against
    the oracle on a small domain with a 60-mode subset mapping."""
    from dataclasses import replace
    from paper_1503_08809_b200 import build_qtilde, default_mode_mapping
    from paper_1503_08809_b200.basis import legendre_on_interval, shifted_legendre
    lmax = 22
    hi = host_inputs("c0", l_max=lmax)
    qk = legendre_on_interval(p, hi.k, hi.spec.k_range[0],
                              hi.spec.k_range[1] - hi.spec.k_range[0])
    hi = replace(hi, qk=qk, q=shifted_legendre(p, 2, lmax))
    C, qt = build_qtilde(hi)
    full = default_mode_mapping(p).entries
    rng = np.random.default_rng(100 + p)
    sub = full[np.unique(np.concatenate([[0, full.shape[0] - 1],
                                         rng.choice(full.shape[0], 58, replace=False)]))]
    got = gamma3d_matrix(BasisTables(hi.q, qt, C, hi.v, 2, lmax), ModeMapping(sub, p),
                         RadialGrid(hi.x)).values
    want = ref.gamma3d(hi.q, qt, C, hi.v, hi.wr2, sub, 2, lmax, workers=4, block=32)
    assert frob_rel(got, want) < 1e-12


def test_distributed_nccl_path_world1(g_c0):
    """The torchrun path (dist.gamma3d_matrix_distributed) with a real NCCL communicator:
    partial Γ written by the plan straight into device memory, all-gathered over NCCL and
    summed in rank order (world size 1 on one GPU; the N > 1 host logic is the gloo test)."""
    import socket

    import torch
    import torch.distributed as dist

    from paper_1503_08809_b200.dist import gamma3d_matrix_distributed
    hi = host_inputs("c0")
    t = BasisTables(hi.q, g_c0["qt"], g_c0["C"], hi.v, 2, 200)
    m, r = ModeMapping(hi.entries, 6), RadialGrid(hi.x)
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0,
                            world_size=1, device_id=torch.device("cuda", 0))
    try:
        g = gamma3d_matrix_distributed(t, m, r, device=0)
    finally:
        dist.destroy_process_group()
    assert g.meta["ranks"] == 1
    assert frob_rel(g.values, g_c0["gamma"]) < 1e-10
    assert frob_rel(g.values, gamma3d_matrix(t, m, r, devices=[0]).values) < 1e-13
