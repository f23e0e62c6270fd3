"""CPU: pin the oracle against the reference's golden vectors and known-answer tests.

Golden vectors come from the unmodified reference (tests/golden/make_golden.py); the
known answers are the reference's own (pkg/tests/test_geometry.py, test_engine3d.py,
test_scheduler.py).  Everything here runs without a GPU.
"""

import math

import numpy as np
import pytest

from conftest import frob_rel, gap_rel
from oracle import ref
from paper_1503_08809_b200.configs import host_inputs
from paper_1503_08809_b200.quadrature import x_weights


class TestEnumeration:
    def test_counts(self, g_domain):
        for m, c in zip(g_domain["count_lmax"], g_domain["count"]):
            assert ref.domain_count(2, int(m)) == int(c)

    def test_counts_large(self):
        # SURVEY.md §8a (measured with the reference enumeration)
        assert ref.domain_count(2, 2000) == 334_831_501
        assert ref.domain_count(2, 64) == 12401            # acceptance criterion 9

    def test_lmax4_golden(self, g_domain):                 # test_geometry.py:187-192
        got = np.stack(ref.domain_triples(2, 4), 1)
        assert np.array_equal(got, g_domain["triples_2_4"])
        assert got.tolist() == [[2, 2, 2], [2, 2, 4], [2, 3, 3], [2, 4, 4], [3, 3, 4], [4, 4, 4]]

    def test_lmin3(self, g_domain):
        a, b, c = ref.domain_triples(3, 40)
        assert np.array_equal(a, g_domain["l1_3_40"])
        assert np.array_equal(b, g_domain["l2_3_40"])
        assert np.array_equal(c, g_domain["l3_3_40"])

    def test_slices_concatenate(self):
        whole = ref.domain_triples(2, 30)
        parts = [ref.domain_triples(2, 30, a, b) for a, b in ((0, 17), (17, 400), (400, 1340))]
        for i in range(3):
            assert np.array_equal(whole[i][:1340], np.concatenate([p[i] for p in parts]))


class TestWeights:
    def test_c_bit_exact(self, g_domain):
        l1, l2, l3 = ref.domain_triples(2, 64)
        zm = ref.zm_c(2, l1, l2, l3, g_domain["zm64_C"], g_domain["zm64_v"])
        assert np.array_equal(zm, g_domain["zm64"])

    def test_numpy_port_bit_exact(self, g_domain):
        l1, l2, l3 = ref.domain_triples(2, 64)
        zm = ref.triple_zm(2, l1, l2, l3, g_domain["zm64_C"], g_domain["zm64_v"])
        assert np.array_equal(zm, g_domain["zm64"])

    def test_exact_mode(self, g_domain):
        l1, l2, l3 = ref.domain_triples(2, 64)
        zm = ref.triple_zm(2, l1, l2, l3, g_domain["zm64_C"], g_domain["zm64_v"], "exact")
        assert np.max(np.abs(zm / g_domain["zm64_exact"] - 1)) < 1e-14

    def test_known_answers(self, g_domain):
        # h2(2,2,2) = 25/(14 pi) (test_geometry.py:67-71); z(2,2,2) = 0.016088 (:175-179)
        assert ref.h2_exact(2, 2, 2)[0] == pytest.approx(25 / (14 * math.pi), rel=1e-14)
        assert float(ref.h2_gosper(2, 2, 2)) == g_domain["h2g_222"]
        assert abs(float(ref.h2_gosper(2, 2, 2)) / (25 / (14 * math.pi)) - 1) \
            == pytest.approx(0.019, abs=0.002)
        z = ref.zm_c(2, [2], [2], [2], np.ones(1), np.ones(1))[0]
        assert z == g_domain["z222_unit"] and abs(z - 0.016088) < 2e-6

    def test_multiplicity(self):
        assert ref.multiplicity([2, 2, 2, 2], [2, 2, 4, 3], [2, 4, 4, 5]).tolist() == [1, 3, 3, 6]


class TestGammaPort:
    def desk(self, g, tag):
        lmin, lmax = (int(x) for x in g[f"{tag}_lrange"])
        wr2 = g[f"{tag}_w_trap"] * g[f"{tag}_r"] ** 2
        return (g[f"{tag}_q"], g[f"{tag}_qt"], g[f"{tag}_C"], g[f"{tag}_v"], wr2,
                g[f"{tag}_entries"], lmin, lmax)

    @pytest.mark.parametrize("tag", ["desk", "small12"])
    def test_matches_reference(self, g_desk, tag):
        q, qt, C, v, wr2, e, lmin, lmax = self.desk(g_desk, tag)
        got = ref.gamma3d(q, qt, C, v, wr2, e, lmin, lmax)
        assert np.array_equal(got, g_desk[f"{tag}_gamma"])    # same code path, same order

    def test_ordered_vs_unordered(self, g_desk):               # test_engine3d.py:96-106
        q, qt, C, v, wr2, e, lmin, lmax = self.desk(g_desk, "small12")
        got = ref.gamma3d(q, qt, C, v, wr2, e, lmin, lmax)
        assert gap_rel(got, g_desk["small12_unordered"]) < 1e-12

    def test_workers_and_block_invariance(self, g_desk):       # test_engine3d.py:52-62
        q, qt, C, v, wr2, e, lmin, lmax = self.desk(g_desk, "desk")
        for w, b in ((1, 1), (2, 7), (3, 64)):
            got = ref.gamma3d(q, qt, C, v, wr2, e, lmin, lmax, workers=w, block=b)
            assert gap_rel(got, g_desk["desk_naive"]) < 1e-12

    def test_c0_partials(self, g_c0):
        hi = host_inputs("c0")
        got = ref.gamma3d(hi.q, g_c0["qt"], g_c0["C"], hi.v, hi.wr2, hi.entries, 2, 200,
                          1000, 20000)
        assert np.array_equal(got, g_c0["partial_1000_20000"])

    def test_naive_entry(self, g_desk):
        q, qt, C, v, wr2, e, lmin, lmax = self.desk(g_desk, "desk")
        l1, l2, l3 = ref.domain_triples(lmin, lmax)
        n, m = 3, 5
        want = 0.0
        for a, b, c in zip(l1, l2, l3):
            z = ref.triple_zm(lmin, [a], [b], [c], C, v)[0]
            want += z * ref.late_product_y(a, b, c, m, q, e, lmin) \
                * ref.radial_integral_x(a, b, c, n, qt, e, wr2, lmin)
        assert want == pytest.approx(g_desk["desk_naive"][m, n], rel=1e-12)


class TestInputs:
    def test_c0_inputs_pinned(self, g_c0):
        hi = host_inputs("c0")
        assert hi.eps.sum() == g_c0["eps_sum"]
        assert np.array_equal(hi.wr2, g_c0["wr2_ref"])        # reference integration_weights

    @pytest.mark.parametrize("integ", ["trap", "hermite", "spline"])
    def test_x_weights_vs_reference(self, g_desk, integ):
        for tag in ("desk", "desk32"):
            r = g_desk[f"{tag}_r"]
            want = g_desk[f"{tag}_w_{integ}"] * r ** 2
            got = x_weights(r, integ)
            if integ == "trap":
                assert np.array_equal(got, want)
            else:
                assert np.max(np.abs(got - want)) <= 1e-12 * np.max(np.abs(want))

    def test_stage1_oracle_c0(self, g_c0):
        """scipy restatement of stage 1 reproduces the committed c0 inputs."""
        from oracle import qtilde_ref
        hi = host_inputs("c0")
        d = qtilde_ref.delta_table(hi.k, hi.eps, 2, 200)
        assert np.array_equal(d[[0, 50, 198]], g_c0["delta_rows"])
        C = qtilde_ref.c_ell(d, hi.k, hi.wk)
        assert np.array_equal(C, g_c0["C"])
        qt = qtilde_ref.qtilde(hi.k, hi.wk, hi.x, hi.qk, d, 2, 200, ells=[2, 77, 200])
        for l in (2, 77, 200):
            assert np.array_equal(qt[:, :, l - 2], g_c0["qt"][:, :, l - 2])


class TestNonsepPin:
    """The config-3 restatement (oracle/nonsep_ref.py) against the unmodified reference's own
    per-triple functions — radial_integral_x, late_product_y, _triple_z,
    permutation_multiplicity in gamma3d_naive's loop structure (engine3d.py:41-83,189-215) —
    on 240 seeded config-3 triples incl. odd-parity and step-10 cells, both h2 modes
    (tests/golden/make_c3_golden.py)."""

    @pytest.mark.parametrize("mode", ["gosper", "exact"])
    def test_sample_matches_reference_functions(self, mode):
        from conftest import golden
        from oracle import nonsep_ref
        from paper_1503_08809_b200.configs import sparse_domain, sparse_grid
        g = golden("c3.npz")
        hi = host_inputs("c3")
        l1, l2, l3, W = sparse_domain(*sparse_grid(l_max=hi.l_max))
        assert l1.size == int(g["count"]) == 724930
        qt = np.zeros((hi.spec.p, hi.x.size, hi.l_max - 1))
        qt[:, :, g["grid"] - 2] = g["qt_grid"]
        i = g["sample_idx"]
        assert ((l1[i] + l2[i] + l3[i]) % 2 == 1).any() and (W[i] != 1.0).any()
        b = nonsep_ref.nonsep(hi.q, qt, g["C"], hi.v, hi.wr2, hi.entries, hi.alpha, 2, l1[i],
                              l2[i], l3[i], W[i], h2_mode=mode)
        assert frob_rel(b, g[f"sample_b_{mode}"]) < 1e-13

    def test_exact_mode_gates_odd_parity(self):
        """h2_exact is exactly 0 off the triangle / even-parity set (geometry.py:67-71)."""
        l1 = np.array([2, 3, 2, 10])
        l2 = np.array([2, 3, 3, 10])
        l3 = np.array([2, 3, 4, 25])          # even ok, odd sum, odd sum, no triangle
        h = ref.h2_exact(l1, l2, l3)
        assert h[0] > 0 and h[1] == 0 and h[2] == 0 and h[3] == 0


class TestGamma2DPin:
    """oracle/gamma2d_ref.py against the reference's own P tables and Γ2d matrices
    (tests/golden/io2d.npz, written by cmbproj.build_ptable / gamma2d_matrix)."""

    @pytest.mark.parametrize("tag", ["desk", "desk32"])
    def test_ptable_and_gamma2d(self, g_desk, tag):
        from conftest import golden
        from oracle import gamma2d_ref
        from paper_1503_08809_b200.quadrature import gauss_legendre, legendre_table
        g2 = golden("io2d.npz")
        lmin, lmax = (int(x) for x in g_desk[f"{tag}_lrange"])
        rule = gauss_legendre(g2[f"{tag}_mu_nodes"].size)
        assert np.array_equal(rule.weights, g2[f"{tag}_mu_weights"])
        leg = legendre_table(lmax, rule)
        P = gamma2d_ref.ptable(g_desk[f"{tag}_q"], g_desk[f"{tag}_qt"], g_desk[f"{tag}_C"],
                               g_desk[f"{tag}_v"], lmin, lmax, leg)
        assert np.array_equal(P, g2[f"{tag}_ptable"])
        wr2 = x_weights(g_desk[f"{tag}_r"], "trap")
        got = gamma2d_ref.gamma2d(P, g_desk[f"{tag}_entries"], rule.weights, wr2)
        assert gap_rel(got, g2[f"{tag}_gamma2d"]) < 1e-13
