"""The reference's own hot-path tests, run through the drop-in.

The unmodified reference package `cmbproj` is imported (from `baseline/_ref`, where
`pip install --no-index --no-deps --target baseline/_ref` put it — it travels to the GPU
box with the repo — or from /root/reference/pkg/src in the build container; skipped when
neither exists), its engine names are rebound to the GPU drop-ins exactly as a maintainer
would (paper_1503_08809_b200.integration; the same mechanism as
test_harness.py:274-281), and the checks of
  pkg/tests/test_engine3d.py:47-106   TestBlockedVsNaive / TestOrderedEnumeration
  pkg/tests/test_acceptance.py:50-57   criterion 1 (2D == 3D exact)
  pkg/tests/test_acceptance.py:86-120  criteria 3 and 4 (optimized == naive, ordered domain)
  pkg/tests/test_acceptance.py:168-185 criterion 7 (determinism)
are re-run with reference-constructed objects against the reference's own naive oracles
(gamma3d_naive, gamma3d_unordered_reference, gamma2d_matrix_naive — not rebound), with the
reference's tolerances.  harness.run_gamma / run_crosscheck go through the rebinding too.
"""

import os
import sys

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _import_cmbproj():
    for path in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(path, "cmbproj")):
            if path not in sys.path:
                sys.path.append(path)
            try:
                import cmbproj
                return cmbproj
            except Exception:
                return None
    return None


cp = _import_cmbproj()
if cp is None:
    pytest.skip("reference package cmbproj not importable (no baseline/_ref)",
                allow_module_level=True)

from paper_1503_08809_b200 import integration  # noqa: E402


def relative_gap(a, b):                                    # test_engine3d.py:7-9
    scale = max(np.max(np.abs(a)), np.max(np.abs(b)))
    return np.max(np.abs(a - b)) / scale


class Problem:                                             # pkg/tests/conftest.py:8-19
    def __init__(self, l_min, l_max, p_max, n_r, n_mu=None):
        from cmbproj.engine2d import default_mu_points
        self.grid = cp.default_radial_grid(n_r)
        self.tables = cp.synthesize_basis(p_max, l_min, l_max, self.grid)
        self.mapping = cp.default_mode_mapping(p_max)
        self.rule = cp.gauss_legendre(n_mu or default_mu_points(l_max))
        self.legendre = cp.legendre_table(l_max, self.rule)


@pytest.fixture(scope="module")
def desk():
    return Problem(2, 16, 3, 54)


@pytest.fixture(scope="module")
def accept():
    return Problem(2, 32, 4, 216, 50)


@pytest.fixture(scope="module")
def naive(desk):
    return cp.gamma3d_naive(desk.tables, desk.mapping, desk.grid)


@pytest.fixture(scope="module")
def accept_naive3d(accept):
    return cp.gamma3d_naive(accept.tables, accept.mapping, accept.grid)


@pytest.fixture(autouse=True)
def rebound(monkeypatch):
    """Every test runs with the reference's engine names bound to the GPU drop-ins."""
    integration.install(cp, setattr_fn=monkeypatch.setattr)
    assert getattr(cp.gamma3d_matrix, "__wrapped_b200__", False)
    assert getattr(cp.harness.gamma3d_matrix, "__wrapped_b200__", False)
    yield


class TestBlockedVsNaive:                                  # test_engine3d.py:47-94
    def test_default_block(self, desk, naive):
        g = cp.gamma3d_matrix(desk.tables, desk.mapping, desk.grid)
        assert isinstance(g, cp.GammaMatrix)
        assert relative_gap(g.values, naive.values) < 1e-12

    @pytest.mark.parametrize("block", [1, 7, 64, 256])
    def test_block_size_invariance(self, desk, naive, block):
        g = cp.gamma3d_matrix(desk.tables, desk.mapping, desk.grid, block=block)
        assert relative_gap(g.values, naive.values) < 1e-12

    @pytest.mark.parametrize("workers", [1, 2, 4, 8])
    def test_worker_count_invariance(self, desk, naive, workers):
        g = cp.gamma3d_matrix(desk.tables, desk.mapping, desk.grid, workers=workers)
        assert relative_gap(g.values, naive.values) < 1e-12

    def test_fixed_config_is_bitwise_reproducible(self, desk):
        a = cp.gamma3d_matrix(desk.tables, desk.mapping, desk.grid, workers=3, block=16)
        b = cp.gamma3d_matrix(desk.tables, desk.mapping, desk.grid, workers=3, block=16)
        assert np.array_equal(a.values, b.values)

    @pytest.mark.parametrize("integrator", ["hermite", "spline"])
    def test_other_integrators(self, desk, integrator):
        g = cp.gamma3d_matrix(desk.tables, desk.mapping, desk.grid, integrator=integrator)
        n = cp.gamma3d_naive(desk.tables, desk.mapping, desk.grid, integrator=integrator)
        assert relative_gap(g.values, n.values) < 1e-12

    def test_exact_mode(self, desk):
        g = cp.gamma3d_matrix(desk.tables, desk.mapping, desk.grid, h2_mode="exact")
        n = cp.gamma3d_naive(desk.tables, desk.mapping, desk.grid, h2_mode="exact")
        assert relative_gap(g.values, n.values) < 1e-12

    def test_unknown_h2_mode(self, desk):
        with pytest.raises(ValueError):
            cp.gamma3d_matrix(desk.tables, desk.mapping, desk.grid, h2_mode="asymptotic")

    def test_rejects_bad_block(self, desk):
        with pytest.raises(ValueError):
            cp.gamma3d_matrix(desk.tables, desk.mapping, desk.grid, block=0)

    def test_reference_domain_slice(self, desk, naive):
        """A reference TriangularDomain (whole, and a _sweep_chunk-style slice) as `domain`."""
        dom = cp.enumerate_domain(2, 16)
        g = cp.gamma3d_matrix(desk.tables, desk.mapping, desk.grid, domain=dom)
        assert relative_gap(g.values, naive.values) < 1e-12


class TestOrderedEnumeration:                              # test_engine3d.py:97-106
    def test_matches_unordered_reference(self):
        grid = cp.default_radial_grid(30)
        tables = cp.synthesize_basis(3, 2, 12, grid)
        mapping = cp.default_mode_mapping(3)
        ordered = cp.gamma3d_matrix(tables, mapping, grid)
        unordered = cp.gamma3d_unordered_reference(tables, mapping, grid)
        assert relative_gap(ordered.values, unordered.values) < 1e-12


class TestEngine2D:                                        # test_engine2d.py:50-135
    """The reference's μ-engine tests with build_ptable / gamma2d_matrix rebound to the GPU;
    gamma2d_entry, gamma2d_entry_naive and gamma2d_matrix_naive stay the reference's own."""

    def test_ptable_shape_and_direct_sum(self, desk):                     # :51-65
        from cmbproj.engine2d import PTable, _l_weight
        assert getattr(cp.build_ptable, "__wrapped_b200__", False)
        pt = cp.build_ptable(desk.tables, desk.grid, desk.rule, desk.legendre)
        assert isinstance(pt, PTable)
        assert pt.values.shape == (3, 3, len(desk.grid), desk.rule.n)
        t = desk.tables
        lw = _l_weight(t)
        pl = desk.legendre[t.l_min:t.l_max + 1]
        for a, b, x, m in [(0, 0, 0, 0), (1, 2, 10, 5), (2, 1, 53, 26)]:
            direct = float(np.sum(lw * t.q[a] * t.q_tilde[b, x] * pl[:, m]))
            assert pt.values[a, b, x, m] == pytest.approx(direct, rel=1e-12)

    def test_ptable_budget_and_determinism(self, desk):                   # :67-75
        with pytest.raises(MemoryError):
            cp.build_ptable(desk.tables, desk.grid, desk.rule, desk.legendre, budget_bytes=1024)
        a = cp.build_ptable(desk.tables, desk.grid, desk.rule, desk.legendre)
        b = cp.build_ptable(desk.tables, desk.grid, desk.rule, desk.legendre)
        assert np.array_equal(a.values, b.values)

    @pytest.mark.parametrize("integrator", ["trap", "hermite", "spline"])
    def test_reference_entries_from_gpu_table(self, desk, integrator):     # :79-97
        pt = cp.build_ptable(desk.tables, desk.grid, desk.rule, desk.legendre)
        for n, n_prime in [(0, 0), (0, 5), (3, 7), (9, 2)]:
            fast = cp.gamma2d_entry(n, n_prime, pt, desk.mapping, desk.grid, desk.rule,
                                    integrator=integrator)
            naive = cp.gamma2d_entry_naive(n, n_prime, desk.tables, desk.mapping, desk.grid,
                                           desk.rule, desk.legendre, integrator=integrator)
            assert fast == pytest.approx(naive, rel=1e-12)

    def test_matrix_vs_naive_matrix(self, desk):                          # :110-116
        fast = cp.gamma2d_matrix(desk.tables, desk.mapping, desk.grid, desk.rule, desk.legendre)
        naive = cp.gamma2d_matrix_naive(desk.tables, desk.mapping, desk.grid, desk.rule,
                                        desk.legendre)
        assert relative_gap(fast.values, naive.values) < 1e-12
        assert np.isfinite(fast.values).all() and np.any(fast.values != 0.0)

    @pytest.mark.parametrize("workers", [2, 3, 5])
    def test_bitwise_identical_across_workers(self, desk, workers):       # :118-123
        base = cp.gamma2d_matrix(desk.tables, desk.mapping, desk.grid, desk.rule, desk.legendre,
                                 workers=1)
        multi = cp.gamma2d_matrix(desk.tables, desk.mapping, desk.grid, desk.rule,
                                  desk.legendre, workers=workers)
        assert np.array_equal(base.values, multi.values)

    def test_meta_and_reference_ptable_argument(self, desk):              # :125-131
        g = cp.gamma2d_matrix(desk.tables, desk.mapping, desk.grid, desk.rule, desk.legendre,
                              workers=2)
        assert g.meta["engine"] == "modal2d" and g.meta["workers"] == 2
        assert g.meta["n_mu"] == desk.rule.n
        assert g.meta["tables"] == desk.tables.fingerprint()
        pt = cp.build_ptable(desk.tables, desk.grid, desk.rule, desk.legendre)
        again = cp.gamma2d_matrix(desk.tables, desk.mapping, desk.grid, desk.rule,
                                  desk.legendre, ptable=pt)
        assert np.array_equal(again.values, g.values)


class TestAcceptance:
    def test_criterion_1_separable_direct_equivalence(self, accept):   # :50-57
        g2 = cp.gamma2d_matrix(accept.tables, accept.mapping, accept.grid, accept.rule,
                               accept.legendre, integrator="trap")
        g3 = cp.gamma3d_matrix(accept.tables, accept.mapping, accept.grid, h2_mode="exact",
                               integrator="trap")
        assert cp.max_rel_deviation(g2, g3) <= 1e-10

    def test_criterion_3_optimized_vs_naive(self, accept, accept_naive3d):   # :86-106
        g2_fast = cp.gamma2d_matrix(accept.tables, accept.mapping, accept.grid, accept.rule,
                                    accept.legendre)
        g2_naive = cp.gamma2d_matrix_naive(accept.tables, accept.mapping, accept.grid,
                                           accept.rule, accept.legendre)
        dev2 = cp.max_rel_deviation(g2_fast, g2_naive)
        dev3 = 0.0
        for block in (1, 7, 64, 256):
            g = cp.gamma3d_matrix(accept.tables, accept.mapping, accept.grid, block=block)
            dev3 = max(dev3, cp.max_rel_deviation(g, accept_naive3d))
        for workers in (1, 2, 4, 8):
            g = cp.gamma3d_matrix(accept.tables, accept.mapping, accept.grid, workers=workers)
            dev3 = max(dev3, cp.max_rel_deviation(g, accept_naive3d))
        assert dev2 <= 1e-12 and dev3 <= 1e-12

    def test_criterion_4_ordered_domain_validity(self):                   # :109-120
        """Criterion 4 with the drop-in as the ordered engine (the reference's criterion
        compares its own naive ordered sum with the unordered sum)."""
        grid = cp.default_radial_grid(54)
        tables = cp.synthesize_basis(4, 2, 12, grid)
        mapping = cp.default_mode_mapping(4)
        ordered = cp.gamma3d_matrix(tables, mapping, grid)
        unordered = cp.gamma3d_unordered_reference(tables, mapping, grid)
        assert cp.max_rel_deviation(ordered, unordered) <= 1e-12

    def test_criterion_7_determinism(self, accept):                       # :168-185
        runs2d = [cp.gamma2d_matrix(accept.tables, accept.mapping, accept.grid, accept.rule,
                                    accept.legendre, workers=w) for w in (1, 2, 4)]
        assert all(np.array_equal(runs2d[0].values, g.values) for g in runs2d[1:])
        a = cp.gamma3d_matrix(accept.tables, accept.mapping, accept.grid, workers=3, block=32)
        b = cp.gamma3d_matrix(accept.tables, accept.mapping, accept.grid, workers=3, block=32)
        assert np.array_equal(a.values, b.values)
        dev_w = max(cp.max_rel_deviation(
            cp.gamma3d_matrix(accept.tables, accept.mapping, accept.grid, workers=w), a)
            for w in (1, 2, 4))
        assert dev_w <= 1e-12


class TestHarness:
    """The reference's drivers reach the drop-in through the rebound module names."""

    def test_run_gamma_3d(self, monkeypatch):
        cfg = cp.harness.RunConfig(mode="gamma3d", l_max=20, p_max=3, r_samples=60)
        got = cp.harness.run_gamma(cfg)
        assert got.meta.get("devices") is not None                # came from the GPU path
        monkeypatch.undo()                                        # original engines back
        want = cp.harness.run_gamma(cfg)
        assert "devices" not in want.meta
        assert relative_gap(got.values, want.values) < 1e-12
        assert got.same_inputs(want)

    def test_run_crosscheck(self):
        """2D engine vs 3D exact engine (both rebound): the reference's crosscheck report."""
        rep = cp.harness.run_crosscheck(cp.harness.RunConfig(l_max=24, p_max=3,
                                                             r_samples=60))
        assert rep.max_rel_dev <= 1e-10

    def test_run_convergence_study(self, monkeypatch):
        """harness.run_convergence_study (harness.py:312-340): every integrator on a ladder of
        radial grids against the dense-spline gold standard, all through the rebound engine;
        the percentage RMSEs must equal the reference's own."""
        cfg = cp.harness.RunConfig(l_max=14, p_max=3, r_samples=54)
        got = cp.harness.run_convergence_study(cfg, ladder=(54, 108))
        monkeypatch.undo()
        want = cp.harness.run_convergence_study(cfg, ladder=(54, 108))
        assert [(r["integrator"], r["r_samples"]) for r in got] == \
               [(r["integrator"], r["r_samples"]) for r in want]
        for a, b in zip(got, want):
            assert abs(a["rmse_percent"] - b["rmse_percent"]) <= 1e-8 * max(1.0, b["rmse_percent"])

    def test_run_bench(self):
        """harness.run_bench (harness.py:353-410) drives the 2D engine and the direct engine
        with an explicit enumerate_domain() object and a worker count through the rebinding."""
        rows = cp.harness.run_bench(cp.harness.RunConfig(l_max=16, p_max=3, r_samples=54,
                                                         workers=2, bench_repeats=1))
        assert [r["path"] for r in rows] == ["2d-optimized", "2d-naive", "2d-speedup", "3d-w1",
                                             "3d-w2"]
        assert all(r["seconds"] == "" or r["seconds"] > 0 for r in rows)

    def test_cli_end_to_end(self, tmp_path, monkeypatch, capsys):
        """The reference's command line (cli.py:105-148) reaches the GPU through the same
        rebinding: `--mode gamma3d --out ...` writes the matrix the reference itself writes."""
        import cmbproj.cli as cli
        args = ["--mode", "gamma3d", "--lmax", "18", "--pmax", "3", "--r-samples", "54",
                "--format", "bin"]
        assert cli.main(args + ["--out", str(tmp_path / "gpu.bin")]) == 0
        monkeypatch.undo()
        assert cli.main(args + ["--out", str(tmp_path / "cpu.bin")]) == 0
        a = cp.harness.deserialize_gamma(tmp_path / "gpu.bin", "bin")
        b = cp.harness.deserialize_gamma(tmp_path / "cpu.bin", "bin")
        assert relative_gap(a.values, b.values) < 1e-12
        assert "wrote 10x10 matrix" in capsys.readouterr().out

    def test_serialize_roundtrip(self, tmp_path, desk):
        g = cp.gamma3d_matrix(desk.tables, desk.mapping, desk.grid)
        for fmt in ("csv", "bin"):
            path = tmp_path / f"g.{fmt}"
            cp.harness.serialize_gamma(g, path, fmt)
            back = cp.harness.deserialize_gamma(path, fmt)
            assert np.array_equal(back.values, g.values)
