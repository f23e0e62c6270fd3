"""CPU: host logic of the drop-in (mirror types, plans, shard balance, configs) and the
C-ABI library (loads, exports every symbol of include/modal_b200.h, fails loudly without a
GPU).  No compute call needs a device here."""

import ctypes
import os
import re

import numpy as np
import pytest

import paper_1503_08809_b200 as mg
from conftest import ROOT
from paper_1503_08809_b200 import _native
from paper_1503_08809_b200.configs import CONFIGS, host_inputs, sparse_domain, sparse_grid
from paper_1503_08809_b200.scheduler import slab_costs


def header_symbols():
    text = open(os.path.join(ROOT, "include", "modal_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|const char\*)\s+(mg_\w+)\(", text, re.M)))


class TestABI:
    def test_library_exports_every_header_symbol(self):
        lib = _native.lib()
        syms = header_symbols()
        assert len(syms) >= 20
        for s in syms:
            assert hasattr(lib, s), s
            assert s in _native._SIGS, f"{s} missing from the ctypes binding"

    def test_library_is_sm100a(self):
        import subprocess
        out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH],
                             capture_output=True, text=True).stdout
        assert "sm_100a" in out

    def test_host_only_entry_points(self):
        lib = _native.lib()
        assert lib.mg_version() >= 100
        c, r = np.zeros(1, np.int64), np.zeros(1, np.int64)
        assert lib.mg_domain_count(2, 2000, _native.ptr(c), _native.ptr(r)) == 0
        assert c[0] == 334_831_501
        assert lib.mg_domain_count(1, 4, _native.ptr(c), None) == 1     # ValueError code
        assert b"l_min" in lib.mg_last_error()

    def test_no_gpu_fails_loudly(self):
        if _native.lib().mg_device_count() > 0:
            pytest.skip("a GPU is present")
        with pytest.raises(RuntimeError, match="no CUDA device"):
            mg.triple_weights(np.ones(3), np.ones(3), 2, 4)

    @pytest.mark.parametrize("lmin,lmax", [(2, 40), (3, 25), (2, 200), (4, 4), (2, 2)])
    def test_range_detection(self, lmin, lmax):
        """mg_domain_match_range (host walk of the enumeration): contiguous flat ranges are
        recognised with their start, anything with a hole or out of order is not."""
        from oracle import ref
        from paper_1503_08809_b200.engine3d import _detect_contiguous
        T = ref.domain_count(lmin, lmax)
        for a, b in {(0, T), (0, 1), (min(5, T - 1), T), (T - 1, T),
                     (min(17, T - 1), min(123, T)), (T // 2, min(T // 2 + 1000, T))}:
            l1, l2, l3 = (x.astype(np.int32) for x in ref.domain_triples(lmin, lmax, a, b))
            assert _detect_contiguous(l1, l2, l3, lmin, lmax) == (a, b)
            if b - a > 2:
                k = np.ones(b - a, bool)
                k[(b - a) // 2] = False
                assert _detect_contiguous(l1[k], l2[k], l3[k], lmin, lmax) is None
                r = [np.ascontiguousarray(x[::-1]) for x in (l1, l2, l3)]
                assert _detect_contiguous(*r, lmin, lmax) is None
        bad = np.array([lmax + 1], np.int32)
        assert _detect_contiguous(bad, bad, bad, lmin, lmax) is None

    def test_slab_plan_matches_python(self):
        b = np.zeros(9, np.int32)
        for spec in CONFIGS.values():
            _native.check(_native.lib().mg_slab_plan(2, spec.l_max, spec.p, spec.n_x, 8,
                                                     _native.ptr(b)))
            assert b.tolist() == mg.slab_plan(2, spec.l_max, spec.p, spec.n_x, 8)


class TestMirrorTypes:
    def test_default_mapping(self):
        m = mg.default_mode_mapping(3)
        assert m.n_max == 10
        assert m.triple(0) == (0, 0, 0) and m.triple(9) == (2, 2, 2)
        assert mg.default_mode_mapping(30).n_max == 4960

    def test_mapping_validation(self):
        with pytest.raises(ValueError):
            mg.ModeMapping(np.array([[1, 0, 0]]), 2)
        with pytest.raises(ValueError):
            mg.ModeMapping(np.array([[0, 0, 1], [0, 0, 1]]), 2)
        with pytest.raises(ValueError):
            mg.ModeMapping(np.zeros((0, 3)), 2)

    def test_tables_validation(self):
        q = np.ones((2, 3))
        qt = np.ones((2, 4, 3))
        with pytest.raises(ValueError):
            mg.BasisTables(q, qt, np.array([1.0, 0.0, 1.0]), np.ones(3), 2, 4)
        with pytest.raises(ValueError):
            mg.BasisTables(q, qt, np.ones(4), np.ones(3), 2, 4)
        t = mg.BasisTables(q, qt, np.ones(3), np.ones(3), 2, 4)
        assert t.p_max == 2 and t.n_radial == 4

    def test_fingerprints_match_reference_scheme(self, g_desk):
        # same sha256 recipe as basis.py:50-54,93-94,189-190,259-262
        import hashlib
        e = g_desk["desk_entries"]
        m = mg.ModeMapping(e, 3)
        h = hashlib.sha256(np.int64(3).tobytes() + e.astype(np.int64).tobytes()).hexdigest()[:16]
        assert m.fingerprint() == h

    def test_gamma_container(self):
        with pytest.raises(ValueError):
            mg.GammaMatrix(np.array([[np.nan]]))
        with pytest.raises(ValueError):
            mg.GammaMatrix(np.zeros(3))

    def test_shifted_legendre_bit_exact(self, g_desk):
        assert np.array_equal(mg.shifted_legendre(3, 2, 16), g_desk["desk_q"])


class TestScheduler:
    def test_make_plan_golden(self, g_domain):                # test_scheduler.py:10-17
        assert np.array_equal(np.array(mg.make_plan(12, 4).ranges), g_domain["plan_12_4"])
        assert np.array_equal(np.array(mg.make_plan(10, 4).ranges), g_domain["plan_10_4"])

    @pytest.mark.parametrize("total,w", [(0, 3), (7, 1), (2, 5), (10**6, 256)])
    def test_make_plan_cover(self, total, w):
        r = mg.make_plan(total, w).ranges
        assert r[0][0] == 0 and r[-1][1] == total
        sizes = [b - a for a, b in r]
        assert max(sizes) - min(sizes) <= 1 and sizes == sorted(sizes, reverse=True)

    def test_merge_partials_order(self):
        meta = {"tables": "t", "grid": "g", "mapping": "m"}
        parts = [mg.GammaMatrix(np.array([[v]]), dict(meta)) for v in (1.0, 10.0, 100.0)]
        out = mg.merge_partials(parts)
        assert out.values[0, 0] == 111.0 and out.meta["workers_merged"] == 3
        bad = mg.GammaMatrix(np.array([[1.0]]), dict(meta, tables="x"))
        with pytest.raises(ValueError):
            mg.merge_partials([parts[0], bad])

    @pytest.mark.parametrize("cfg", ["c1", "c2", "c4"])
    def test_slab_balance(self, cfg):
        spec = CONFIGS[cfg]
        cost = slab_costs(2, spec.l_max, spec.p, spec.n_x)
        for n in (2, 4, 8):
            b = mg.slab_plan(2, spec.l_max, spec.p, spec.n_x, n)
            assert b[0] == 2 and b[-1] == spec.l_max + 1 and b == sorted(b)
            shares = [cost[b[i] - 2:b[i + 1] - 2].sum() for i in range(n)]
            assert max(shares) / (sum(shares) / n) < 1.01


class TestConfigs:
    def test_shapes(self):
        hi = host_inputs("c1")
        assert hi.eps.shape == (1999, 3000) and hi.q.shape == (15, 1999)
        assert hi.qk.shape == (15, 3000) and hi.entries.shape == (680, 3)

    def test_alpha_drawn_after_eps(self):
        hi = host_inputs("c3")
        rng = np.random.default_rng(3)
        rng.standard_normal((1999, 2000))
        e = mg.default_mode_mapping(8).entries
        assert np.array_equal(hi.alpha, rng.standard_normal(120) / (1.0 + e.sum(1)))

    def test_sparse_grid(self):
        g, w = sparse_grid()
        assert g.size == 244 and g[48] == 50 and g[49] == 60 and g[-1] == 2000
        assert w[0] == 1.0 and w[48] == 5.5 and w[49] == 10.0 and w[-1] == 5.5
        # step-1 grid: unit weights and exactly the reference domain
        g1, w1 = sparse_grid(l_max=30, dense_to=30)
        assert np.all(w1 == 1.0)
        l1, l2, l3, W = sparse_domain(g1, w1)
        from oracle import ref
        want = ref.domain_triples(2, 30)
        assert np.array_equal(l1, want[0]) and np.array_equal(l2, want[1])
        assert np.array_equal(l3, want[2]) and np.all(W == 1.0)


def test_device_selection(monkeypatch):
    """Device list of the one-shot call: devices > device > MG_DEVICES > LOCAL_RANK under
    torchrun > every visible device."""
    from paper_1503_08809_b200 import resolve_devices
    monkeypatch.delenv("MG_DEVICES", raising=False)
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    assert resolve_devices(None, [1, 0]) == [1, 0]
    assert resolve_devices(3, None) == [3]
    monkeypatch.setenv("MG_DEVICES", "0,0")
    assert resolve_devices() == [0, 0]
    monkeypatch.delenv("MG_DEVICES")
    monkeypatch.setenv("WORLD_SIZE", "8")
    monkeypatch.setenv("LOCAL_RANK", "5")
    assert resolve_devices() == [5]
    monkeypatch.delenv("WORLD_SIZE")
    assert resolve_devices() == [0]                          # no GPU here: one (failing) device
    with pytest.raises(ValueError):
        resolve_devices(None, [])


def test_integration_shim_rebinds_reference_names():
    """paper_1503_08809_b200.integration.install rebinds exactly the reference's engine
    names (cmbproj, engine3d, harness; harness.py:19-21) and uninstall restores them."""
    import sys
    for path in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(path, "cmbproj")):
            if path not in sys.path:
                sys.path.append(path)
            break
    cp = pytest.importorskip("cmbproj")
    from paper_1503_08809_b200 import integration
    before = (cp.gamma3d_matrix, cp.engine3d.gamma3d_matrix, cp.harness.gamma3d_matrix,
              cp.gamma2d_matrix, cp.engine2d.gamma2d_matrix, cp.harness.gamma2d_matrix)
    saved = integration.install(cp)
    try:
        for fn in (cp.gamma3d_matrix, cp.engine3d.gamma3d_matrix, cp.harness.gamma3d_matrix,
                   cp.gamma2d_matrix, cp.engine2d.gamma2d_matrix, cp.harness.gamma2d_matrix):
            assert getattr(fn, "__wrapped_b200__", False)
        assert cp.gamma3d_naive is not None and not hasattr(cp.gamma3d_naive, "__wrapped_b200__")
        import inspect
        ref_sig = inspect.signature(before[1])
        assert list(inspect.signature(cp.gamma3d_matrix).parameters) == list(ref_sig.parameters)
        assert list(inspect.signature(cp.gamma2d_matrix).parameters) == \
            list(inspect.signature(before[4]).parameters)
    finally:
        integration.uninstall(saved)
    after = (cp.gamma3d_matrix, cp.engine3d.gamma3d_matrix, cp.harness.gamma3d_matrix,
             cp.gamma2d_matrix, cp.engine2d.gamma2d_matrix, cp.harness.gamma2d_matrix)
    assert all(a is b for a, b in zip(before, after))


def test_shape_checks_before_the_c_call():
    """The C-ABI reads raw pointers, so the drop-ins reject inconsistent shapes up front
    (a radial grid whose length differs from q̃'s n_radial would otherwise be read out of
    bounds): ValueError like the reference's einsum / BasisTables validation."""
    from paper_1503_08809_b200 import BasisTables, GammaPlan, ModeMapping, RadialGrid
    from paper_1503_08809_b200.quadrature import x_weights
    L, p, nx = 15, 3, 20
    rng = np.random.default_rng(0)
    t = BasisTables(rng.standard_normal((p, L)), rng.standard_normal((p, nx, L)),
                    rng.uniform(1, 2, L), np.ones(L), 2, 16)
    m = mg.default_mode_mapping(p)
    short = RadialGrid(np.linspace(1.0, 2.0, nx - 3))
    with pytest.raises(ValueError, match="n_radial"):
        mg.gamma3d_matrix(t, m, short, devices=[0])
    with pytest.raises(ValueError, match="n_radial"):
        mg.gamma_nonsep(t, m, short, np.ones(m.n_max),
                        mg.SparseDomain([2], [2], [2], [1.0]))
    with pytest.raises(ValueError):
        GammaPlan(t.q, t.q_tilde, t.C, t.v, x_weights(short.r), m.entries, 2, 16)
