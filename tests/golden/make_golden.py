"""Generate the golden vectors that pin the CPU oracle (and, through it, the CUDA path).

Runs ONLY in the build container, where the reference package is importable read-only from
/root/reference/pkg/src.  The GPU box never reads /root/reference: the tests there use the
committed .npz files written by this script.

    python -B tests/golden/make_golden.py

Every array below is produced by calling the UNMODIFIED reference (`cmbproj`) through its
public API (or, for flat-range partials, its `_sweep_chunk` worker, engine3d.py:123-136) —
except the config-0 q̃/C inputs, which come from the stage-1 oracle (oracle/qtilde_ref.py,
scipy), because the reference has no stage 1.
"""

from __future__ import annotations

import os
import sys

sys.dont_write_bytecode = True
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import cmbproj as cp  # noqa: E402
from cmbproj import engine3d as e3  # noqa: E402


class _Slice:
    """Duck-typed domain slice accepted by _sweep_chunk (engine3d.py:130-132)."""

    def __init__(self, l1, l2, l3):
        self.l1, self.l2, self.l3 = l1, l2, l3
        self.count = len(l1)


def domain_golden():
    out = {}
    lmaxes = np.array([2, 3, 4, 5, 8, 13, 21, 40, 64, 100, 200])
    out["count_lmax"] = lmaxes
    out["count"] = np.array([cp.enumerate_domain(2, int(m)).count for m in lmaxes])
    d = cp.enumerate_domain(2, 4)
    out["triples_2_4"] = np.stack([d.l1, d.l2, d.l3], 1)
    d = cp.enumerate_domain(3, 40)
    out["l1_3_40"], out["l2_3_40"], out["l3_3_40"] = d.l1, d.l2, d.l3
    # bit-exact weights at l_max=64 (test_geometry.py:161-173 draws C, v the same way)
    rng = np.random.default_rng(7)
    C = rng.uniform(0.5, 2.0, 63)
    v = rng.uniform(0.5, 2.0, 63)
    d = cp.enumerate_domain(2, 64)
    zm = e3._triple_z(_Tab(C, v, 2), d.l1, d.l2, d.l3, "gosper") \
        * cp.permutation_multiplicity(d.l1, d.l2, d.l3)
    out["zm64_C"], out["zm64_v"], out["zm64"] = C, v, zm
    out["zm64_exact"] = e3._triple_z(_Tab(C, v, 2), d.l1, d.l2, d.l3, "exact") \
        * cp.permutation_multiplicity(d.l1, d.l2, d.l3)
    out["h2g_222"] = np.array(cp.h2_gosper(2, 2, 2))
    out["h2e_222"] = np.array(cp.h2_exact(2, 2, 2))
    ones = np.ones(1)
    out["z222_unit"] = np.array(cp.geometric_prefactor(2, 2, 2, ones, ones, l_min=2))
    out["plan_12_4"] = np.array(cp.make_plan(12, 4).ranges)
    out["plan_10_4"] = np.array(cp.make_plan(10, 4).ranges)
    return out


class _Tab:
    def __init__(self, C, v, l_min):
        self.C, self.v, self.l_min = C, v, l_min


def desk_golden():
    out = {}
    for tag, (lmin, lmax, p, nr) in {"desk": (2, 16, 3, 54), "desk32": (2, 32, 4, 216),
                                      "small12": (2, 12, 3, 30)}.items():
        grid = cp.default_radial_grid(nr)
        t = cp.synthesize_basis(p, lmin, lmax, grid)
        m = cp.default_mode_mapping(p)
        out[f"{tag}_q"], out[f"{tag}_qt"] = t.q, t.q_tilde
        out[f"{tag}_C"], out[f"{tag}_v"] = t.C, t.v
        out[f"{tag}_r"], out[f"{tag}_entries"] = grid.r, m.entries
        out[f"{tag}_lrange"] = np.array([lmin, lmax])
        out[f"{tag}_gamma"] = cp.gamma3d_matrix(t, m, grid).values
        for integ in ("trap", "hermite", "spline"):
            out[f"{tag}_w_{integ}"] = cp.integration_weights(grid.r, integ)
        if tag == "desk":
            out["desk_naive"] = cp.gamma3d_naive(t, m, grid).values
            out["desk_exact"] = cp.gamma3d_matrix(t, m, grid, h2_mode="exact").values
            out["desk_hermite"] = cp.gamma3d_matrix(t, m, grid, integrator="hermite").values
            out["desk_spline"] = cp.gamma3d_matrix(t, m, grid, integrator="spline").values
        if tag == "small12":
            out["small12_unordered"] = cp.gamma3d_unordered_reference(t, m, grid).values
        if tag == "desk32":
            out["desk32_w4"] = cp.gamma3d_matrix(t, m, grid, workers=4).values
    return out


def c0_golden():
    from paper_1503_08809_b200.configs import host_inputs
    from oracle import qtilde_ref

    hi = host_inputs("c0")
    C, qt, delta = qtilde_ref.build(hi)
    grid = cp.RadialGrid(hi.x, (hi.x[0], hi.x[-1]))
    tables = cp.BasisTables(q=hi.q, q_tilde=qt, C=C, v=hi.v, l_min=hi.l_min,
                            l_max=hi.l_max)
    mapping = cp.ModeMapping(hi.entries, hi.spec.p)
    out = {"C": C, "qt": qt, "delta_rows": delta[[0, 50, 198]], "eps_sum": hi.eps.sum(),
           "wr2_ref": cp.integration_weights(hi.x, "trap") * hi.x ** 2}
    out["gamma"] = cp.gamma3d_matrix(tables, mapping, grid, workers=8).values
    dom = cp.enumerate_domain(hi.l_min, hi.l_max)
    for a, b in ((0, 1000), (1000, 20000), (200000, 348151)):
        sl = _Slice(dom.l1[a:b], dom.l2[a:b], dom.l3[a:b])
        out[f"partial_{a}_{b}"] = e3._sweep_chunk(
            (0, b - a, tables, mapping, grid, sl, "gosper", "trap", 64))
    out["gamma_exact"] = cp.gamma3d_matrix(tables, mapping, grid, h2_mode="exact",
                                           workers=8).values
    return out


def io_and_2d_golden():
    """Reference Γ files (harness.serialize_gamma) and the 2D engine's Γ (engine2d)."""
    from cmbproj import harness
    out = {}
    for tag, (lmin, lmax, p, nr, nmu) in {"desk": (2, 16, 3, 54, None),
                                          "desk32": (2, 32, 4, 216, 50)}.items():
        grid = cp.default_radial_grid(nr)
        t = cp.synthesize_basis(p, lmin, lmax, grid)
        m = cp.default_mode_mapping(p)
        rule = cp.gauss_legendre(nmu or cp.default_mu_points(lmax))
        leg = cp.legendre_table(lmax, rule)
        out[f"{tag}_mu_nodes"], out[f"{tag}_mu_weights"] = rule.nodes, rule.weights
        out[f"{tag}_gamma2d"] = cp.gamma2d_matrix(t, m, grid, rule, leg).values
        out[f"{tag}_ptable"] = cp.build_ptable(t, grid, rule, leg).values
        out[f"{tag}_gamma2d_naive_00"] = np.array(
            cp.gamma2d_entry_naive(0, 0, t, m, grid, rule, leg))
        out[f"{tag}_gamma3d_exact"] = cp.gamma3d_matrix(t, m, grid, h2_mode="exact").values
        if tag == "desk":
            g = cp.gamma3d_matrix(t, m, grid)
            harness.serialize_gamma(g, os.path.join(HERE, "desk_gamma.csv"), "csv")
            harness.serialize_gamma(g, os.path.join(HERE, "desk_gamma.bin"), "bin")
    return out


def main():
    if "--only-io2d" in sys.argv:
        np.savez_compressed(os.path.join(HERE, "io2d.npz"), **io_and_2d_golden())
        print("io2d.npz")
        return
    np.savez_compressed(os.path.join(HERE, "io2d.npz"), **io_and_2d_golden())
    print("io2d.npz")
    np.savez_compressed(os.path.join(HERE, "domain.npz"), **domain_golden())
    print("domain.npz")
    np.savez_compressed(os.path.join(HERE, "desk.npz"), **desk_golden())
    print("desk.npz")
    np.savez_compressed(os.path.join(HERE, "c0.npz"), **c0_golden())
    print("c0.npz")


if __name__ == "__main__":
    main()
