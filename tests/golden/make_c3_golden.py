"""Golden vectors for the full-size non-separable path (BASELINE config 3).

Runs ONLY in the build container (needs /root/reference/pkg/src for the pin and ~5 min of
8 cores for the full restatement):

    python -B tests/golden/make_c3_golden.py

Writes tests/golden/c3.npz with
  * the config-3 inputs the GPU tests need at the sparse-grid multipoles only: C [L] (all l),
    q̃ at the 244 grid l's (scipy stage-1 oracle, oracle/qtilde_ref.py), the grid and its
    1D weights;
  * b_gosper / b_exact: the restatement oracle/nonsep_ref.nonsep over ALL 724,930 sparse
    triples (fork pool) with h2_mode "gosper" / "exact" — the exact mode gives odd-parity
    and only-triangle cells weight 0, like the reference's theta gate (geometry.py:67-71);
  * a PIN of that restatement to the unmodified reference: b over a seeded sample of 240
    config-3 triples computed with the reference's own per-triple functions in the loop
    structure of gamma3d_naive (engine3d.py:189-215): radial_integral_x (:56-70, α-contracted
    inside the x integral), late_product_y (:73-83), _triple_z (:41-53) and
    permutation_multiplicity (geometry.py:114-123), times the volume weight W_t.
"""

from __future__ import annotations

import os
import sys
import time

sys.dont_write_bytecode = True
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)
os.environ.setdefault("OMP_NUM_THREADS", "1")
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

import numpy as np  # noqa: E402

import cmbproj as cp  # noqa: E402
from cmbproj import engine3d as e3  # noqa: E402
from cmbproj.geometry import permutation_multiplicity  # noqa: E402

from oracle import nonsep_ref, qtilde_ref  # noqa: E402
from paper_1503_08809_b200.configs import host_inputs, sparse_domain, sparse_grid  # noqa: E402


def reference_sample_b(tables, mapping, grid, alpha, l1, l2, l3, W, h2_mode):
    """b over a triple list with the reference's own per-triple functions (gamma3d_naive's
    loop structure, engine3d.py:189-215, with the primordial sum contracted against α)."""
    n = mapping.n_max
    b = np.zeros(n)
    for t in range(l1.size):
        a1, a2, a3 = int(l1[t]), int(l2[t]), int(l3[t])
        x = sum(alpha[np_] * e3.radial_integral_x(a1, a2, a3, np_, tables, mapping, grid)
                for np_ in range(n))
        z = float(e3._triple_z(tables, a1, a2, a3, h2_mode)) * permutation_multiplicity(a1, a2, a3)
        for m in range(n):
            b[m] += W[t] * z * x * e3.late_product_y(a1, a2, a3, m, tables, mapping)
    return b


def main():
    t0 = time.time()
    hi = host_inputs("c3")
    g, w1 = sparse_grid(l_max=hi.l_max)
    l1, l2, l3, W = sparse_domain(g, w1)
    d = qtilde_ref.delta_table(hi.k, hi.eps, hi.l_min, hi.l_max)
    C = qtilde_ref.c_ell(d, hi.k, hi.wk)
    qt = qtilde_ref.qtilde(hi.k, hi.wk, hi.x, hi.qk, d, hi.l_min, hi.l_max, ells=g)
    print(f"stage 1 at {g.size} grid multipoles: {time.time() - t0:.1f} s", flush=True)

    # pin: reference functions on a seeded sample (incl. odd-parity and step-10 cells)
    rng = np.random.default_rng(33)
    odd = np.flatnonzero((l1 + l2 + l3) % 2 == 1)
    dense = np.flatnonzero(W == 1.0)
    idx = np.unique(np.concatenate([rng.choice(l1.size, 200, replace=False),
                                    rng.choice(odd, 20, replace=False),
                                    rng.choice(dense, 20, replace=False)]))
    tables = cp.BasisTables(hi.q, qt, C, hi.v, hi.l_min, hi.l_max)
    mapping = cp.ModeMapping(hi.entries, hi.spec.p)
    rgrid = cp.RadialGrid(hi.x, (hi.x[0], hi.x[-1]))
    pin = {}
    for mode in ("gosper", "exact"):
        pin[mode] = reference_sample_b(tables, mapping, rgrid, hi.alpha, l1[idx], l2[idx],
                                       l3[idx], W[idx], mode)
    print(f"reference pin over {idx.size} triples: {time.time() - t0:.1f} s", flush=True)

    full = {}
    for mode in ("gosper", "exact"):
        full[mode] = nonsep_ref.nonsep_parallel(hi.q, qt, C, hi.v, hi.wr2, hi.entries, hi.alpha,
                                                hi.l_min, l1, l2, l3, W, h2_mode=mode)
        print(f"restatement ({mode}) over {l1.size} triples: {time.time() - t0:.1f} s",
              flush=True)
    np.savez_compressed(os.path.join(HERE, "c3.npz"), grid=g, w1d=w1, C=C,
                        qt_grid=qt[:, :, g - hi.l_min], count=l1.size,
                        b_gosper=full["gosper"], b_exact=full["exact"], sample_idx=idx,
                        sample_b_gosper=pin["gosper"], sample_b_exact=pin["exact"])


if __name__ == "__main__":
    main()
