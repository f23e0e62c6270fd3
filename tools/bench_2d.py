"""Performance evidence for the μ-quadrature engine (engine2d.py:62-211):
the GPU P table + Γ2d against the reference's own optimized 2D engine (cmbproj, imported
unmodified from baseline/_ref) on all host cores, same reference-constructed inputs.

    python tools/bench_2d.py [--lmax 128 --pmax 4 --r 216 --reps 3]

Prints one JSON line (GPU seconds, reference seconds, ratio, parity of the two matrices).
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
for path in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
    if os.path.isdir(os.path.join(path, "cmbproj")):
        sys.path.append(path)
        break
os.environ.setdefault("OMP_NUM_THREADS", "1")

import numpy as np  # noqa: E402

import cmbproj as cp  # noqa: E402
from paper_1503_08809_b200 import build_ptable, gamma2d_matrix  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--lmax", type=int, default=128)
ap.add_argument("--pmax", type=int, default=4)
ap.add_argument("--r", type=int, default=216)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--no-ref", action="store_true", help="skip the CPU reference (large sizes)")
a = ap.parse_args()
grid = cp.default_radial_grid(a.r)
tables = cp.synthesize_basis(a.pmax, 2, a.lmax, grid)
mapping = cp.default_mode_mapping(a.pmax)
rule = cp.gauss_legendre(cp.engine2d.default_mu_points(a.lmax))
leg = cp.legendre_table(a.lmax, rule)
cores = os.cpu_count() or 1

gpu = []
for i in range(a.reps + 1):
    t0 = time.perf_counter()
    g = gamma2d_matrix(tables, mapping, grid, rule, leg)
    if i:
        gpu.append(time.perf_counter() - t0)
t0 = time.perf_counter()
pt = build_ptable(tables, grid, rule, leg)
t_pt = time.perf_counter() - t0
if a.no_ref:
    # executed FP64 operations: P table 5 per (element, l) (1 mul + 4 Kahan adds; the A operand's
    # two multiplies are shared by a row), cells 23 per (cell, x, μ) (12 mul + 5 add of the
    # permanent, 1 FMA of the μ rule, counted as issued instructions)
    print(json.dumps({
        "engine": "modal2d (mu quadrature)", "l_max": a.lmax, "p_max": a.pmax, "n_r": a.r,
        "n_mu": rule.n, "n_modes": mapping.n_max, "gpu_s": float(np.median(gpu)),
        "gpu_ptable_s": t_pt,
        "ptable_ops": 5.0 * a.pmax ** 2 * a.r * rule.n * (a.lmax - 1),
        "cell_ops": 23.0 * mapping.n_max ** 2 * a.r * rule.n,
        "ptable_bytes": 8.0 * a.pmax ** 2 * a.r * rule.n}))
    sys.exit(0)
ref = []
for i in range(max(1, a.reps // 2)):
    t0 = time.perf_counter()
    r = cp.gamma2d_matrix(tables, mapping, grid, rule, leg, workers=cores)
    ref.append(time.perf_counter() - t0)
ref_pt = cp.build_ptable(tables, grid, rule, leg)
gap = float(np.max(np.abs(g.values - r.values)) / np.max(np.abs(r.values)))
print(json.dumps({
    "engine": "modal2d (mu quadrature)", "l_max": a.lmax, "p_max": a.pmax, "n_r": a.r,
    "n_mu": rule.n, "n_modes": mapping.n_max,
    "gpu_s": float(np.median(gpu)), "gpu_ptable_s": t_pt,
    "reference_s": float(np.median(ref)), "reference_workers": cores,
    "speedup": float(np.median(ref) / np.median(gpu)),
    "ptable_bit_identical": bool(np.array_equal(pt.values, ref_pt.values)),
    "gamma2d_relative_gap": gap,
    "note": "GPU times are end to end through the drop-in call (host inputs, P table built on "
            "the device, Γ copied back); reference = cmbproj.gamma2d_matrix(workers=cores)"}))
