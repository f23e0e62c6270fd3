"""Bounds-checked run (the stand-in for compute-sanitizer, which is closed on this pool).

    bash tools/build_variant.sh checked -DMG_CHECKED=1
    MG_LIB_PATH=$PWD/paper_1503_08809_b200/_native/variants/checked.so python tools/checked_run.py

Runs every pipeline kernel of the separable path (panels, pair products, run / x / pair
contractions, gather) and the non-separable DMMA kernel with the checked library — the small
oracle-checked case of tools/sanitize_case.py plus long-window slabs at p = 15, 22 and 30,
multi-batch and multi-group row counts — then reads the per-site violation counters
(mg_debug_checks) and fails if any global write or bulk-copy (TMA) source range left its
buffer's extent.
"""
import os
import runpy
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1503_08809_b200 import GammaPlan, _native, build_qtilde_device  # noqa: E402
from paper_1503_08809_b200.configs import host_inputs  # noqa: E402

checked, _ = _native.debug_checks(reset=True)
assert checked, "MG_LIB_PATH must point at a library built with -DMG_CHECKED=1"

runpy.run_path(os.path.join(ROOT, "tools", "sanitize_case.py"), run_name="__main__")
cases = [("c1", 1400, 1420), ("c1", 2, 400), ("c2", 2400, 2403), ("c4", 2990, 3001),
         ("c4", 1200, 1203)]
for cfg, a, b in cases:
    hi = host_inputs(cfg)
    C, qt = build_qtilde_device(hi)
    plan = GammaPlan(hi.q, qt, C.cpu().numpy(), hi.v, hi.wr2, hi.entries, 2, hi.l_max)
    plan.execute(a, b)
    g = plan.fetch()
    print(f"{cfg} l2 [{a},{b}): launches {plan.stats()['launches']}, |Γ| {abs(g).sum():.3e}")
    plan.close()
    del qt, C
_, counts = _native.debug_checks()
print("checked build, violations per site:", counts)
assert not any(counts.values()), counts
print("no bounds violations")
