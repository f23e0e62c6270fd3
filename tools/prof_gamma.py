"""Profiling driver: one config's q̃ on the GPU, then Γ over a small l2 slab (for ncu).

    python tools/prof_gamma.py [--config c1] [--l2 1400 1420] [--reps 2]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1503_08809_b200 import GammaPlan, build_qtilde_device  # noqa: E402
from paper_1503_08809_b200.configs import host_inputs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c1")
ap.add_argument("--l2", type=int, nargs=2, default=[1400, 1420])
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
hi = host_inputs(a.config)
C, qt = build_qtilde_device(hi)
plan = GammaPlan(hi.q, qt, C.cpu().numpy(), hi.v, hi.wr2, hi.entries, 2, hi.l_max)
plan.set_profile(True)
for r in range(a.reps):
    torch.cuda.synchronize()
    t = time.perf_counter()
    plan.execute(*a.l2)
    torch.cuda.synchronize()
    print(f"rep {r}: {time.perf_counter() - t:.4f} s", plan.stats(), plan.kernel_ms())
