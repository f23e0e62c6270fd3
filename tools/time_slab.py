"""Time the resident Γ plan on an l2 slab of a config and extrapolate to the full Γ.

    python tools/time_slab.py --config c4 --l2 1500 1530
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1503_08809_b200 import GammaPlan, build_qtilde_device  # noqa: E402
from paper_1503_08809_b200.configs import CONFIGS, host_inputs  # noqa: E402
from paper_1503_08809_b200.scheduler import slab_costs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--l2", type=int, nargs=2, default=[1500, 1530])
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
spec = CONFIGS[a.config]
hi = host_inputs(a.config)
t0 = time.perf_counter()
C, qt = build_qtilde_device(hi)
torch.cuda.synchronize()
print(f"q-tilde build {time.perf_counter() - t0:.2f} s")
plan = GammaPlan(hi.q, qt, C.cpu().numpy(), hi.v, hi.wr2, hi.entries, 2, hi.l_max)
plan.set_profile(True)
cost = slab_costs(2, hi.l_max, spec.p, spec.n_x)
frac = cost[a.l2[0] - 2:a.l2[1] - 2].sum() / cost.sum()
for r in range(a.reps):
    torch.cuda.synchronize()
    t = time.perf_counter()
    plan.execute(*a.l2)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    st = plan.stats()
    fl = st["flops_run"] + st["flops_x"] + st["flops_pair"]
    print(f"rep {r}: {dt:.3f} s, slab = {frac * 100:.2f}% of modelled work -> full Γ ~ {dt / frac:.1f} s; "
          f"executed {fl / dt / 1e12:.1f} TF/s")
ms = plan.kernel_ms()
print({k: round(v / a.reps, 1) for k, v in ms.items()})
