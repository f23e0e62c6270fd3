"""Time each rank's l2 slab of an N-way split on one GPU (sequentially) to measure the
load balance the multi-GPU run will see: max/mean of the per-slab times.

    python tools/slab_balance.py --config c1 --shards 8
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1503_08809_b200 import GammaPlan, build_qtilde_device, slab_plan  # noqa: E402
from paper_1503_08809_b200.configs import CONFIGS, host_inputs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c1")
ap.add_argument("--shards", type=int, default=8)
ap.add_argument("--bounds", type=int, nargs="*", default=None)
ap.add_argument("--profile", action="store_true")
ap.add_argument("--rounds", type=int, default=1)
a = ap.parse_args()
spec = CONFIGS[a.config]
hi = host_inputs(a.config)
C, qt = build_qtilde_device(hi)
plan = GammaPlan(hi.q, qt, C.cpu().numpy(), hi.v, hi.wr2, hi.entries, 2, hi.l_max)
b = a.bounds or slab_plan(2, hi.l_max, spec.p, spec.n_x, a.shards)
plan.execute(b[0], b[1])  # warm-up (allocations)
times = []
fam = []
for i in [k for _ in range(a.rounds) for k in range(len(b) - 1)]:
    plan.set_profile(a.profile)
    torch.cuda.synchronize()
    t = time.perf_counter()
    plan.execute(b[i], b[i + 1])
    torch.cuda.synchronize()
    times.append(time.perf_counter() - t)
    if a.profile:
        fam.append({k: round(v, 1) for k, v in plan.kernel_ms().items()} | plan.stats())
    plan.set_profile(False)
for f in fam:
    print(f)
t = np.array(times)
print(json.dumps({"config": a.config, "bounds": b, "slab_s": t.round(4).tolist(),
                  "sum_s": float(t.sum()), "max_over_mean": float(t.max() / t.mean()),
                  "ideal_scaling_eff": float(t.mean() / t.max())}))
