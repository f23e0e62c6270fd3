"""Time the on-device q̃ build (stage 1) of a config: python tools/time_qtilde.py c1 [reps]."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1503_08809_b200 import build_qtilde_device  # noqa: E402
from paper_1503_08809_b200.configs import CONFIGS, host_inputs  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c1"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
spec = CONFIGS[cfg]
hi = host_inputs(cfg)
L = spec.l_max - 1
flops = 2.0 * spec.p * L * spec.n_x * spec.n_k
for r in range(reps):
    torch.cuda.synchronize()
    t = time.perf_counter()
    C, qt = build_qtilde_device(hi)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(f"{cfg} rep {r}: {dt:.3f} s  contraction {flops / dt / 1e12:.1f} TF/s "
          f"(2pLNxNk = {flops:.3g}), q-tilde write {qt.numel() * 8 / dt / 1e9:.1f} GB/s")
