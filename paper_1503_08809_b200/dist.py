"""Multi-GPU Γ: one process per GPU, l2-slab shards, one exchange of the small Γ.

Reference equivalent: make_plan + fork pool + merge_partials (engine3d.py:175-186,
scheduler.py:32-66) — contiguous, balanced chunks whose private partial Γ's are summed once
in worker order.  Here a rank owns a contiguous l2 slab (`slab_plan`, balanced by the cost
model of the row-factorised kernel), computes its partial Γ on its own GPU
with no communication, and the partials are combined by one all-gather followed by a sum in
rank order — the exact analogue of merge_partials, bitwise reproducible for a fixed world
size (an NCCL all-reduce would let the ring order vary the last bit).

`torch.distributed` is the plumbing (NCCL between GPUs; gloo works for the CPU tests).
"""

from __future__ import annotations

import numpy as np

from . import _native as nat
from .engine3d import _FP_POOL, _meta_dict, check_shapes
from .gamma import GammaMatrix
from .quadrature import x_weights
from .scheduler import slab_plan

__all__ = ["rank_slab", "merge_rank_partials", "gamma3d_matrix_distributed", "slab_partial"]


def rank_slab(l_min: int, l_max: int, p: int, n_x: int, rank: int, world: int):
    """[l2_begin, l2_end) of `rank` out of `world` cost-balanced contiguous slabs."""
    b = slab_plan(l_min, l_max, p, n_x, world)
    return b[rank], b[rank + 1]


def merge_rank_partials(partial, group=None):
    """All-gather every rank's partial Γ (torch tensor, any device) and sum in rank order."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    bufs = [torch.empty_like(partial) for _ in range(world)]
    dist.all_gather(bufs, partial.contiguous(), group=group)
    out = bufs[0].clone()
    for b in bufs[1:]:
        out += b
    return out


def slab_partial(tables, mapping, wr2, l2_begin, l2_end, h2_mode="gosper", device=0):
    """Partial Γ of one l2 slab on one GPU (host in / host out)."""
    q = np.ascontiguousarray(tables.q, np.float64)
    qt = np.ascontiguousarray(tables.q_tilde, np.float64)
    C = np.ascontiguousarray(tables.C, np.float64)
    v = np.ascontiguousarray(tables.v, np.float64)
    e = np.ascontiguousarray(mapping.entries, np.int64)
    wr2 = np.ascontiguousarray(wr2, np.float64)
    check_shapes(q, qt, C, v, wr2, int(tables.l_min), int(tables.l_max))
    n = e.shape[0]
    out = np.zeros((n, n))
    nat.check(nat.lib().mg_gamma_sep_slab(
        nat.ptr(q), nat.ptr(qt), nat.ptr(C), nat.ptr(v), nat.ptr(wr2), nat.ptr(e), q.shape[0],
        qt.shape[1], n, int(tables.l_min), int(tables.l_max), nat.MG_H2[h2_mode],
        int(l2_begin), int(l2_end), int(device), nat.ptr(out)))
    return out


def gamma3d_matrix_distributed(tables, mapping, grid, h2_mode="gosper", integrator="trap",
                               block=64, workers=1, *, device=None, group=None,
                               partial_fn=None) -> GammaMatrix:
    """gamma3d_matrix over all ranks of the default process group: every rank returns the
    full Γ.  `partial_fn(tables, mapping, wr2, l2_begin, l2_end, h2_mode)` replaces the GPU
    slab kernel (used by the CPU multi-process tests to drive the host logic)."""
    import torch
    import torch.distributed as dist

    if block < 1:
        raise ValueError("block must be >= 1")
    if h2_mode not in nat.MG_H2:
        raise ValueError(f"unknown h2_mode {h2_mode!r}")
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    wr2 = x_weights(grid.r, integrator)
    fp = _FP_POOL.submit(lambda: (tables.fingerprint(), grid.fingerprint(),
                                  mapping.fingerprint()))   # hashed beside the slab's GPU work
    a, b = rank_slab(int(tables.l_min), int(tables.l_max), tables.p_max, wr2.size, rank, world)
    if partial_fn is None:
        import os
        # the rank's own GPU on its node (LOCAL_RANK), never the global rank
        dev = int(os.environ.get("LOCAL_RANK", "0")) if device is None else int(device)
        if dist.get_backend(group) == "nccl":
            # partial Γ stays in device memory for the NCCL exchange (no host round trip)
            from .plan import GammaPlan
            n = mapping.n_max
            t = torch.empty((n, n), dtype=torch.float64, device=torch.device("cuda", dev))
            plan = GammaPlan.from_tables(tables, mapping, grid, h2_mode, integrator, device=dev)
            try:
                with torch.cuda.device(dev):
                    s = torch.cuda.current_stream()
                    plan.execute(a, b, out=t, stream=s)
                    s.synchronize()
            finally:
                plan.close()
        else:
            t = torch.from_numpy(slab_partial(tables, mapping, wr2, a, b, h2_mode, dev))
    else:
        t = torch.from_numpy(np.ascontiguousarray(partial_fn(tables, mapping, wr2, a, b,
                                                             h2_mode)))
    merged = merge_rank_partials(t, group).cpu().numpy()
    meta = _meta_dict(tables, grid, mapping, integrator, h2_mode, block, workers, *fp.result())
    meta["ranks"] = world
    return GammaMatrix(merged, meta)
