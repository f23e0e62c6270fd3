"""Static partitioning and ordered merging — mirror of `cmbproj.scheduler` plus the
l2-slab shard plan of the multi-GPU path.

  make_plan       scheduler.py:32-45  balanced contiguous ranges, remainder first
  merge_partials  scheduler.py:48-66  entrywise sum in list order (deterministic)
  slab_plan       (new) contiguous l2 slabs balanced by the row-factorised kernel's cost
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .gamma import GammaMatrix

__all__ = ["ChunkPlan", "make_plan", "merge_partials", "slab_costs", "slab_plan"]

RUN_PAD = 20          # padded l1 values per row in the run contraction (measured)
ROW_FACTOR = 1.35     # per-row work relative to the x contraction (measured)


@dataclass(frozen=True)
class ChunkPlan:
    total: int
    ranges: tuple

    @property
    def worker_count(self) -> int:
        return len(self.ranges)


def make_plan(total: int, workers: int) -> ChunkPlan:
    if total < 0 or workers < 1:
        raise ValueError("require total >= 0 and workers >= 1")
    q, r = divmod(total, workers)
    bounds = [0]
    for w in range(workers):
        bounds.append(bounds[-1] + q + (w < r))
    return ChunkPlan(total, tuple(zip(bounds[:-1], bounds[1:])))


def merge_partials(partials) -> GammaMatrix:
    partials = list(partials)
    if not partials:
        raise ValueError("no partials to merge")
    head = partials[0]
    if any(not head.same_inputs(p) for p in partials[1:]):
        raise ValueError("partial matrices have mismatched shape or input fingerprints")
    acc = head.values.copy()
    for p in partials[1:]:
        acc += p.values
    meta = dict(head.meta)
    meta["workers_merged"] = len(partials)
    return GammaMatrix(acc, meta)


def slab_costs(l_min: int, l_max: int, p: int, n_x: int) -> np.ndarray:
    """Modelled FP64 work of every l2 value for the row-factorised Γ kernel.

    A (l2,l3)-row with an l1-run of m triples costs p^2·Nx·m FMAs (run contraction) plus
    p(p+1)/2·p^2·Nx FMAs (x contraction) — see DESIGN.md §3.  Calibrated on a B200 (tools/
    slab_balance.py): the run contraction pays ~20 padded l1 values per row (tile union and
    k-tile rounding), and per-row work outside the two contractions (operand builds, gather,
    pair contraction) adds ~35 % to the x contraction's cost.  Returns cost[l2 - l_min].
    """
    pairs = p * (p + 1) // 2
    out = np.zeros(l_max - l_min + 1)
    for l2 in range(l_min, l_max + 1):
        l3 = np.arange(l2, min(2 * l2, l_max) + 1)
        lo = np.maximum(l3 - l2, l_min)
        lo = lo + ((lo + l2 + l3) & 1)
        hi = np.where((l3 & 1) == 0, l2, l2 - 1)        # l1 <= l2, l1+l2+l3 even
        m = np.maximum((hi - lo) // 2 + 1, 0)
        m = m[hi >= lo]
        out[l2 - l_min] = p * p * n_x * (m + RUN_PAD).sum() + m.size * ROW_FACTOR * pairs * p * p * n_x
    return out


def slab_plan(l_min: int, l_max: int, p: int, n_x: int, nshards: int) -> list[int]:
    """Contiguous l2 slabs with (modelled) equal work: bounds[0]=l_min .. bounds[-1]=l_max+1."""
    if nshards < 1:
        raise ValueError("nshards must be >= 1")
    cost = slab_costs(l_min, l_max, p, n_x)
    cum = np.concatenate([[0.0], np.cumsum(cost)])
    bounds = [l_min]
    for s in range(1, nshards):
        target = cum[-1] * s / nshards
        idx = int(np.searchsorted(cum, target))
        bounds.append(max(bounds[-1], min(l_min + idx, l_max + 1)))
    bounds.append(l_max + 1)
    return bounds
