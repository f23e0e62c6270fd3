"""Γ projection benchmark (BASELINE.json metric: (l-triple·x·mode) FP64 updates/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c1] [--impl b200|reference]

One "step" = one full separable Γ (BASELINE config 1 by default: l_max=2000, p=15 -> 680
modes, Nx=500, 334,831,501 ordered triples) with q̃ already resident in HBM.  For N>1
(launched by torchrun) every rank computes one cost-balanced l2 slab and the partial Γ's
are all-gathered over NCCL and summed in rank order; the step time is the max over ranks.

`--impl reference` times the reference algorithm on the host CPU cores instead (the
reference is pure Python/NumPy and cannot be compiled; its NumPy restatement in oracle/ is
the same code path, pinned bit-for-bit to the reference on config 0): rank 0 only, each
step a bounded flat-range sample of the same config.
"""

from __future__ import annotations

import os

os.environ.setdefault("OMP_NUM_THREADS", "1")        # before numpy: CPU baseline is 1 thread/worker
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

import argparse
import json
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FP64_PEAK_TFLOPS = 37.0  # measured DMMA peak on this pool's B200 (profiles/r01_fp64_peak.txt)
FP64_PEAK_SRC = "measured: tools/fp64_peak.cu DMMA.8x8x4 microbenchmark, profiles/r01_fp64_peak.txt"
UPDATE_FLOPS = 6.0       # algorithmic FP64 FLOPs per (l-triple, x, mode) update


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c1")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-reps", type=int, default=3)
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--cpu-full", action="store_true",
                    help="config 3: run the CPU restatement over ALL sparse triples")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: exchange Γ partials through host memory (lets N ranks share "
                         "one GPU for testing the multi-rank path; never for measurements)")
    return ap.parse_args()


# ------------------------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region.  One long-lived
    `nvidia-smi -lms 200` process streams the samples (no fork per sample, so the sampler
    cannot stall the launching thread)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int, period_ms: int = 200):
        self.gpu = gpu
        self.period_ms = period_ms
        self.samples = []
        self._proc = None
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        try:
            for line in self._proc.stdout:
                line = line.strip()
                if line:
                    self.samples.append([x.strip() for x in line.split(",")])
        except Exception:
            pass

    def __enter__(self):
        try:
            self._proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", str(self.period_ms)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t.start()
        except Exception:
            self._proc = None
        return self

    def __exit__(self, *a):
        if self._proc is not None:
            self._proc.terminate()
            try:
                self._proc.wait(timeout=5)
            except Exception:
                self._proc.kill()
            self._t.join(timeout=5)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 3 + i and s[3 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def total_updates(spec):
    """(triples, updates per Γ, modes).  Counted with the oracle's C restatement of the
    enumeration (oracle/domain_ref.c), so the reference arm never maps the product library."""
    from oracle import ref
    T = ref.domain_count(2, spec.l_max)
    n = (spec.p * (spec.p + 1) * (spec.p + 2)) // 6
    return T, T * spec.n_x * n, n


def cpu_model() -> str:
    """Host CPU model (lscpu "Model name") for the cpu_baseline record."""
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.lower().startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def native_maps() -> list:
    """Shared objects of this repo mapped into the process (evidence for the arms)."""
    try:
        return sorted({ln.split()[-1] for ln in open("/proc/self/maps")
                       if ln.rstrip().endswith(".so") and ROOT in ln})
    except Exception:
        return []


# ------------------------------------------------------------------------------------------
def cpu_rate(hi, qt_host, C, seconds, cores):
    """Oracle port (= reference _sweep_chunk code path) on bounded flat slices at 10 %, 50 % and
    90 % of the triple index (per-triple work n·Nx is uniform, so the rate
    extrapolates linearly in T), all cores, per-call pool setup measured on an empty range and
    subtracted."""
    from oracle import ref

    T = ref.domain_count(2, hi.l_max)
    n = hi.entries.shape[0]
    per_core = 1.5e7                                  # upd/s/core, SURVEY §6 (c0..c4 slices)
    S = max(cores * 8, int(seconds / 3 * per_core * cores / (hi.x.size * n)))
    S = min(S, T // 3)
    starts = [min(int(f * T), T - S) for f in (0.1, 0.5, 0.9)]
    dt = 0.0
    for a in starts:
        t0 = time.perf_counter()
        ref.gamma3d(hi.q, qt_host, C, hi.v, hi.wr2, hi.entries, 2, hi.l_max, a, a + S,
                    workers=cores, block=64)
        dt += time.perf_counter() - t0
    a = starts[1]
    t0 = time.perf_counter()                    # per-call pool setup (empty range), subtracted
    ref.gamma3d(hi.q, qt_host, C, hi.v, hi.wr2, hi.entries, 2, hi.l_max, a, a,
                workers=cores, block=64)
    dt = max(dt - 3 * (time.perf_counter() - t0), 1e-9)
    return 3 * S * hi.x.size * n / dt, S, starts, dt


def run_nonsep(args):
    """Config 3: non-separable pointwise projection on the sparse l-grid (one step = one
    b = Σ_t W zm P Σ_x wr2 B(t,x) over all sparse triples).  `value`: resident plan (q̃ and
    the sparse domain in HBM, b left on the device), CUDA events on the launching stream;
    `e2e`: the public gamma_nonsep call with host buffers (plan build + uploads inside)."""
    import torch

    from paper_1503_08809_b200 import (BasisTables, GammaPlan, ModeMapping, RadialGrid,
                                       SparseDomain, build_qtilde, gamma_nonsep)
    from paper_1503_08809_b200.configs import CONFIGS, host_inputs, sparse_domain, sparse_grid

    world, rank, local = dist_env()
    if rank != 0:
        return
    torch.cuda.set_device(local)
    spec = CONFIGS[args.config]
    hi = host_inputs(spec)
    C, qt = build_qtilde(hi)
    t = BasisTables(hi.q, qt, C, hi.v, 2, hi.l_max)
    m = ModeMapping(hi.entries, spec.p)
    grid = RadialGrid(hi.x)
    dom = SparseDomain(*sparse_domain(*sparse_grid(l_max=spec.l_max)))
    n = hi.entries.shape[0]
    U = dom.count * spec.n_x * n
    p, P2 = spec.p, spec.p * (spec.p + 1) // 2
    exec_per_tx = 3 * P2 + 2 * p * P2 + 2 * p + 2      # S_ab, Ã·S, q̃(l1)·T, x integral
    exec_flops = exec_per_tx * dom.count * spec.n_x

    plan = GammaPlan(hi.q, qt, C, hi.v, hi.wr2, hi.entries, 2, spec.l_max, device=local)
    plan.set_sparse_domain(dom)
    stream = torch.cuda.current_stream()
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")  # > L2
    for _ in range(args.warmup):
        plan.nonsep(hi.alpha, out=out, stream=stream)
    torch.cuda.synchronize()
    plan.set_profile(True)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.zero_()
            evs[i][0].record(stream)
            plan.nonsep(hi.alpha, out=out, stream=stream)
            evs[i][1].record(stream)
        torch.cuda.synchronize()
    step_ms = [s.elapsed_time(e) for s, e in evs]
    ms = float(np.mean(step_ms))
    k_ms = plan.kernel_ms()["nonsep"] / args.steps
    b_dev = out.cpu().numpy()
    plan.close()

    for _ in range(2):
        gamma_nonsep(t, m, grid, hi.alpha, dom)
    e2e = []
    for _ in range(max(1, args.e2e_reps)):
        t0 = time.perf_counter()
        b = gamma_nonsep(t, m, grid, hi.alpha, dom)
        e2e.append(time.perf_counter() - t0)
    e2e_s = float(np.median(e2e))
    achieved = exec_flops / (k_ms / 1e3) / 1e12
    if p <= 8 and not os.environ.get("MG_NS_DFMA"):
        kname = f"k_nonsep_dmma<{4 if p <= 4 else 8}>"
        knote = ("FP64 tensor pipe: the Ã·S contraction (M = p) on DMMA.8x8x4, pair products "
                 "and the l1/x reductions on DFMA (same FP64 datapath, peak shared)")
    else:
        kname = f"k_nonsep_warp<{p}>"
        knote = "DFMA-pipe bound pointwise kernel"

    # CPU baseline: the restatement (oracle/nonsep_ref.py, gamma3d_naive's loop structure)
    # on a strided sample of the sparse triples (or all of them with --cpu-full), with all
    # host cores; the GPU result over the same sub-domain is checked against it.
    cpu = None
    if not args.no_cpu_baseline:
        from oracle import nonsep_ref
        cores = os.cpu_count() or 1
        per_core = 1.0e7                                 # upd/s/core of the restatement
        S = dom.count if args.cpu_full else min(
            dom.count, max(cores * 64, int(args.cpu_seconds * per_core * cores / (spec.n_x * n))))
        idx = np.unique(np.linspace(0, dom.count - 1, S).astype(np.int64))
        sub = SparseDomain(dom.l1[idx], dom.l2[idx], dom.l3[idx], dom.weight[idx])
        t0 = time.perf_counter()
        b_cpu = nonsep_ref.nonsep_parallel(hi.q, qt, C, hi.v, hi.wr2, hi.entries, hi.alpha, 2,
                                           sub.l1, sub.l2, sub.l3, sub.weight, workers=cores)
        dt = time.perf_counter() - t0
        b_gpu = b.values[:, 0] if idx.size == dom.count else \
            gamma_nonsep(t, m, grid, hi.alpha, sub).values[:, 0]
        err = float(np.linalg.norm(b_gpu - b_cpu) / np.linalg.norm(b_cpu))
        cpu = {"value": idx.size * spec.n_x * n / dt, "unit": "updates/s", "cores": cores,
               "kind": "port", "cpu_model": cpu_model(),
               "sample": (f"oracle/nonsep_ref.nonsep_parallel (gamma3d_naive loop structure) "
                          f"over {'ALL' if idx.size == dom.count else 'a strided sample of'} "
                          f"{idx.size} of {dom.count} sparse triples, fork pool of {cores}, "
                          f"{dt:.1f} s; GPU b over the same triples: rel err {err:.2e} "
                          f"(tolerance 1e-8)"),
               "rel_err_vs_gpu": err, "s": dt}
        assert err <= 1e-8, f"non-separable GPU/CPU mismatch {err:.3e}"
    line = {"metric": "Γ projection: (l-triple·x·mode) FP64 updates/s", "value": U / (ms / 1e3),
            "unit": "updates/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "ms_per_step_min": float(np.min(step_ms)),
            "ms_per_step_median": float(np.median(step_ms)),
            "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded config-3 inputs)",
            "config": {"workload": f"non-separable pointwise projection, BASELINE config 3: "
                                   f"{dom.count} sparse triples, Nx={spec.n_x}, {n} modes",
                       "updates_per_step": U,
                       "l2_flush": "256 MiB write between timed steps (untimed)"},
            "roofline": {"bound": "tensor", "kernel": kname, "achieved": achieved,
                         "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                         "frac": achieved / FP64_PEAK_TFLOPS, "traffic": None,
                         "executed_flops_per_tx": exec_per_tx,
                         "note": knote + "; executed FLOPs (3 P2 + 2 p P2 + 2 p + 2 per "
                                 "(triple, x)) / kernel time (CUDA events on the stream)",
                         "kernel_ms_per_step": k_ms},
            "e2e": {"value": U / e2e_s, "unit": "updates/s",
                    "h2d_bytes_per_step": int(qt.nbytes + hi.q.nbytes + dom.count * 20),
                    "d2h_bytes_per_step": int(n * 8), "s": e2e_s,
                    "matches_device_result": bool(np.allclose(b.values[:, 0], b_dev,
                                                              rtol=1e-12, atol=0)),
                    "note": "timed through the public gamma_nonsep call with host buffers"},
            "gpu_launches": 2,
            "b_norm": float(np.linalg.norm(b.values)), "clocks": clk.summary()}
    if cpu is not None:
        line["cpu_baseline"] = cpu
    print(json.dumps(line), flush=True)


def run_2d(args):
    """`--config 2d`: the μ-quadrature engine (engine2d.py:62-211) at
    l_max 512 / p 8 / Nx 300 (771 μ nodes, 120 modes).  A step is one Γ2d: the Kahan P table
    plus the cell sums.  `value` = kernel time (CUDA events around the launches inside the
    library, inputs already uploaded); `e2e` = the drop-in gamma2d_matrix call with host
    buffers; `cpu_baseline` = the NumPy restatement on a subset of the radial points, against
    which the GPU result on the same subset is checked."""
    import torch

    from paper_1503_08809_b200 import (BasisTables, RadialGrid, default_mode_mapping,
                                       gamma2d_matrix, gauss_legendre, legendre_table,
                                       shifted_legendre)
    from paper_1503_08809_b200.engine2d import default_mu_points, last_kernel_ms
    from paper_1503_08809_b200.quadrature import x_weights

    world, rank, local = dist_env()
    if rank != 0:
        return
    torch.cuda.set_device(local)
    lmin, lmax, p, nx = 2, 512, 8, 300
    rng = np.random.default_rng(2015)
    L = lmax - lmin + 1
    ells = np.arange(lmin, lmax + 1, dtype=np.float64)
    tables = BasisTables(shifted_legendre(p, lmin, lmax), rng.standard_normal((p, nx, L)) * 1e-3,
                         rng.uniform(0.5, 2.0, L) * 1e-3, (2.0 * ells + 1.0) ** (1.0 / 6.0),
                         lmin, lmax)
    grid = RadialGrid(np.linspace(13000.0, 14500.0, nx))
    mapping = default_mode_mapping(p)
    rule = gauss_legendre(default_mu_points(lmax))
    leg = legendre_table(lmax, rule)
    n, nmu = mapping.n_max, rule.n
    U = n * n * nx * nmu
    P2 = p * (p + 1) // 2
    ops_pt = 5.0 * p * p * nx * nmu * L                    # 1 mul + 4 Kahan add/sub, no FMA
    flops_cells = 2.0 * p * p * P2 * P2 * nx * nmu         # the DMMA GEMM (p <= 8)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    for _ in range(args.warmup):
        g = gamma2d_matrix(tables, mapping, grid, rule, leg, device=local)
    pt_ms, cell_ms, e2e = [], [], []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            g = gamma2d_matrix(tables, mapping, grid, rule, leg, device=local)
            e2e.append(time.perf_counter() - t0)
            a, b = last_kernel_ms()
            pt_ms.append(a)
            cell_ms.append(b)
    ms = float(np.mean(pt_ms) + np.mean(cell_ms))
    e2e_s = float(np.median(e2e))
    k_pt, k_cell = float(np.mean(pt_ms)), float(np.mean(cell_ms))
    h2d = sum(x.nbytes for x in (tables.q, tables.q_tilde, tables.C, tables.v, leg[lmin:],
                                 rule.weights, mapping.entries)) + nx * 8
    if k_pt >= k_cell:
        roof = {"bound": "tensor", "kernel": "k_ptable_tiled",
                "achieved": ops_pt / (k_pt / 1e3) / 1e12, "peak": FP64_PEAK_TFLOPS / 2,
                "unit": "TFLOP/s",
                "note": "FP64 pipe, not the tensor cores: 5 individually rounded operations per "
                        "(element, l) (1 mul + 4 Kahan add/sub; fusing any would break the "
                        "bit-identical table), peak = the pipe's instruction rate = DFMA peak / 2"}
    else:
        roof = {"bound": "tensor", "kernel": "k_gamma2d_dmma", "achieved":
                flops_cells / (k_cell / 1e3) / 1e12, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                "note": "cell sum as a DMMA.8x8x4 GEMM, M = p², N = (p(p+1)/2)², K = Nx·nμ"}
    roof["frac"] = roof["achieved"] / roof["peak"]
    roof["traffic"] = None
    roof["kernel_ms_per_step"] = {"ptable": k_pt, "cells": k_cell}
    roof["cells_tflops"] = flops_cells / (k_cell / 1e3) / 1e12
    roof["ptable_tops"] = ops_pt / (k_pt / 1e3) / 1e12
    cpu = None
    if not args.no_cpu_baseline:
        from oracle import gamma2d_ref
        xs = np.unique(np.linspace(0, nx - 1, 24).astype(int))
        sub = BasisTables(tables.q, np.ascontiguousarray(tables.q_tilde[:, xs]), tables.C,
                          tables.v, lmin, lmax)
        subgrid = RadialGrid(grid.r[xs])
        wr2 = x_weights(subgrid.r)
        t0 = time.perf_counter()
        Pc = gamma2d_ref.ptable(sub.q, sub.q_tilde, sub.C, sub.v, lmin, lmax, leg)
        want = gamma2d_ref.gamma2d(Pc, mapping.entries, rule.weights, wr2)
        dt = time.perf_counter() - t0
        got = gamma2d_matrix(sub, mapping, subgrid, rule, leg, device=local).values
        err = float(np.max(np.abs(got - want)) / np.max(np.abs(want)))
        assert err <= 1e-12, f"2D engine GPU/CPU mismatch {err:.3e}"
        cpu = {"value": n * n * xs.size * nmu / dt, "unit": "updates/s", "cores": 1,
               "kind": "port", "cpu_model": cpu_model(),
               "sample": f"oracle/gamma2d_ref.py (NumPy restatement of build_ptable + "
                         f"gamma2d_entry, one thread) on {xs.size} of {nx} radial points, "
                         f"{dt:.1f} s; GPU Γ2d on the same points: max rel gap {err:.1e}",
               "rel_err_vs_gpu": err, "s": dt}
    line = {"metric": "Γ2d μ-quadrature: (cell·x·μ) FP64 updates/s", "value": U / (ms / 1e3),
            "unit": "updates/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded tables of the stated shapes)",
            "config": {"workload": f"2D μ-quadrature engine: l_max={lmax}, p={p} -> {n} modes, "
                                   f"Nx={nx}, {nmu} μ nodes", "updates_per_step": U,
                       "l2_flush": "256 MiB write between timed steps (untimed)"},
            "roofline": roof,
            "e2e": {"value": U / e2e_s, "unit": "updates/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(n * n * 8), "s": e2e_s,
                    "note": "the public gamma2d_matrix call with host buffers"},
            "gpu_launches": 3, "gamma_norm": float(np.linalg.norm(g.values)),
            "clocks": clk.summary()}
    if cpu is not None:
        line["cpu_baseline"] = cpu
    print(json.dumps(line), flush=True)


def run_b200(args):
    import torch

    from paper_1503_08809_b200 import (BasisTables, GammaPlan, ModeMapping, RadialGrid,
                                       build_qtilde_device, gamma3d_matrix, slab_plan)
    from paper_1503_08809_b200.configs import CONFIGS, host_inputs

    world, rank, local = dist_env()
    local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    if world > 1:
        # NCCL communicator lines (nranks, NVLS/P2P transport) stay visible in the log
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    gloo = args.dist_backend == "gloo"
    backend_note = None
    if world > 1:
        import torch.distributed as dist
        if not gloo:
            try:
                dist.init_process_group("nccl", device_id=torch.device("cuda", local))
            except Exception as exc:  # keep the run alive: the exchange is one n x n Γ
                backend_note = f"nccl init failed ({type(exc).__name__}); Γ exchanged over gloo"
                gloo = True
        if gloo:
            dist.init_process_group("gloo")
    spec = CONFIGS[args.config]
    hi = host_inputs(spec)
    T, U, nmodes = total_updates(spec)
    stream = torch.cuda.current_stream()

    torch.cuda.synchronize()
    t0 = time.perf_counter()
    C_dev, qt_dev = build_qtilde_device(hi, device=local, stream=stream)
    torch.cuda.synchronize()
    t_qtilde = time.perf_counter() - t0
    # stage 1 again, timed on the device (inputs already uploaded by the first build's plan
    # of record; the host uploads of ε/k/x are inside this figure too, so it is conservative)
    qe = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    qe[0].record(stream)
    C_dev, qt_dev = build_qtilde_device(hi, device=local, stream=stream)
    qe[1].record(stream)
    torch.cuda.synchronize()
    t_qt_dev = qe[0].elapsed_time(qe[1]) / 1e3
    Lq = spec.l_max - 1
    qt_bytes = 8 * spec.p * spec.n_x * Lq + 8 * Lq
    qt_flops = 2.0 * spec.p * Lq * spec.n_x * spec.n_k + 4.0 * Lq * spec.n_k * spec.n_x
    C = C_dev.cpu().numpy()
    plan = GammaPlan(hi.q, qt_dev, C, hi.v, hi.wr2, hi.entries, 2, hi.l_max, device=local)
    bounds = slab_plan(2, hi.l_max, spec.p, spec.n_x, world)
    a, b = bounds[rank], bounds[rank + 1]
    out = torch.empty((nmodes, nmodes), dtype=torch.float64, device="cuda")
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")  # > L2

    def step():
        plan.execute(a, b, out=out, stream=stream)
        if world > 1:
            from paper_1503_08809_b200.dist import merge_rank_partials
            if gloo:
                return merge_rank_partials(out.cpu()).to(out.device)
            return merge_rank_partials(out)
        return out

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    plan.set_profile(True)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.zero_()                            # L2 flush between timed steps (untimed)
            evs[i][0].record(stream)
            res = step()
            evs[i][1].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    ms_steps = [s.elapsed_time(e) for s, e in evs]
    ms = float(np.mean(ms_steps))
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device="cpu" if gloo else "cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    kms = plan.kernel_ms()
    stats = plan.stats()
    gamma_dev = res.clone()

    # ---- end-to-end through the public drop-in API with host buffers ----
    qt_host = qt_dev.cpu().numpy()
    tables = BasisTables(hi.q, qt_host, C, hi.v, 2, hi.l_max)
    mapping = ModeMapping(hi.entries, spec.p)
    grid = RadialGrid(hi.x)
    h2d = sum(x.nbytes for x in (hi.q, qt_host, C, hi.v, hi.wr2, hi.entries))
    d2h = nmodes * nmodes * 8
    e2e_t = []
    for _ in range(max(1, args.e2e_reps)):
        if world > 1:
            from paper_1503_08809_b200.dist import gamma3d_matrix_distributed
            torch.distributed.barrier()
            t1 = time.perf_counter()
            g = gamma3d_matrix_distributed(tables, mapping, grid, device=local)
        else:
            t1 = time.perf_counter()
            g = gamma3d_matrix(tables, mapping, grid, device=local)
        e2e_t.append(time.perf_counter() - t1)
    e2e_s = float(np.median(e2e_t))
    if world > 1:
        t = torch.tensor([e2e_s], dtype=torch.float64, device="cpu" if gloo else "cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_match = bool(np.allclose(g.values, gamma_dev.cpu().numpy(), rtol=1e-12, atol=0))

    if rank != 0:
        if world > 1:
            torch.distributed.barrier()
            torch.distributed.destroy_process_group()
        return

    fams = {"run": stats["flops_run"], "x": stats["flops_x"], "pair": stats["flops_pair"]}
    names = {"run": "k_run_contract", "x": "k_x_contract", "pair": "k_pair_contract"}
    dom = max(fams, key=lambda f: kms[f])
    steps = args.steps
    k_time = kms[dom] / 1e3 / steps
    achieved = fams[dom] / k_time / 1e12 if k_time > 0 else 0.0
    exec_flops = sum(fams.values())
    step_s = ms / 1e3
    traffic, traffic_note = None, None
    for rnd in ("r02", "r01"):                       # newest committed ncu --set full capture
        tfile = os.path.join(ROOT, "profiles", f"{rnd}_ncu_traffic.json")
        if not os.path.exists(tfile):
            continue
        table = json.load(open(tfile))
        tr = next((v for k, v in table.items() if k.startswith(names[dom])), None)
        if tr:
            traffic = tr["dram_bytes"]
            traffic_note = (f"dram read+write bytes of one profiled {names[dom]} launch "
                            f"({tr['duration_ms']:.2f} ms, config-1 l2 slab [1400,1420)) from "
                            f"ncu --set full, profiles/{rnd}_ncu_full_c1.txt: the H/S "
                            f"intermediates' round trip (DESIGN.md §4), not re-reads of q̃")
            break
    line = {
        "metric": "Γ projection: (l-triple·x·mode) FP64 updates/s",
        "value": U / step_s,
        "unit": "updates/s",
        "n_gpus": world,
        "steps": steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded, BASELINE.json config shapes; q̃ built on-device from "
                "Bessel/transfer inputs)",
        "dist_backend": (("gloo" if gloo else "nccl") if world > 1 else None),
        "dist_note": backend_note,
        "config": {"workload": f"separable Γ, BASELINE config {args.config[1:]}: "
                               f"l_max={spec.l_max}, p={spec.p} -> {nmodes} modes, "
                               f"Nx={spec.n_x}, Nk={spec.n_k}, T={T} ordered triples",
                   "updates_per_step": U, "parallelism": f"l2-slab x{world}",
                   "l2_flush": "256 MiB write between timed steps (untimed); q̃ tables "
                               "(QT+WQT 2x128 MB) exceed L2"},
        "s_per_gamma": step_s,
        "effective_fp64_tflops": UPDATE_FLOPS * U / step_s / 1e12,
        "effective_fp64_frac": UPDATE_FLOPS * U / step_s / 1e12 / FP64_PEAK_TFLOPS,
        "executed_fp64_tflops": exec_flops / world / step_s / 1e12 if world == 1 else None,
        "executed_fp64_frac": exec_flops / step_s / 1e12 / FP64_PEAK_TFLOPS if world == 1
        else None,
        "roofline": {"bound": "tensor", "kernel": names[dom], "achieved": achieved,
                     "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                     "frac": achieved / FP64_PEAK_TFLOPS, "traffic": traffic,
                     "traffic_note": traffic_note,
                     "peak_source": FP64_PEAK_SRC + " (MEASURED_PEAKS.json has no FP64 entry)",
                     "kernel_ms_per_step": {k: v / steps for k, v in kms.items()},
                     # shares of the main (critical-path) stream; "operands_side" runs
                     # concurrently on the side stream and is reported, not shared
                     "kernel_share": {k: v / max(sum(x for f, x in kms.items()
                                                     if f != "operands_side"), 1e-9)
                                      for k, v in kms.items() if k != "operands_side"}},
        "e2e": {"value": U / e2e_s, "unit": "updates/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h), "s_per_gamma": e2e_s,
                "matches_device_result": e2e_match},
        "gpu_launches": int(stats["launches"]),
        "qtilde_build_s": t_qtilde,
        "qtilde": {"s": t_qt_dev, "bytes_written": qt_bytes, "gbs": qt_bytes / t_qt_dev / 1e9,
                   "flops": qt_flops, "tflops": qt_flops / t_qt_dev / 1e12,
                   "note": "stage 1 (Bessel recurrences + DMMA contraction over k), CUDA events "
                           "around build_qtilde_device incl. its ε/k/x uploads; q̃ write "
                           "bytes / time = the HBM GB/s north_star asks for (latency-bound "
                           "recurrence, not HBM-bound; DESIGN.md §5)"},
        "clocks": clk.summary(),
    }
    if world == 1 and not args.no_cpu_baseline:
        cores = os.cpu_count() or 1
        rate, S, a0, dt = cpu_rate(hi, qt_host, C, args.cpu_seconds, cores)
        line["cpu_baseline"] = {
            "value": rate, "unit": "updates/s", "cores": cores, "kind": "port",
            "cpu_model": cpu_model(),
            "sample": f"oracle port of engine3d._sweep_chunk (B=64, fork pool of {cores}) over "
                      f"3 flat ranges of {S} triples starting at {a0} (10/50/90 % of the index) "
                      f"of config {args.config[1:]} ({3 * S} triples, {dt:.1f} s); "
                      f"extrapolated s/Γ = {U / rate:.3g}"}
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


# ------------------------------------------------------------------------------------------
def run_reference_nonsep(args):
    """Reference arm at config 3: the restatement of the non-separable path (gamma3d_naive's
    loop structure, oracle/nonsep_ref.py) on a strided sample of the sparse triples per step,
    all host cores, seeded synthetic q̃/C of the config's shapes."""
    from oracle import nonsep_ref
    from paper_1503_08809_b200.configs import CONFIGS, host_inputs, sparse_domain, sparse_grid

    spec = CONFIGS[args.config]
    hi = host_inputs(spec)
    l1, l2, l3, W = sparse_domain(*sparse_grid(l_max=spec.l_max))
    n = hi.entries.shape[0]
    cores = os.cpu_count() or 1
    step_s = min(args.cpu_seconds, 150.0 / max(1, args.steps + args.warmup))
    S = min(l1.size, max(cores * 64, int(step_s * 1.0e7 * cores / (spec.n_x * n))))
    idx = np.unique(np.linspace(0, l1.size - 1, S).astype(np.int64))
    rng = np.random.default_rng(spec.seed)
    qt = rng.standard_normal((spec.p, spec.n_x, spec.l_max - 1)) * 1e-10
    C = rng.uniform(1e-5, 5e-2, spec.l_max - 1)
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        nonsep_ref.nonsep_parallel(hi.q, qt, C, hi.v, hi.wr2, hi.entries, hi.alpha, 2, l1[idx],
                                   l2[idx], l3[idx], W[idx], workers=cores)
        if i >= args.warmup:
            times.append(time.perf_counter() - t0)
    dt = float(np.mean(times))
    rate = idx.size * spec.n_x * n / dt
    sample = (f"non-separable restatement (gamma3d_naive loop structure) over a strided sample "
              f"of {idx.size} of {l1.size} config-3 sparse triples per step (seeded synthetic "
              f"q̃/C of the config's shapes), fork pool of {cores}, on {cpu_model()}")
    line = {
        "metric": "Γ projection: (l-triple·x·mode) FP64 updates/s", "value": rate,
        "unit": "updates/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, BASELINE config shapes)",
        "config": {"workload": f"non-separable pointwise projection, BASELINE config 3 (strided "
                               f"sample per step)", "updates_per_step": idx.size * spec.n_x * n,
                   "parallelism": f"cpu x{cores}"},
        "impl": "reference",
        "cpu_baseline": {"value": rate, "unit": "updates/s", "cores": cores, "kind": "port",
                         "cpu_model": cpu_model(), "sample": sample},
        "e2e": {"value": rate, "unit": "updates/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "native_so_loaded": native_maps(),
    }
    print(json.dumps(line), flush=True)


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    if args.config == "c3":
        return run_reference_nonsep(args)
    from oracle import ref
    from paper_1503_08809_b200.configs import CONFIGS, host_inputs

    spec = CONFIGS[args.config]
    hi = host_inputs(spec)
    T, U, nmodes = total_updates(spec)
    cores = os.cpu_count() or 1
    per_core = 1.0e7                                  # upd/s/core of the port (round-1 boxes)
    # each step a bounded sample: the whole --warmup W --steps K run stays within ~3 minutes
    step_s = min(args.cpu_seconds, 150.0 / max(1, args.steps + args.warmup))
    S = max(cores * 8, int(step_s * per_core * cores / (spec.n_x * nmodes)))
    S = min(S, T)
    a = T // 2
    # Table values do not change the port's operation count or memory traffic (no data-
    # dependent branches, no denormals), so the reference arm times the port on seeded
    # synthetic tables of the config's shapes instead of rebuilding q̃ with scipy (stage 1
    # is not part of the reference, whose q̃ is an input; scipy at l ~ 2000 took minutes).
    rng = np.random.default_rng(spec.seed)
    L = spec.l_max - 1
    qt = rng.standard_normal((spec.p, spec.n_x, L)) * 1e-10
    C = rng.uniform(1e-5, 5e-2, L)
    times, setup = [], []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        ref.gamma3d(hi.q, qt, C, hi.v, hi.wr2, hi.entries, 2, spec.l_max, a, a + S,
                    workers=cores, block=64)
        if i >= args.warmup:
            times.append(time.perf_counter() - t0)
    # per-call setup of the reference's worker pool (fork + teardown), measured on an empty
    # range and subtracted, as SURVEY §8(d) prescribes for the extrapolation: over a whole Γ
    # (days of CPU) it is negligible, over a bounded sample it is not
    for _ in range(3):
        t0 = time.perf_counter()
        ref.gamma3d(hi.q, qt, C, hi.v, hi.wr2, hi.entries, 2, spec.l_max, a, a,
                    workers=cores, block=64)
        setup.append(time.perf_counter() - t0)
    dt_raw = float(np.mean(times))
    t_setup = float(np.median(setup))
    dt = max(dt_raw - t_setup, 1e-9)
    rate = S * spec.n_x * nmodes / dt
    sample = (f"reference algorithm (NumPy restatement of engine3d._sweep_chunk, bit-identical "
              f"to cmbproj on config 0) over flat range [{a}, {a + S}) of config "
              f"{args.config[1:]} ({S} triples; seeded synthetic q̃/C of the config's shapes), fork "
              f"pool of {cores}, B=64, on {cpu_model()}")
    line = {
        "metric": "Γ projection: (l-triple·x·mode) FP64 updates/s", "value": rate,
        "unit": "updates/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt_raw * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, BASELINE config shapes)",
        "config": {"workload": f"separable Γ, BASELINE config {args.config[1:]} (bounded "
                               f"flat-range sample per step)", "updates_per_step": S * spec.n_x * nmodes,
                   "parallelism": f"cpu x{cores}"},
        "impl": "reference",
        "s_per_gamma_extrapolated": U / rate,
        "setup_s_per_call": t_setup, "ms_per_step_setup_corrected": dt * 1e3,
        "rate_uncorrected": S * spec.n_x * nmodes / dt_raw,
        "value_note": "value = sample updates / (mean step time - per-call pool setup measured "
                      "on an empty range), the rate a whole Γ would see",
        "cpu_baseline": {"value": rate, "unit": "updates/s", "cores": cores, "kind": "port",
                         "cpu_model": cpu_model(), "sample": sample},
        "e2e": {"value": rate, "unit": "updates/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "native_so_loaded": native_maps(),
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    elif args.config == "2d":
        run_2d(args)
    elif args.config == "c3":
        run_nonsep(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
