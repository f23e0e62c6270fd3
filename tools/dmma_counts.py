"""Summarise ncu DMMA instruction counts of the three contractions next to the plan's
executed-FLOP formula (mg_plan_stats):  python tools/dmma_counts.py gpurun_out/c_plain.log
gpurun_out/c_dmma_counts.csv [label]  — one DMMA.8x8x4 = 8*8*4 FMA = 512 FP64 FLOPs."""
import ast
import csv
import re
import sys
from collections import defaultdict

plain, counts = sys.argv[1], sys.argv[2]
label = sys.argv[3] if len(sys.argv) > 3 else counts
stats = ast.literal_eval(re.search(r"(\{'flops_run'.*?\})", open(plain).read()).group(1))
fam = {"k_run_contract": "flops_run", "k_x_contract": "flops_x", "k_pair_contract": "flops_pair"}
inst, ns, pipe = defaultdict(float), defaultdict(float), defaultdict(list)
for row in csv.DictReader(l for l in open(counts) if l.startswith('"')):
    k = next(f for f in fam if f in row["Kernel Name"])
    v = float(row["Metric Value"].replace(",", ""))
    if row["Metric Name"] == "sm__inst_executed_pipe_tensor_subpipe_dmma.sum":
        inst[k] += v
    elif row["Metric Name"] == "gpu__time_duration.sum":
        ns[k] += v
    elif "dmma_cycles_active" in row["Metric Name"]:
        pipe[k].append(v)
print(f"## {label}")
print(f"{'kernel':18s} {'DMMA inst':>14s} {'x512 FLOP':>12s} {'formula FLOP':>13s} {'ratio':>7s} "
      f"{'ms':>8s} {'TF/s (ncu)':>10s} {'DMMA pipe %':>11s}")
for k, f in fam.items():
    if k not in inst:
        continue
    ex = inst[k] * 512
    print(f"{k:18s} {inst[k]:14.0f} {ex:12.4e} {stats[f]:13.4e} {ex / stats[f]:7.4f} "
          f"{ns[k] / 1e6:8.2f} {stats[f] / ns[k] / 1e3:10.2f} "
          f"{sum(pipe[k]) / max(len(pipe[k]), 1):11.1f}")
