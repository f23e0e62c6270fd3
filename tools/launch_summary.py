"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel, next to
the live kernel shares bench.py measured with CUDA events.

    python tools/launch_summary.py gpurun_out/launches.csv gpurun_out/bench.json "<cmd>"
"""
import collections
import csv
import json
import sys

path, bench, cmd = sys.argv[1], sys.argv[2], sys.argv[3]
lines = [ln for ln in open(path) if ln.startswith('"')]
tot = collections.OrderedDict()
cnt = collections.Counter()
for r in csv.DictReader(lines):
    if r["Metric Name"] != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"].split("(")[0].split("<")[0].replace("void ", "").split("::")[-1]
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}.get(
        r["Metric Unit"], 1e-6)
    tot[name] = tot.get(name, 0.0) + float(r["Metric Value"].replace(",", "")) * scale
    cnt[name] += 1
live = json.load(open(bench))["roofline"]["kernel_share"]
fam = {"k_run_contract": "run", "k_x_contract_p": "x", "k_x_contract_ns": "x", "k_pair_contract": "pair",
       "k_gather": "gather", "k_final": "final"}
S = sum(tot.values())
print(f"# ncu launch list: {cmd}")
print("# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised "
      "per-launch times: compare SHARES with bench.py's live kernel_share, right column)")
print(f"{'kernel':34s} {'launches':>9s} {'total_ms':>10s} {'ncu share':>10s} {'live share':>10s}")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    ls = f"{live[fam[k]] * 100:9.2f}%" if k in fam else ""
    print(f"{k:34s} {cnt[k]:9d} {v:10.3f} {v / S * 100:9.2f}% {ls:>10s}")
