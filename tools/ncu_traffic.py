"""DRAM bytes (read + write) and duration per kernel of an ncu --set full report, as the JSON
bench.py reads for `roofline.traffic`.

    python tools/ncu_traffic.py gpurun_out/prof_full_r02.ncu-rep > profiles/r02_ncu_traffic.json
"""
import csv
import io
import json
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv", "--print-units", "base"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, data = rows[0], rows[2:]
col = {h: i for i, h in enumerate(hdr)}


def num(d, key):
    return float(d[col[key]].replace(",", ""))


out = {}
for d in data:
    name = d[col["Kernel Name"]].split("(")[0].split("<")[0].replace("void ", "").strip()
    out[name] = {"dram_bytes": num(d, "dram__bytes_read.sum") + num(d, "dram__bytes_write.sum"),
                 "duration_ms": num(d, "gpu__time_duration.sum") / 1e6}
print(json.dumps(out, indent=1))
