"""Summarise an ncu --set full report (raw page) into the profiles/ text format.

    python tools/ncu_summary.py gpurun_out/prof_full.ncu-rep > profiles/rNN_ncu_full_c1.txt
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
col = {h: i for i, h in enumerate(hdr)}
M = [("duration", "gpu__time_duration.sum"),
     ("DMMA pipe % (active)", "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active"),
     ("FP64 pipe % (active)", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
     ("issue %", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
     ("regs/thread", "launch__registers_per_thread"),
     ("grid", "launch__grid_size"), ("block", "launch__block_size"),
     ("DRAM read", "dram__bytes_read.sum"), ("DRAM write", "dram__bytes_write.sum"),
     ("L2 hit %", "lts__t_sector_hit_rate.pct"),
     ("smem ld bank conflicts", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum")]
stall_prefix = "smsp__average_warps_issue_stalled_"
for d in data:
    name = d[col["Kernel Name"]].split("(")[0]
    print(f"## {name}")
    for label, key in M:
        if key in col:
            print(f"  {label:24s} {d[col[key]]} {units[col[key]]}")
    st = []
    for h, i in col.items():
        if h.startswith(stall_prefix) and h.endswith("_per_issue_active.ratio"):
            try:
                st.append((float(d[i]), h[len(stall_prefix):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    st.sort(reverse=True)
    print("  top stalls (warps per issue): " + ", ".join(f"{n}={v:.2f}" for v, n in st[:7]))
