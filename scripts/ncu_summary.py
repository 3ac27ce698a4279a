"""Key counters of one kernel from an ncu report (raw page): time, DRAM bytes / throughput,
tensor-pipe and issue utilisation, stall reasons.   python scripts/ncu_summary.py rep.ncu-rep [title]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
title = sys.argv[2] if len(sys.argv) > 2 else rep
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, units, v = rows[0], rows[1], rows[2]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_op_imma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_uma.avg.pct_of_peak_sustained_active",
        "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "lts__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed"]
print(title)
idx = {k: i for i, k in enumerate(h)}
for k in want:
    if k in idx:
        print(f"  {k:70s} {units[idx[k]]:>10s} {v[idx[k]]}")
tc = [k for k in h if ("tcgen05" in k or "pipe_tc" in k or "utc" in k.lower()) and "pct" in k]
for k in tc[:8]:
    if k not in want:
        print(f"  {k:70s} {units[idx[k]]:>10s} {v[idx[k]]}")
print("  stall reasons (warps per issue-active cycle):")
for k, x in zip(h, v):
    if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("per_issue_active.ratio"):
        try:
            if float(x) > 0.1:
                print(f"    {k[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]:28s} {float(x):.3f}")
        except ValueError:
            pass
