"""Key metrics of the first kernel in an ncu report (the format bench.py's ncu_traffic reads):
python tools/ncu_keymetrics.py REP "title line" > profiles/<name>_key_metrics.txt"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "dram__cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, u, v = rows[0], rows[1], rows[2]
print(sys.argv[2] if len(sys.argv) > 2 else sys.argv[1])
print(f"{'kernel':70s} {v[h.index('Kernel Name')][:80]}")
for k in KEYS:
    if k in h:
        i = h.index(k)
        print(f"{k:70s} {v[i]} {u[i]}")
