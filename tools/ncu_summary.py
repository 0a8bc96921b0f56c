"""Summarise an ncu report: key metrics + stall reasons by code region (staging / compute / epilogue)."""
import csv
import io
import subprocess
import sys


def run(rep, page, *extra):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv", *extra], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def num(x):
    try:
        return float(x.replace(",", ""))
    except Exception:
        return 0.0


rep = sys.argv[1]
rows = run(rep, "details")
keep = ["Duration", "DRAM Throughput", "Memory Throughput", "Issue Slots Busy", "Registers Per Thread",
        "Achieved Occupancy", "Eligible Warps Per Scheduler", "Executed Instructions", "L2 Hit Rate",
        "Grid Size", "Dynamic Shared Memory Per Block", "Theoretical Occupancy", "Warp Cycles Per Issued Instruction"]
for r in rows[1:]:
    if len(r) > 4 and r[-3] in keep:
        print(f"{r[-3]:40s} {r[-1]} {r[-2]}")
raw = run(rep, "raw")
h, v = raw[0], raw[2]
for k, x in zip(h, v):
    if k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum"):
        print(f"{k:40s} {x} {raw[1][h.index(k)]}")
src = run(rep, "source", "--print-source", "sass")
hh = src[1]
idx = {k: i for i, k in enumerate(hh)}
data = src[2:]
ops = [r[idx["Source"]] for r in data]
dfma = [i for i, s in enumerate(ops) if "DFMA" in s]
first, last = (min(dfma), max(dfma)) if dfma else (0, 0)
stalls = [k for k in hh if k.startswith("stall_") and "Not Issued" not in k]
reg = {}
for i, r in enumerate(data):
    name = "pre" if i < first else ("compute" if i <= last else "post")
    d = reg.setdefault(name, {"samples": 0, "inst": 0, **{k: 0 for k in stalls}})
    d["samples"] += num(r[idx["Warp Stall Sampling (All Samples)"]])
    d["inst"] += num(r[idx["Instructions Executed"]])
    for k in stalls:
        d[k] += num(r[idx[k]])
for name, d in reg.items():
    top = sorted(((k, d[k]) for k in stalls), key=lambda kv: -kv[1])[:5]
    print(f"{name:8s} samples={d['samples']:.0f} inst={d['inst']:.0f} top={[(k[6:], int(v)) for k, v in top]}")
