"""Top SASS instructions of an ncu report by warp-stall samples: python tools/ncu_top.py REP [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hh = rows[1]
idx = {k: i for i, k in enumerate(hh)}
data = rows[2:]


def num(x):
    try:
        return float(x.replace(",", ""))
    except Exception:
        return 0.0


stalls = [k for k in hh if k.startswith("stall_") and "Not Issued" not in k]
tot = sum(num(r[idx["Warp Stall Sampling (All Samples)"]]) for r in data)
ranked = sorted(range(len(data)), key=lambda i: -num(data[i][idx["Warp Stall Sampling (All Samples)"]]))
for i in ranked[:n]:
    r = data[i]
    s = num(r[idx["Warp Stall Sampling (All Samples)"]])
    top = sorted(((k[6:], num(r[idx[k]])) for k in stalls), key=lambda kv: -kv[1])[:3]
    print(f"{i:5d} {100 * s / tot:5.1f}% {r[idx['Source']][:60]:60s} {top}")
