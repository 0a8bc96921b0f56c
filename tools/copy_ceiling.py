"""Practical HBM ceiling at the bench's size: torch copy of an ndof-double vector into another,
rotating over 4 (x, y) pairs (> L2) exactly like bench.py, CUDA events, back to back.
Prints one JSON line per size: the achievable read+write rate for a 16 B/DOF stream of that
length (launch ramp and tail included), the denominator that the kernel's frac is judged
against in practice."""
import json
import sys

import torch

sizes = [int(s) for s in sys.argv[1:]] or [10475520, 41922560]
for n in sizes:
    NB = 4
    xs = [torch.rand(n, dtype=torch.float64, device="cuda") for _ in range(NB)]
    ys = [torch.empty_like(xs[0]) for _ in range(NB)]
    for k in range(20):
        ys[k % NB].copy_(xs[k % NB])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 400
    e0.record()
    for k in range(reps):
        ys[k % NB].copy_(xs[k % NB])
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / reps
    print(json.dumps({"ndof": n, "copy_us": us, "gbs": 16 * n / us / 1e3}), flush=True)
