"""Time the hand-written condensation / Galerkin kernels against the batched library path.
python tools/setup_kernel_timing.py [n] [p]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1705_09907_b200 import discretization as D

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
p = int(sys.argv[2]) if len(sys.argv) > 2 else 8
E = n * n
pc = D.PiecewiseCondenser(p, 1.0 / n, 1.0 / n, 1.0)
K = np.exp(np.random.default_rng(2).uniform(np.log(1e-2), np.log(1e2), E))
out = {"n": n, "p": p, "elements": E}


def timed(fn, reps=2):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        r = fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps, r


t, S = timed(lambda: pc.blocks(K))
out["condense_kernel_s"] = round(t, 4)
kx, ky = pc._kpair(K)
t, S2 = timed(lambda: pc._blocks_library(kx, ky, torch.empty_like(S)), reps=1)
out["condense_library_s"] = round(t, 4)
out["condense_max_rel_diff"] = float((S - S2).abs().max() / S2.abs().max())
del S2
V = D.p_transfer_matrix(p)
t, Sc = timed(lambda: D.galerkin_p(S, V))
out["galerkin_p_kernel_s"] = round(t, 4)
Q = torch.as_tensor(np.kron(np.eye(4), V), device="cuda")
t, Sc2 = timed(lambda: Q.T @ S @ Q, reps=1)
out["galerkin_p_library_s"] = round(t, 4)
out["galerkin_p_max_rel_diff"] = float((Sc - Sc2).abs().max() / Sc2.abs().max())
print(json.dumps(out))
