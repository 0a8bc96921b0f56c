"""Run one trace-apply case a few times (for ncu): python tools/prof_case.py N P [stored] [epi]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1705_09907_b200._lib as L
from paper_1705_09907_b200.mesh import build_cartesian
from paper_1705_09907_b200.problem import constant_problem
from paper_1705_09907_b200.trace import TraceSystem

n, p = int(sys.argv[1]), int(sys.argv[2])
stored = len(sys.argv) > 3 and sys.argv[3] == "stored"
epi = sys.argv[4] if len(sys.argv) > 4 else "y"
s = TraceSystem(build_cartesian(n, n), p, constant_problem(0.0, 1.0))
if stored:
    E = n * n
    s = TraceSystem.from_blocks(build_cartesian(n, n), p, np.repeat(s.operator.S_cls, E, axis=0), np.arange(E))
h = s.operator.handle
if epi == "bj":
    s.operator.set_blockjacobi(0.8)
xs = [torch.rand(s.ndof, dtype=torch.float64, device="cuda") for _ in range(4)]
ys = [torch.empty_like(xs[0]) for _ in range(4)]
st = torch.cuda.current_stream().cuda_stream
for k in range(8):
    if epi == "y":
        L.check(L.lib.hdg_matvec(h, xs[k % 4].data_ptr(), ys[k % 4].data_ptr(), st))
    elif epi == "bj":
        L.check(L.lib.hdg_bj_sweep(h, xs[(k + 1) % 4].data_ptr(), xs[k % 4].data_ptr(), ys[k % 4].data_ptr(), st))
    else:
        L.check(L.lib.hdg_residual(h, xs[(k + 1) % 4].data_ptr(), xs[k % 4].data_ptr(), ys[k % 4].data_ptr(), None, st))
torch.cuda.synchronize()
print("ok", n, p, stored, epi)
