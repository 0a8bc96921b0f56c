"""Run the facet-record apply a few times (for ncu): python tools/prof_planes.py N P"""
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
s = TraceSystem(build_cartesian(n, n), p, constant_problem(0.0, 1.0), with_rhs=False)
op = s.operator
xs = [op.to_planes(torch.rand(s.ndof, dtype=torch.float64, device="cuda")) for _ in range(3)]
ys = [torch.empty_like(xs[0]) for _ in range(3)]
st = torch.cuda.current_stream().cuda_stream
for k in range(8):
    L.check(L.lib.hdg_matvec_soa(op.handle, xs[k % 3].data_ptr(), ys[k % 3].data_ptr(), st))
torch.cuda.synchronize()
print("ok", n, p)
