"""Run V(2,2) block-Jacobi cycles on the configs[1] hierarchy (1024^2, p=4, K=I) for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1705_09907_b200 import _lib
from paper_1705_09907_b200.mesh import build_cartesian
from paper_1705_09907_b200.multigrid import _native_mg, attach_smoothers, build_hierarchy
from paper_1705_09907_b200.problem import constant_problem

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
p = int(sys.argv[2]) if len(sys.argv) > 2 else 4
levels = build_hierarchy(build_cartesian(n, n), p, constant_problem(0.0, 1.0), smoother=None)
attach_smoothers(levels, "blockjacobi", 0.8)
mg = _native_mg(levels)
b = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, levels[0].ndof)).cuda()
x = torch.zeros_like(b)
st = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    _lib.check(_lib.lib.hdg_mg_cycle(mg.handle, b.data_ptr(), 0, x.data_ptr(), 2, 2, 1, 0, st))
torch.cuda.synchronize()
print("ok", [(l.mesh.n_x, l.p, l.ndof) for l in levels])
