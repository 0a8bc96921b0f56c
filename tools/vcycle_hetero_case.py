"""V(2,2) block-Jacobi cycles on a heterogeneous-K hierarchy (configs[2] coefficient law) for ncu
launch lists: python tools/vcycle_hetero_case.py N P"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1705_09907_b200 import _lib
from paper_1705_09907_b200.mesh import build_cartesian
from paper_1705_09907_b200.multigrid import _native_mg, attach_smoothers, build_hierarchy
from paper_1705_09907_b200.problem import ProblemSpec, piecewise_coefficient

n, p = int(sys.argv[1]), int(sys.argv[2])
rng = np.random.default_rng(2)
Kg = np.exp(rng.uniform(np.log(1e-2), np.log(1e2), (n, n)))
zero = lambda x, y: np.zeros_like(np.asarray(x, float))
levels = build_hierarchy(build_cartesian(n, n), p, ProblemSpec(piecewise_coefficient(Kg), zero, zero, 1.0), smoother=None)
attach_smoothers(levels, "blockjacobi", 0.8)
mg = _native_mg(levels)
b = torch.from_numpy(rng.uniform(-1, 1, levels[0].ndof)).cuda()
x = torch.zeros_like(b)
st = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    _lib.check(_lib.lib.hdg_mg_cycle(mg.handle, b.data_ptr(), 0, x.data_ptr(), 2, 2, 1, 0, st))
torch.cuda.synchronize()
print("ok", [(l.mesh.n_x, l.p, l.ndof) for l in levels])
