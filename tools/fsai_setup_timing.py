"""FSAI setup (fsai_build, multigrid.py:123-159) host vs device row solves on a K = I level."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import torch
import specs
from paper_1705_09907_b200.fsai import fsai_build
from paper_1705_09907_b200.mesh import build_cartesian
from paper_1705_09907_b200.multigrid import build_hierarchy
from paper_1705_09907_b200.problem import ProblemSpec

n, p = int(sys.argv[1]), int(sys.argv[2])
lev = build_hierarchy(build_cartesian(n, n), p, specs.constant(ProblemSpec), smoother=None)[0]
t = time.time(); A = lev.operator.tocsr(); t_csr = time.time() - t
out = {"mesh": n, "p": p, "rows": A.shape[0], "csr_s": round(t_csr, 2)}
for power in (1, 2):
    fsai_build(A, power, device=True)            # warm-up (CUDA context, kernels)
    torch.cuda.synchronize()
    t = time.time(); fd = fsai_build(A, power, device=True); td = time.time() - t
    out[f"power{power}_device_s"] = round(td, 2)
    if A.shape[0] <= 200000:
        t = time.time(); fh = fsai_build(A, power, device=False); th = time.time() - t
        out[f"power{power}_host_s"] = round(th, 2)
        out[f"power{power}_rel_diff"] = float(np.abs(fd.G.data - fh.G.data).max() / np.abs(fh.G.data).max())
print(json.dumps(out))
