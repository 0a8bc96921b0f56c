"""Device FSAI apply (t = G r, z = G' t; hdg_fsai.cuh) against the trace apply on the same
level: heterogeneous K (configs[2] law), CUDA events, bytes = the factor stream + vectors.
python tools/fsai_apply_bench.py n:p ..."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1705_09907_b200 import _lib
from paper_1705_09907_b200.fsai import StructuredFSAI
from paper_1705_09907_b200.mesh import build_cartesian
from paper_1705_09907_b200.problem import ProblemSpec, piecewise_coefficient
from paper_1705_09907_b200.trace import TraceSystem

HBM = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]
zero = lambda x, y: np.zeros_like(np.asarray(x, float))


def timeit(fn, R=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(R):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / R


for arg in sys.argv[1:] or ["1024:8", "1024:4"]:
    n, p = (int(v) for v in arg.split(":"))
    Kg = np.exp(np.random.default_rng(2).uniform(np.log(1e-2), np.log(1e2), (n, n)))
    s = TraceSystem(build_cartesian(n, n), p, ProblemSpec(piecewise_coefficient(Kg), zero, zero, 1.0), with_rhs=False)
    op = s.operator
    sm = StructuredFSAI(op, 1.0)
    r = torch.rand(op.ndof, dtype=torch.float64, device="cuda")
    z = torch.empty_like(r)
    st = torch.cuda.current_stream().cuda_stream
    us_fsai = timeit(lambda: _lib.check(_lib.lib.hdg_fsai_apply(op.handle, r.data_ptr(), z.data_ptr(), st)))
    us_a = timeit(lambda: _lib.check(_lib.lib.hdg_matvec(op.handle, r.data_ptr(), z.data_ptr(), st)))
    n1 = p + 1
    nh, nv = n * (n - 1), (n - 1) * n
    gbytes = 8 * (nh * n1 * 2 * n1 + nv * n1 * 6 * n1)
    alg = 2 * gbytes + 32 * op.ndof       # G read twice (G, G'), r read, t written+read, z written
    print(json.dumps({"n": n, "p": p, "fsai_apply_us": round(us_fsai, 1), "matvec_us": round(us_a, 1),
                      "G_GB": round(gbytes / 1e9, 3), "fsai_frac": round(alg / us_fsai / 1e3 / HBM, 3),
                      "matvec_frac": round((op.operator_bytes() + 16 * op.ndof) / us_a / 1e3 / HBM, 3)}), flush=True)
