"""Stored-block (general K) trace apply across orders: heterogeneous piecewise-constant K
(configs[2] law), CUDA events over back-to-back applies on 2 rotating vectors, fraction of the
measured HBM peak on the algorithmic bytes (half-stored operator stream + x read + y written).
python tools/stored_sweep.py n:p ..."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1705_09907_b200 import _lib
from paper_1705_09907_b200.mesh import build_cartesian
from paper_1705_09907_b200.problem import ProblemSpec, piecewise_coefficient
from paper_1705_09907_b200.trace import RowChunkedOperator

HBM = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]
zero = lambda x, y: np.zeros_like(np.asarray(x, float))
for arg in sys.argv[1:] or ["2048:8", "1024:8", "2048:4"]:
    n, p = (int(v) for v in arg.split(":"))
    rng = np.random.default_rng(2)
    Kg = np.exp(rng.uniform(np.log(1e-2), np.log(1e2), (n, n)))
    t0 = time.time()
    op = RowChunkedOperator(build_cartesian(n, n), p, ProblemSpec(piecewise_coefficient(Kg), zero, zero, 1.0),
                            rows_per_chunk=256)
    setup = time.time() - t0
    xs = [torch.rand(op.ndof, dtype=torch.float64, device="cuda") for _ in range(2)]
    ys = [torch.empty_like(xs[0]) for _ in range(2)]
    st = torch.cuda.current_stream().cuda_stream
    run = lambda k: _lib.check(_lib.lib.hdg_matvec(op.handle, xs[k % 2].data_ptr(), ys[k % 2].data_ptr(), st))
    for k in range(5):
        run(k)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    R = 20
    e0.record()
    for k in range(R):
        run(k)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / R
    alg = op.operator_bytes() + 16 * op.ndof
    print(json.dumps({"n": n, "p": p, "ndof": op.ndof, "us": round(us, 1), "alg_GB": round(alg / 1e9, 3),
                      "GBs": round(alg / us / 1e3, 1), "frac": round(alg / us / 1e3 / HBM, 3),
                      "gdofs": round(op.ndof / us / 1e3, 2), "setup_s": round(setup, 1)}), flush=True)
    del op, xs, ys
    torch.cuda.empty_cache()
