"""BASELINE configs[3]: order sweep at ~64M trace DOFs, K = I, fp64 (meshes per SURVEY 8(d)):
trace matvec throughput + V(2,2) block-Jacobi cycle time per order.  One JSON line per p."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1705_09907_b200 import _lib
from paper_1705_09907_b200.mesh import build_cartesian
from paper_1705_09907_b200.multigrid import _native_mg, attach_smoothers, build_hierarchy
from paper_1705_09907_b200.problem import constant_problem

MESH = {1: 4096, 2: 3328, 4: 2560, 8: 1920, 12: 1536}
orders = [int(a) for a in sys.argv[1:]] or sorted(MESH)
peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                    "MEASURED_PEAKS.json")))
for p in orders:
    n = MESH[p]
    levels = build_hierarchy(build_cartesian(n, n), p, constant_problem(0.0, 1.0), smoother=None)
    attach_smoothers(levels, "blockjacobi", 0.8)
    fine = levels[0]
    h = fine.block_op.handle
    ndof = fine.ndof
    st = torch.cuda.current_stream()
    xs = [torch.rand(ndof, dtype=torch.float64, device="cuda") for _ in range(2)]
    ys = [torch.empty_like(xs[0]) for _ in range(2)]
    for k in range(10):
        _lib.check(_lib.lib.hdg_matvec(h, xs[k % 2].data_ptr(), ys[k % 2].data_ptr(), st.cuda_stream))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    R = 50
    e0.record(st)
    for k in range(R):
        _lib.check(_lib.lib.hdg_matvec(h, xs[k % 2].data_ptr(), ys[k % 2].data_ptr(), st.cuda_stream))
    e1.record(st)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / R
    nb = fine.system.n_blocks
    flops = nb * (16 * (p + 1) ** 2 - (p + 1))
    mg = _native_mg(levels)
    b, x = xs[0], ys[0]
    for _ in range(2):
        _lib.check(_lib.lib.hdg_mg_cycle(mg.handle, b.data_ptr(), 0, x.data_ptr(), 2, 2, 1, 1, st.cuda_stream))
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(5):
        _lib.check(_lib.lib.hdg_mg_cycle(mg.handle, b.data_ptr(), 0, x.data_ptr(), 2, 2, 1, 1, st.cuda_stream))
    e1.record(st)
    torch.cuda.synchronize()
    print(json.dumps({"p": p, "mesh": n, "ndof": ndof, "matvec_us": round(us, 2),
                      "GDOF_s": round(ndof / us / 1e3, 1), "GB_s_16B_per_dof": round(16 * ndof / us / 1e3, 1),
                      "hbm_frac": round(16 * ndof / us / 1e3 / peaks["hbm_gbs"], 3),
                      "fp64_TF_s_ref_formula": round(flops / us / 1e6, 2),
                      "vcycle_ms": round(e0.elapsed_time(e1) / 5, 3), "levels": len(levels)}), flush=True)
    del levels, mg, xs, ys
    torch.cuda.empty_cache()
