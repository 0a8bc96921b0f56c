"""Time the facet-plane trace apply (hdg_matvec_soa) next to the reference-layout kernel
(hdg_matvec): CUDA events, 200 applies over rotating (x, y) pairs larger than L2.
python tools/tune_planes.py [n:p ...]   (HDG_SOA_J overrides the segment height)"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1705_09907_b200._lib as L
from paper_1705_09907_b200.mesh import build_cartesian
from paper_1705_09907_b200.problem import constant_problem
from paper_1705_09907_b200.trace import TraceSystem

HBM = 6553.9   # GB/s, MEASURED_PEAKS.json (the driver-measured copy bandwidth)


def timed(fn, R=200):
    for k in range(20):
        fn(k)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for k in range(R):
        fn(k)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / R


cases = [tuple(int(v) for v in a.split(":")) for a in sys.argv[1:]] or [(1024, 4), (2048, 4), (1024, 2), (768, 8)]
st = torch.cuda.current_stream().cuda_stream
for n, p in cases:
    s = TraceSystem(build_cartesian(n, n), p, constant_problem(0.0, 1.0))
    op = s.operator
    h = op.handle
    NR = max(2, int(np.ceil(4 * 670e6 / (16 * s.ndof * 4))))
    NR = min(NR, 8)
    xr = [torch.rand(s.ndof, dtype=torch.float64, device="cuda") for _ in range(NR)]
    yr = [torch.empty_like(xr[0]) for _ in range(NR)]
    xs = [op.to_planes(x) for x in xr]
    ys = [torch.empty_like(xs[0]) for _ in range(NR)]
    us_ref = timed(lambda k: L.check(L.lib.hdg_matvec(h, xr[k % NR].data_ptr(), yr[k % NR].data_ptr(), st)))
    us_soa = timed(lambda k: L.check(L.lib.hdg_matvec_soa(h, xs[k % NR].data_ptr(), ys[k % NR].data_ptr(), st)))
    us_pack = timed(lambda k: L.check(L.lib.hdg_soa_pack(h, xr[k % NR].data_ptr(), xs[k % NR].data_ptr(), st)), 50)
    us_unpack = timed(lambda k: L.check(L.lib.hdg_soa_unpack(h, ys[k % NR].data_ptr(), yr[k % NR].data_ptr(), st)), 50)
    # parity vs the reference-layout kernel
    L.check(L.lib.hdg_matvec(h, xr[0].data_ptr(), yr[0].data_ptr(), st))
    L.check(L.lib.hdg_matvec_soa(h, xs[0].data_ptr(), ys[0].data_ptr(), st))
    err = float((op.from_planes(ys[0]) - yr[0]).abs().max() / yr[0].abs().max())
    alg = 16 * s.ndof
    print(json.dumps({"n": n, "p": p, "ndof": s.ndof, "J": os.environ.get("HDG_SOA_J", "auto"), "rot": NR,
                      "ref_us": round(us_ref, 2), "soa_us": round(us_soa, 2),
                      "soa_gdofs": round(s.ndof / us_soa / 1e3, 1),
                      "soa_frac": round(alg / (us_soa * 1e-6) / 1e9 / HBM, 3),
                      "ref_frac": round(alg / (us_ref * 1e-6) / 1e9 / HBM, 3),
                      "pack_us": round(us_pack, 1), "unpack_us": round(us_unpack, 1), "rel_err": err}), flush=True)
