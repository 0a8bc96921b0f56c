"""V(2,2) block-Jacobi cycle on a K = I hierarchy: reference layout vs facet records
(hdg_mg_set_records), zero and nonzero initial guess.  python tools/vcycle_records.py [n] [p] [ncu]"""
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

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
p = int(sys.argv[2]) if len(sys.argv) > 2 else 4
ncu = len(sys.argv) > 3
levels = build_hierarchy(build_cartesian(n, n), p, constant_problem(0.0, 1.0), smoother=None)
attach_smoothers(levels, "blockjacobi", 0.8)
mg = _native_mg(levels)
b = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, levels[0].ndof)).cuda()
x = torch.zeros_like(b)
st = torch.cuda.current_stream()
L = _lib.lib
if ncu:
    _lib.check(L.hdg_mg_set_records(mg.handle, 2))
    for _ in range(2):
        _lib.check(L.hdg_mg_cycle(mg.handle, b.data_ptr(), 0, x.data_ptr(), 2, 2, 1, 0, st.cuda_stream))
    torch.cuda.synchronize()
    sys.exit(0)
out = {"n": n, "p": p, "ndof": levels[0].ndof, "levels": len(levels)}
for mode in (0, 2, 3):
    _lib.check(L.hdg_mg_set_records(mg.handle, mode))
    for x0 in (0, x.data_ptr()):
        for _ in range(3):
            _lib.check(L.hdg_mg_cycle(mg.handle, b.data_ptr(), x0, x.data_ptr(), 2, 2, 1, 1, st.cuda_stream))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(20):
            _lib.check(L.hdg_mg_cycle(mg.handle, b.data_ptr(), x0, x.data_ptr(), 2, 2, 1, 1, st.cuda_stream))
        e1.record(st)
        torch.cuda.synchronize()
        out[f"mode{mode}_{'x0' if x0 else 'zero'}_ms"] = round(e0.elapsed_time(e1) / 20, 4)
    out[f"mode{mode}_record_levels"] = int(L.hdg_mg_record_levels(mg.handle))
# record-resident vectors (hdg_mg_cycle_records): no pack / unpack
_lib.check(L.hdg_mg_set_records(mg.handle, 2))
sysf = levels[0].system
bp = sysf.facet_planes(b).data
xp = torch.zeros_like(bp)
for x0 in (0, xp.data_ptr()):
    for _ in range(3):
        _lib.check(L.hdg_mg_cycle_records(mg.handle, bp.data_ptr(), x0, xp.data_ptr(), 2, 2, 1, 1, st.cuda_stream))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(20):
        _lib.check(L.hdg_mg_cycle_records(mg.handle, bp.data_ptr(), x0, xp.data_ptr(), 2, 2, 1, 1, st.cuda_stream))
    e1.record(st)
    torch.cuda.synchronize()
    out[f"records_{'x0' if x0 else 'zero'}_ms"] = round(e0.elapsed_time(e1) / 20, 4)
for name, fn in (("pack_us", lambda: sysf.operator.to_planes(b, out=bp)), ("unpack_us", lambda: sysf.operator.from_planes(bp, out=x))):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(20):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    out[name] = round(e0.elapsed_time(e1) / 20 * 1e3, 1)
print(json.dumps(out))
