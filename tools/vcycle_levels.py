"""In-graph V(2,2) cycle time of the sub-hierarchies levels[k:] of the configs[1] hierarchy
(k = L-2 .. 0): the increments are the cost of each level's own work in a cycle."""
import json, os, sys
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
st = torch.cuda.current_stream()
out = []
for k in range(len(levels) - 2, -1, -1):
    b = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, levels[k].ndof)).cuda()
    x = torch.zeros_like(b)
    mg = _native_mg(levels[k:])
    for _ in range(3):
        _lib.check(_lib.lib.hdg_mg_cycle(mg.handle, b.data_ptr(), 0, x.data_ptr(), 2, 2, 1, 1, st.cuda_stream))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(20):
        _lib.check(_lib.lib.hdg_mg_cycle(mg.handle, b.data_ptr(), 0, x.data_ptr(), 2, 2, 1, 1, st.cuda_stream))
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    out.append({"top_level": k, "mesh_p_ndof": [levels[k].mesh.n_x, levels[k].p, levels[k].ndof],
                "cycle_ms": round(ms, 4), "this_level_ms": round(ms - (out[-1]["cycle_ms"] if out else 0.0), 4)})
    print(json.dumps(out[-1]), flush=True)
