"""Time the shared-block matvec for one (n, p) with a given library (HDGB200_LIB env)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1705_09907_b200 import _lib
from paper_1705_09907_b200.mesh import build_cartesian
from paper_1705_09907_b200.problem import constant_problem
from paper_1705_09907_b200.trace import TraceSystem
n, p = int(sys.argv[1]), int(sys.argv[2])
s = TraceSystem(build_cartesian(n, n), p, constant_problem(0.0, 1.0))
h = s.operator.handle
xs = [torch.rand(s.ndof, dtype=torch.float64, device="cuda") for _ in range(2)]
ys = [torch.empty_like(xs[0]) for _ in range(2)]
st = torch.cuda.current_stream()
for k in range(5):
    _lib.check(_lib.lib.hdg_matvec(h, xs[k % 2].data_ptr(), ys[k % 2].data_ptr(), st.cuda_stream))
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for k in range(20):
    _lib.check(_lib.lib.hdg_matvec(h, xs[k % 2].data_ptr(), ys[k % 2].data_ptr(), st.cuda_stream))
e1.record(st)
torch.cuda.synchronize()
print(json.dumps({"lib": os.path.basename(os.environ.get("HDGB200_LIB", "main")), "n": n, "p": p,
                  "us": round(e0.elapsed_time(e1) * 1e3 / 20, 2)}))
