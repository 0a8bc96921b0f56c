"""Host-side cost of the public matvec_free call (e2e is host-issue bound if this exceeds the kernel time)."""
import sys, time, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_1705_09907_b200.mesh import build_cartesian
from paper_1705_09907_b200.problem import constant_problem
from paper_1705_09907_b200.trace import TraceSystem
s = TraceSystem(build_cartesian(1024, 1024), 4, constant_problem(0.0, 1.0))
x = torch.rand(s.ndof, dtype=torch.float64, device="cuda")
for _ in range(20): y = s.matvec_free(x)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(100): y = s.matvec_free(x)
t_issue = time.perf_counter() - t
torch.cuda.synchronize()
t_all = time.perf_counter() - t
print(f"host issue of 100 matvec_free: {t_issue*1e3:.2f} ms; with completion {t_all*1e3:.2f} ms; per call host {t_issue*1e4:.1f} us")
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
for _ in range(100): y = s.matvec_free(x)
pr.disable(); torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("cumulative").print_stats(12)
