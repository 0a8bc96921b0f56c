"""MG-PCG preconditioner variants on configs[2]'s coefficient generator (log-U[1e-2,1e2] per
element, seed 2) at a reduced mesh: iterations to 1e-10 and device time per variant.
    PCG_VARIANTS="V(2,2);W(2,2);V(4,4)" python tools/pcg_variants.py 512 8
W(2,2) visits level k 2^k times: with 18 levels its latency-bound coarse tail dominates.
"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1705_09907_b200.mesh import build_cartesian
from paper_1705_09907_b200.multigrid import attach_smoothers, build_hierarchy, v_cycle, w_cycle
from paper_1705_09907_b200.problem import ProblemSpec, piecewise_coefficient


def zero(x, y):
    return np.zeros_like(np.asarray(x, float))


n, p = int(sys.argv[1]), int(sys.argv[2])
maxit = int(sys.argv[3]) if len(sys.argv) > 3 else 1500
rng = np.random.default_rng(2)
Kg = np.exp(rng.uniform(np.log(1e-2), np.log(1e2), (n, n)))
spec = ProblemSpec(piecewise_coefficient(Kg), zero, zero, 1.0)
levels = build_hierarchy(build_cartesian(n, n), p, spec, smoother="baseline")   # keeps the blocks for FSAI
b = torch.from_numpy(rng.uniform(-1.0, 1.0, levels[0].ndof)).cuda()
bn = float(b.norm())
for smoother in ("blockjacobi", "bj-chebyshev", "baseline"):
    t0 = time.time()
    attach_smoothers(levels, smoother)
    torch.cuda.synchronize()
    ts = time.time() - t0
    variants = [v for v in (("V(2,2)", v_cycle, 2), ("W(2,2)", w_cycle, 2), ("V(4,4)", v_cycle, 4))
                if v[0] in os.environ.get("PCG_VARIANTS", "V(2,2);V(4,4)").split(";")]
    for name, cyc, nu in variants:
        M = lambda r, cyc=cyc, nu=nu: cyc(levels, r, None, nu, nu)
        M(b); torch.cuda.synchronize()
        t1 = time.time()
        xs, it = levels[0].system.solve_cg(tol=1e-10, maxiter=maxit, precond=M, b=b)
        torch.cuda.synchronize()
        dt = time.time() - t1
        tr = float((b - levels[0].matvec(xs)).norm()) / bn
        print(json.dumps({"n": n, "p": p, "ndof": levels[0].ndof, "smoother": smoother, "setup_s": round(ts, 2),
                          "precond": name, "pcg_iterations": it, "solve_s": round(dt, 2),
                          "true_rel_residual": tr}), flush=True)
