"""BASELINE configs[2] (and scaled variants): heterogeneous piecewise-constant isotropic K,
log-uniform in [1e-2, 1e2] (seed 2), fp64; MG-preconditioned CG to relative
residual 1e-10 with b ~ U[-1, 1] (same generator, after K).  Prints one JSON line.

    python tools/run_config.py --n 2048 --p 8        # full configs[2]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1705_09907_b200 import _lib
from paper_1705_09907_b200.mesh import build_cartesian
from paper_1705_09907_b200.multigrid import _native_mg, attach_smoothers, build_hierarchy
from paper_1705_09907_b200.problem import ProblemSpec, piecewise_coefficient


def zero(x, y):
    return np.zeros_like(np.asarray(x, float))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=2048)
    ap.add_argument("--p", type=int, default=8)
    ap.add_argument("--tol", type=float, default=1e-10)
    ap.add_argument("--maxiter", type=int, default=500)
    ap.add_argument("--smoother", default="baseline", help="baseline (the reference FSAI, device setup) | blockjacobi")
    ap.add_argument("--nu", type=int, default=2, help="pre- and post-smoothing sweeps")
    ap.add_argument("--hist", default=None, help="write the PCG residual history here")
    ap.add_argument("--true-residual", action="store_true",
                    help="after the reference stopping test (recursive residual, trace.py:153) passes, recompute "
                         "b - A x and restart PCG from x while the TRUE residual is above tol (at most 3 restarts)")
    a = ap.parse_args()
    rng = np.random.default_rng(2)
    Kg = np.exp(rng.uniform(np.log(1e-2), np.log(1e2), (a.n, a.n)))
    spec = ProblemSpec(piecewise_coefficient(Kg), zero, zero, 1.0)
    t0 = time.time()
    # the smoother is attached while the hierarchy is built: the device FSAI of each level is set
    # up from its element blocks before the large levels release them
    levels = build_hierarchy(build_cartesian(a.n, a.n), a.p, spec, smoother=a.smoother)
    mg = _native_mg(levels)
    torch.cuda.synchronize()
    t_setup = time.time() - t0
    fsai_s = sum(getattr(lev.smoother, "setup_s", 0.0) for lev in levels[:-1])
    ndof = levels[0].ndof
    b = torch.from_numpy(rng.uniform(-1.0, 1.0, ndof)).cuda()
    free, total = torch.cuda.mem_get_info()
    # V-cycle time (graph replay)
    x = torch.zeros_like(b)
    st = torch.cuda.current_stream()
    for _ in range(2):
        _lib.check(_lib.lib.hdg_mg_cycle(mg.handle, b.data_ptr(), 0, x.data_ptr(), a.nu, a.nu, 1, 1, st.cuda_stream))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    R = 5
    e0.record(st)
    for _ in range(R):
        _lib.check(_lib.lib.hdg_mg_cycle(mg.handle, b.data_ptr(), 0, x.data_ptr(), a.nu, a.nu, 1, 1, st.cuda_stream))
    e1.record(st)
    torch.cuda.synchronize()
    vms = e0.elapsed_time(e1) / R
    # MG-PCG solve (trace.py:142-163 with mg_preconditioner, multigrid.py:457-463)
    from paper_1705_09907_b200.multigrid import mg_preconditioner
    torch.cuda.synchronize()
    t1 = time.time()
    xs, iters = levels[0].system.solve_cg(tol=a.tol, maxiter=a.maxiter, precond=mg_preconditioner(levels, a.nu, a.nu), b=b)
    torch.cuda.synchronize()
    t_solve = time.time() - t1
    r = b - levels[0].matvec(xs)
    relres = float(torch.linalg.vector_norm(r) / torch.linalg.vector_norm(b))
    first_relres, restarts, restart_iters = relres, 0, 0
    first_hist = getattr(levels[0].system, "cg_residuals", None)
    while a.true_residual and relres > a.tol and restarts < 3:
        del r
        # restart: hdg_pcg with x0 recomputes r = b - A x0, so its stopping test starts from the true residual
        xs, it2 = levels[0].system.solve_cg(tol=a.tol, maxiter=a.maxiter, precond=mg_preconditioner(levels, a.nu, a.nu),
                                            b=b, x0=xs)
        torch.cuda.synchronize()
        restarts, restart_iters = restarts + 1, restart_iters + it2
        r = b - levels[0].matvec(xs)
        relres = float(torch.linalg.vector_norm(r) / torch.linalg.vector_norm(b))
    t_total = time.time() - t1
    if first_hist is not None:
        levels[0].system.cg_residuals = first_hist
    hist = getattr(levels[0].system, "cg_residuals", None)
    if a.hist and hist is not None:
        np.savetxt(a.hist, np.asarray(hist) / float(torch.linalg.vector_norm(b)), header="||r_k|| / ||b||, k = 0..iters")
    print(json.dumps({"config": f"{a.n}^2 p={a.p} heterogeneous K log-U[1e-2,1e2] seed 2, MG-PCG ({a.smoother} V({a.nu},{a.nu}))",
                      "ndof": ndof, "levels": len(levels), "setup_s": round(t_setup, 2),
                      "fsai_setup_s": round(fsai_s, 2),
                      "vcycle_ms": round(vms, 3), "pcg_iterations": iters, "solve_s": round(t_solve, 3),
                      "final_rel_residual": relres, "true_residual_restarts": restarts,
                      "restart_iterations": restart_iters, "rel_residual_at_reference_stop": first_relres,
                      "solve_with_restarts_s": round(t_total, 3), "gpu_mem_used_GB": round((total - free) / 1e9, 1),
                      "torch_reserved_GB": round(torch.cuda.memory_reserved() / 1e9, 1),
                      "operator_stream_GB": round(sum(lev.block_op.operator_bytes() for lev in levels) / 1e9, 1)}))


if __name__ == "__main__":
    main()
