"""Diagnostic: MG-PCG on heterogeneous K (configs[2] generator) at a given size; prints the
recursive and the true residual per iteration and whether the preconditioner mutates its input."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1705_09907_b200.mesh import build_cartesian
from paper_1705_09907_b200.multigrid import attach_smoothers, build_hierarchy, mg_preconditioner
from paper_1705_09907_b200.problem import ProblemSpec, piecewise_coefficient


def zero(x, y):
    return np.zeros_like(np.asarray(x, float))


n, p = int(sys.argv[1]), int(sys.argv[2])
rng = np.random.default_rng(2)
Kg = np.exp(rng.uniform(np.log(1e-2), np.log(1e2), (n, n)))
levels = build_hierarchy(build_cartesian(n, n), p, ProblemSpec(piecewise_coefficient(Kg), zero, zero, 1.0), smoother=None)
attach_smoothers(levels, "blockjacobi")
A = levels[0].matvec
b = torch.from_numpy(rng.uniform(-1.0, 1.0, levels[0].ndof)).cuda()
M = mg_preconditioner(levels)
r0 = b.clone()
z = M(b)
print("precond mutates input:", bool((b != r0).any()), "z aliases b:", z.data_ptr() == b.data_ptr())
z2 = M(b)
print("precond repeatable max|dz|:", float((z2 - z).abs().max()) if z2.data_ptr() != z.data_ptr() else "same buffer")
print("symmetry <Mb,c> vs <b,Mc>:")
c = torch.from_numpy(rng.uniform(-1.0, 1.0, levels[0].ndof)).cuda()
Mb = M(b).clone(); Mc = M(c).clone()
print(float(torch.dot(Mb, c)), float(torch.dot(b, Mc)))
Ab = A(b).clone(); Ac = A(c).clone()
print("A symmetry", float(torch.dot(Ab, c)), float(torch.dot(b, Ac)))
x = torch.zeros_like(b); r = b.clone(); zz = M(r).clone(); d = zz.clone(); rz = float(torch.dot(r, zz))
bn = float(b.norm())
for it in range(40):
    ad = A(d).clone()
    al = rz / float(torch.dot(d, ad))
    x += al * d; r -= al * ad
    zz = M(r).clone(); rzn = float(torch.dot(r, zz)); d = zz + (rzn / rz) * d; rz = rzn
    tr = float((b - A(x)).norm()) / bn
    print(it, float(r.norm()) / bn, tr)
    if float(r.norm()) / bn < 1e-10:
        break
xs, iters = levels[0].system.solve_cg(tol=1e-10, maxiter=500, precond=M, b=b)
print("solve_cg iters", iters, "true", float((b - A(xs)).norm()) / bn)
