import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
import specs
import paper_1705_09907_b200.multigrid as mg
import paper_1705_09907_b200.problem as pb
from paper_1705_09907_b200.mesh import build_cartesian
from paper_1705_09907_b200.fsai import StructuredFSAI, fsai_build
np.set_printoptions(linewidth=200, precision=4, suppress=True)
for n, p in [(2, 1), (3, 1), (3, 2)]:
    levels = mg.build_hierarchy(build_cartesian(n, n), p, specs.constant(pb.ProblemSpec), smoother=None)
    lev = levels[0]
    A = lev.operator.tocsr()
    ref = fsai_build(A, 1, 1.0, device=False)
    sm = StructuredFSAI(lev.block_op, 1.0)
    G, Gr = sm.G.toarray(), ref.G.toarray()
    print(n, p, "ndof", lev.ndof, "maxdiff", np.abs(G - Gr).max(), "lam", sm.lam_max, ref.lam_max)
    if np.abs(G - Gr).max() > 1e-10:
        bad = np.argwhere(np.abs(G - Gr) > 1e-10)
        print(bad[:20])
        r = bad[0][0]
        print("row", r, "\n ours", G[r], "\n ref ", Gr[r])
