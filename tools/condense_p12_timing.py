"""p = 12 local condensation: packed shared-memory kernel (hdg_condense_piecewise) against the
batched library solve it replaces.  Prints one JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1705_09907_b200.discretization import PiecewiseCondenser


def main():
    p = int(sys.argv[1]) if len(sys.argv) > 1 else 12
    E = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 15
    pc = PiecewiseCondenser(p, 1.0 / 64, 1.0 / 64, 1.0)
    rng = np.random.default_rng(2)
    k = np.exp(rng.uniform(np.log(1e-2), np.log(1e2), E))
    kx, ky = pc._kpair(k)
    out = torch.empty((E, 4 * (p + 1), 4 * (p + 1)), dtype=torch.float64, device="cuda")

    def timed(fn, reps=3):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            r = fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps, r

    t_k, S = timed(lambda: pc.blocks(k))
    t_l, S_lib = timed(lambda: pc._blocks_library(kx, ky, out))
    err = float((S - S_lib).abs().max() / S_lib.abs().max())
    print(json.dumps({"p": p, "elements": E, "packed_kernel_ms": round(t_k, 2), "library_solve_ms": round(t_l, 2),
                      "max_rel_diff": err}))


if __name__ == "__main__":
    main()
