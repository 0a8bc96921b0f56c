"""Strip-partitioned V-cycle on CPU: world 2 and 3 over gloo.  The per-window
operations are CSR restrictions of the oracle's global level operators, so this checks the
distributed orchestration (operator and residual halos, h-restriction across strips,
agglomeration of the coarse levels) against the oracle's global V-cycle."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import specs
from oracle import hdg_oracle as O
from strip_oracle import OracleWindowBackend


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, n, p, visits, out):
    import torch
    import torch.distributed as dist
    from paper_1705_09907_b200.distributed import StripLayout, StripMG, plan_strips
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    from threadpoolctl import threadpool_limits
    lim = threadpool_limits(1)  # noqa: F841  (world processes share the host: no BLAS oversubscription)
    torch.set_num_threads(1)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        levels = O.build_levels(O.Grid(n, n), p, specs.manufactured(O.Spec), smoother="blockjacobi")
        shapes = [(l.grid.n_x, l.grid.n_y, l.p, None) for l in levels]
        d, rows = plan_strips(shapes, world)
        assert d >= 1
        layouts = [StripLayout(shapes[l][0], shapes[l][1], shapes[l][2], world, rank, rows=rows[l][rank])
                   for l in range(d + 2)]
        mg = StripMG(OracleWindowBackend(levels, layouts, d), layouts, d)
        b = levels[0].rhs
        bl = torch.from_numpy(b[layouts[0].local_to_global].copy())
        x = mg.v_cycle(bl, None, 2, 2, visits)
        li, gi = layouts[0].owned_pairs()
        out[rank] = (gi, x.numpy()[li], d)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,p,visits", [(2, 16, 2, 1), (3, 24, 2, 1), (2, 16, 3, 2)])
def test_strip_vcycle_matches_global(world, n, p, visits):
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(world, _free_port(), n, p, visits, out), nprocs=world, join=True)
        res = dict(out)
    levels = O.build_levels(O.Grid(n, n), p, specs.manufactured(O.Spec), smoother="blockjacobi")
    b = levels[0].rhs
    ref = O.cycle(levels, 0, b, np.zeros_like(b), 2, 2, visits)
    x = np.full(ref.size, np.nan)
    for g in range(world):
        gi, vals, d = res[g]
        x[gi] = vals
    assert np.isfinite(x).all()
    assert np.abs(x - ref).max() <= 1e-12 * np.abs(ref).max()
