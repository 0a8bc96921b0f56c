"""Strip decomposition on CPU: world_size 2 and 3 over gloo, the local
operator is the CPU oracle on each rank's local mesh.  Checks ownership coverage, halo
index symmetry and that the distributed apply equals the global oracle apply."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import specs
from oracle import hdg_oracle as O
from paper_1705_09907_b200.distributed import StripLayout, split_rows


def test_split_rows():
    assert split_rows(10, 3) == [(0, 4), (4, 7), (7, 10)]
    assert split_rows(16, 4, align=4) == [(0, 4), (4, 8), (8, 12), (12, 16)]
    with pytest.raises(ValueError):
        split_rows(3, 4)


@pytest.mark.parametrize("world", [2, 3, 4])
def test_ownership_and_halo_symmetry(world):
    nx, ny, p = 7, 12, 2
    Ls = [StripLayout(nx, ny, p, world, g) for g in range(world)]
    owned = np.concatenate([L.owned_pairs()[1] for L in Ls])
    assert np.array_equal(np.sort(owned), np.arange(Ls[0].ndof_g))       # each dof owned once
    for g in range(world - 1):
        a, b = Ls[g], Ls[g + 1]
        np.testing.assert_array_equal(a.local_to_global[a.send_up], b.local_to_global[b.recv_down])
        np.testing.assert_array_equal(b.local_to_global[b.send_down], a.local_to_global[a.recv_up])
        assert not a.owned[a.recv_up].any() and b.owned[b.send_down].all()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, nx, ny, p, kind, out):
    import torch
    import torch.distributed as dist
    from paper_1705_09907_b200.distributed import StripLayout, StripOperator
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    from threadpoolctl import threadpool_limits
    lim = threadpool_limits(1)  # noqa: F841  (world processes share the host: no BLAS oversubscription)
    torch.set_num_threads(1)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        L = StripLayout(nx, ny, p, world, rank)
        spec = specs.manufactured(O.Spec) if kind == "tanh" else specs.constant(O.Spec)
        dy = 1.0 / ny
        loc = O.OracleTrace(O.Grid(nx, L.nyl, 0.0, 1.0, L.lo * dy, L.hi * dy), p, spec)
        op = StripOperator(L, lambda x: torch.from_numpy(loc.matvec(x.numpy())))
        x = torch.from_numpy(np.random.default_rng(5).standard_normal(L.ndof_g))
        xl = x[torch.from_numpy(L.local_to_global)].clone()
        xl[torch.from_numpy(~L.owned)] = float("nan")           # ghosts must come from neighbours
        op.exchange(xl)
        need = np.concatenate([L.recv_down, L.recv_up]).astype(np.int64)
        assert torch.isfinite(xl[torch.from_numpy(need)]).all()
        y = op.apply(xl)
        li, gi = L.owned_pairs()
        out[rank] = (gi, y.numpy()[li], float(op.dot(xl.nan_to_num(), xl.nan_to_num())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,kind", [(2, "tanh"), (3, "const")])
def test_distributed_apply_matches_global(world, kind):
    nx, ny, p = 6, 9, 2
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(world, _free_port(), nx, ny, p, kind, out), nprocs=world, join=True)
        res = dict(out)
    spec = specs.manufactured(O.Spec) if kind == "tanh" else specs.constant(O.Spec)
    glob = O.OracleTrace(O.Grid(nx, ny), p, spec)
    x = np.random.default_rng(5).standard_normal(glob.ndof)
    ref = glob.matvec(x)
    y = np.full(glob.ndof, np.nan)
    for g in range(world):
        gi, vals, d = res[g]
        y[gi] = vals
        assert abs(d - x @ x) < 1e-10 * (x @ x)                 # owned-dof dot, all-reduced
    assert np.isfinite(y).all()
    assert np.abs(y - ref).max() <= 1e-12 * np.abs(ref).max()
