"""hdg_dist_* (include/hdgb200.h, csrc/hdg_dist.cu): strip halo exchange and all-reduce over an NCCL
communicator created by the caller.  One GPU: a one-rank communicator; the loopback flag makes
the rank its own lower and upper neighbour, so packing, the grouped ncclSend / ncclRecv on the
stream and unpacking are exercised against the row lists of distributed.StripLayout."""

import ctypes
import glob
import os

import numpy as np
import pytest

import specs

pytestmark = pytest.mark.gpu


def _nccl():
    import torch
    cands = glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "nccl", "lib", "libnccl.so.2"))
    for path in cands + ["libnccl.so.2"]:
        try:
            return ctypes.CDLL(path, mode=ctypes.RTLD_GLOBAL)
        except OSError:
            continue
    pytest.skip("libnccl.so.2 not found")


class UniqueId(ctypes.Structure):
    _fields_ = [("internal", ctypes.c_char * 128)]


def test_halo_loopback_and_allreduce(P):
    import torch
    nccl = _nccl()
    uid = UniqueId()
    assert nccl.ncclGetUniqueId(ctypes.byref(uid)) == 0
    comm = ctypes.c_void_p()
    nccl.ncclCommInitRank.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int, UniqueId, ctypes.c_int]
    assert nccl.ncclCommInitRank(ctypes.byref(comm), 1, uid, 0) == 0
    d = ctypes.c_void_p()
    P.lib_check(P.lib.hdg_dist_init(comm, 0, 1, ctypes.byref(d)))
    nx, nyl, p = 37, 12, 3
    n1 = p + 1
    sysw = P.tr.TraceSystem(P.mesh(nx, nyl), p, specs.constant(P.pb.ProblemSpec), with_rhs=False)
    nh = nx * (nyl - 1)

    def h_row(jl):
        b = (jl - 1) * nx + np.arange(nx)
        return (b[:, None] * n1 + np.arange(n1)).ravel()

    def v_row(jl):
        b = nh + np.arange(nx - 1) * nyl + jl
        return (b[:, None] * n1 + np.arange(n1)).ravel()

    lo, r0, r1, nyg = 5, 7, 15, 64          # window rows 5..16 of a 64-row mesh, owned 7..14
    x0 = np.random.default_rng(0).standard_normal(sysw.ndof)
    st = torch.cuda.current_stream().cuda_stream
    # one rank, no loopback: no neighbours, nothing moves
    x = torch.from_numpy(x0).cuda()
    P.lib_check(P.lib.hdg_dist_halo(d, sysw.operator.handle, lo, r0, r1, nyg, 0, x.data_ptr(), st))
    np.testing.assert_array_equal(x.cpu().numpy(), x0)
    # operator halo, loopback: recv_up <- send_down, recv_down <- send_up (distributed.py: StripLayout)
    P.lib_check(P.lib.hdg_dist_halo(d, sysw.operator.handle, lo, r0, r1, nyg, 0x100, x.data_ptr(), st))
    ref = x0.copy()
    ref[h_row(r1 - lo)] = x0[h_row(r0 - lo)]
    ref[np.concatenate([h_row(r0 - 1 - lo), v_row(r0 - 1 - lo)])] = \
        x0[np.concatenate([h_row(r1 - 1 - lo), v_row(r1 - 1 - lo)])]
    np.testing.assert_array_equal(x.cpu().numpy(), ref)
    # residual halo, loopback: [v(r0-2), v(r0-1), h(r0-1)] <- [v(r1-2), v(r1-1), h(r1-1)]
    x = torch.from_numpy(x0).cuda()
    P.lib_check(P.lib.hdg_dist_halo(d, sysw.operator.handle, lo, r0, r1, nyg, 0x101, x.data_ptr(), st))
    ref = x0.copy()
    ref[np.concatenate([v_row(r0 - 2 - lo), v_row(r0 - 1 - lo), h_row(r0 - 1 - lo)])] = \
        x0[np.concatenate([v_row(r1 - 2 - lo), v_row(r1 - 1 - lo), h_row(r1 - 1 - lo)])]
    np.testing.assert_array_equal(x.cpu().numpy(), ref)
    # a window without the ghost rows is refused
    from paper_1705_09907_b200._lib import HDGError
    with pytest.raises(HDGError):
        P.lib_check(P.lib.hdg_dist_halo(d, sysw.operator.handle, lo, lo, r1, nyg, 0x100, x.data_ptr(), st))
    v = torch.tensor([1.5, -2.0], dtype=torch.float64, device="cuda")
    P.lib_check(P.lib.hdg_dist_allreduce_sum(d, v.data_ptr(), 2, st))
    torch.cuda.synchronize()
    np.testing.assert_array_equal(v.cpu().numpy(), [1.5, -2.0])
    P.lib_check(P.lib.hdg_dist_destroy(d))
    nccl.ncclCommDestroy.argtypes = [ctypes.c_void_p]
    nccl.ncclCommDestroy(comm)
