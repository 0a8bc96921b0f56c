"""Device-array plumbing (torch is used only for allocation, copies and streams).

Entry points accept numpy arrays (copied host->device, result copied back, as a
reference caller expects) or CUDA float64 torch tensors (zero-copy)."""

from __future__ import annotations

import numpy as np
import torch


def require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1705_09907_b200 needs a CUDA device (B200); there is no CPU path")


def to_device(x, n=None):
    """-> (contiguous cuda float64 tensor, was_numpy)."""
    if isinstance(x, torch.Tensor):
        if not x.is_cuda:
            return x.to(device="cuda", dtype=torch.float64).contiguous(), True
        if x.dtype != torch.float64:
            x = x.to(torch.float64)
        return x.contiguous(), False
    require_cuda()
    arr = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    t = torch.from_numpy(arr).to("cuda", non_blocking=False)
    return t, True


def back(t, was_numpy):
    return t.cpu().numpy() if was_numpy else t


def ptr(t):
    return 0 if t is None else t.data_ptr()


try:
    _raw_stream = torch._C._cuda_getCurrentRawStream   # C call: the per-apply host cost matters (e2e)
except AttributeError:                                  # pragma: no cover
    _raw_stream = None


def stream():
    if _raw_stream is not None:
        return _raw_stream(torch._C._cuda_getDevice())
    return torch.cuda.current_stream().cuda_stream


def empty(n):
    return torch.empty(int(n), dtype=torch.float64, device="cuda")


def zeros(n):
    return torch.zeros(int(n), dtype=torch.float64, device="cuda")


def cuda_available():
    return torch.cuda.is_available()
