"""Device plumbing: torch owns device memory and streams; libhga computes."""

from __future__ import annotations

import numpy as np
import torch

from ._lib import HgaError, check, lib


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise HgaError("a CUDA device is required (this package has no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


def ptr(t: torch.Tensor | None):
    return None if t is None else t.data_ptr()


def to_device(a, dtype: torch.dtype) -> tuple[torch.Tensor, bool]:
    """(contiguous device tensor, came_from_host)."""
    dev = require_cuda()
    if isinstance(a, torch.Tensor):
        if a.is_cuda:
            t = a if a.dtype == dtype else a.to(dtype)
            return t.contiguous(), False
        return a.to(device=dev, dtype=dtype).contiguous(), True
    arr = np.ascontiguousarray(np.asarray(a))
    t = torch.from_numpy(arr)
    if t.dtype != dtype:
        t = t.to(dtype)
    if arr.nbytes >= (1 << 20):
        t = t.pin_memory()
    return t.to(dev, non_blocking=True), True


def new_flag() -> torch.Tensor:
    return torch.zeros(1, dtype=torch.int32, device=require_cuda())


def words_for(m: int) -> int:
    return (m + 31) // 32


def sm_count() -> int:
    dev = require_cuda()
    return int(lib.hga_sm_count(dev.index or 0))


__all__ = ["require_cuda", "stream_ptr", "ptr", "to_device", "new_flag", "words_for", "sm_count",
           "check", "lib", "HgaError"]
