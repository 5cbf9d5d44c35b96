"""Device-buffer plumbing: torch owns HBM allocations and streams.

Limb data is uint64 (canonical residues); the C-ABI receives raw pointers.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

_device_index = None


def device() -> torch.device:
    global _device_index
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2604_11659_b200 needs a CUDA device (B200); no CPU fallback")
    if _device_index is None:
        _device_index = torch.cuda.current_device()
    return torch.device("cuda", _device_index)


def set_device(index: int) -> None:
    global _device_index
    _device_index = index
    torch.cuda.set_device(index)


def empty(shape) -> torch.Tensor:
    return torch.empty(shape, dtype=torch.uint64, device=device())


def zeros(shape) -> torch.Tensor:
    return torch.zeros(shape, dtype=torch.uint64, device=device())


def to_dev(a, dtype=torch.uint64) -> torch.Tensor:
    """numpy (or tensor) -> contiguous device tensor (non_blocking from pinned memory)."""
    if isinstance(a, torch.Tensor):
        return a.to(device(), non_blocking=True).contiguous()
    a = np.ascontiguousarray(a)
    return torch.from_numpy(a).to(device(), non_blocking=False).contiguous()


def to_host(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy()


def ptr(t) -> ctypes.c_void_p:
    if t is None:
        return ctypes.c_void_p(0)
    return ctypes.c_void_p(t.data_ptr())


def stream() -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(device()).cuda_stream)


def sync() -> None:
    torch.cuda.current_stream(device()).synchronize()
