"""Host/device conversion at the drop-in boundary.

The reference API takes and returns NumPy arrays.  The drop-in accepts NumPy
arrays or torch tensors; NumPy inputs are copied to the current CUDA device
(float64 stays float64 -> exact mode, float32 -> fp32 validation mode) and
results are copied back to NumPy.  torch CUDA tensors stay on the device
(bfloat16 selects the tcgen05 fast path).
"""

from __future__ import annotations

import numpy as np
import torch

from .errors import DimsError


def cuda_device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2507_01004_b200 needs a CUDA device (there is no CPU implementation)")
    return torch.device("cuda", torch.cuda.current_device())


def is_numpy(x) -> bool:
    return isinstance(x, np.ndarray) or np.isscalar(x)


def any_numpy(*xs) -> bool:
    return any(isinstance(x, np.ndarray) for x in xs if x is not None)


def to_dev(x, dtype: torch.dtype | None = None) -> torch.Tensor:
    if x is None:
        return None
    if isinstance(x, torch.Tensor):
        t = x
    elif isinstance(x, np.ndarray):
        t = torch.from_numpy(np.ascontiguousarray(x))
    else:
        raise DimsError(f"expected a numpy array or torch tensor, got {type(x).__name__}")
    if dtype is not None and t.dtype != dtype:
        t = t.to(dtype)
    if not t.is_cuda:
        t = t.to(cuda_device(), non_blocking=False)
    return t.contiguous()


def compute_dtype(x) -> torch.dtype:
    """tensor dtype the kernels run q/k/v in, from a user array."""
    if isinstance(x, np.ndarray):
        if x.dtype == np.float64:
            return torch.float64
        if x.dtype == np.float32:
            return torch.float32
        return torch.float64
    if isinstance(x, torch.Tensor):
        if x.dtype in (torch.bfloat16, torch.float32, torch.float64):
            return x.dtype
        if x.dtype == torch.float16:
            return torch.bfloat16
        return torch.float32
    raise DimsError(f"expected a numpy array or torch tensor, got {type(x).__name__}")


def acc_of(dtype: torch.dtype) -> torch.dtype:
    return torch.float64 if dtype == torch.float64 else torch.float32


def back(t: torch.Tensor, as_numpy: bool, np_dtype=None):
    if not as_numpy:
        return t
    a = t.detach().cpu()
    if a.dtype == torch.bfloat16:
        a = a.float()
    a = a.numpy()
    return a.astype(np_dtype, copy=False) if np_dtype is not None else a


def shape_of(x):
    return tuple(x.shape)
