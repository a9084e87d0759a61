"""Device/buffer helpers: torch tensors are the only buffer type crossing the C ABI."""

from __future__ import annotations

import numpy as np
import torch


def device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2210_06160_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


_NP_TO_TORCH = {
    np.dtype(np.float32): torch.float32,
    np.dtype(np.float64): torch.float64,
    np.dtype(np.int32): torch.int32,
    np.dtype(np.int64): torch.int64,
    np.dtype(np.uint8): torch.uint8,
    np.dtype(np.bool_): torch.bool,
}


def to_device(a, dtype=None) -> torch.Tensor:
    """numpy / torch / sequence -> contiguous CUDA tensor (no copy if already there)."""
    dev = device()
    if isinstance(a, torch.Tensor):
        t = a
        if dtype is not None and t.dtype != dtype:
            t = t.to(dtype)
        if t.device != dev:
            t = t.to(dev, non_blocking=True)
        return t.contiguous()
    arr = np.asarray(a)
    if dtype is not None:
        np_dtype = {torch.float32: np.float32, torch.float64: np.float64,
                    torch.int32: np.int32, torch.int64: np.int64,
                    torch.uint8: np.uint8, torch.bool: np.bool_}[dtype]
        arr = arr.astype(np_dtype, copy=False)
    arr = np.ascontiguousarray(arr)
    return torch.from_numpy(arr).to(dev, non_blocking=False)


def to_numpy(t) -> np.ndarray:
    if isinstance(t, torch.Tensor):
        return t.detach().cpu().numpy()
    return np.asarray(t)


def empty(shape, dtype) -> torch.Tensor:
    return torch.empty(shape, dtype=dtype, device=device())


def zeros(shape, dtype) -> torch.Tensor:
    return torch.zeros(shape, dtype=dtype, device=device())
