"""GPU hidden-state codec (`SP/quantize.py:36-58`) over torch device tensors,
through the C ABI (`sp_quantize_blockwise` / `sp_dequantize_blockwise`)."""

from __future__ import annotations

import numpy as np
import torch

from . import _lib

BLOCK_SIZE = 64


def default_device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("the spanpipe codec runs on the GPU only (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def to_device(a: np.ndarray, device=None) -> torch.Tensor:
    dev = device or default_device()
    t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32))
    return t.to(dev, non_blocking=False)


def _stream(t: torch.Tensor) -> int:
    return torch.cuda.current_stream(t.device).cuda_stream


def quantize_device(x: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
    """x f32 (any shape, contiguous) -> (codes int8 [n], scales f32 [ceil(n/64)])."""
    x = x.contiguous()
    n = x.numel()
    codes = torch.empty(n, dtype=torch.int8, device=x.device)
    scales = torch.empty((n + BLOCK_SIZE - 1) // BLOCK_SIZE, dtype=torch.float32, device=x.device)
    with torch.cuda.device(x.device):      # the kernel runs where the data lives
        _lib.check(_lib.load().sp_quantize_blockwise(x.data_ptr(), codes.data_ptr(),
                                                     scales.data_ptr(), n, _stream(x)))
    return codes, scales


def dequantize_device(codes: torch.Tensor, scales: torch.Tensor, n: int) -> torch.Tensor:
    out = torch.empty(n, dtype=torch.float32, device=codes.device)
    with torch.cuda.device(codes.device):
        _lib.check(_lib.load().sp_dequantize_blockwise(codes.data_ptr(), scales.data_ptr(),
                                                       out.data_ptr(), n, _stream(codes)))
    return out
