"""Blockwise absmax int8 hidden-state codec — CPU oracle (test infrastructure).

Restates `SP/quantize.py:36-58` (`SP/` = /root/reference/pkg/src/swarmpipe/):

* flatten row-major, zero-pad to a multiple of ``block`` (`:37-42`)
* ``scale = f32(absmax / 127)`` — a float32 IEEE division (`:44`)
* ``codes = int8(rint(x / scale))`` — f32 division, round-half-even (`:45-46`)
* a scale-0 block gives all-zero codes (`:47`)
* dequant: ``f32(code) * scale`` — one f32 rounding (`:56-57`)
"""

from __future__ import annotations

import numpy as np

BLOCK_SIZE = 64


def n_scale_blocks(n: int, block: int = BLOCK_SIZE) -> int:
    return (n + block - 1) // block


def quantize(h: np.ndarray, block: int = BLOCK_SIZE) -> tuple[np.ndarray, np.ndarray]:
    """Returns (codes int8 [n], scales f32 [ceil(n/block)])."""
    flat = np.ascontiguousarray(h, dtype=np.float32).ravel()
    n = flat.size
    nb = n_scale_blocks(n, block)
    padded = np.zeros(nb * block, np.float32)
    padded[:n] = flat
    blocks = padded.reshape(nb, block)
    absmax = np.abs(blocks).max(axis=1) if nb else np.zeros(0, np.float32)
    scales = (absmax / np.float32(127.0)).astype(np.float32)
    safe = np.where(scales > 0, scales, np.float32(1.0)).astype(np.float32)
    codes = np.rint(blocks / safe[:, None]).astype(np.int8)
    codes[scales == 0] = 0
    return codes.ravel()[:n].copy(), scales


def dequantize(codes: np.ndarray, scales: np.ndarray, shape, block: int = BLOCK_SIZE) -> np.ndarray:
    n = int(np.prod(shape))
    nb = scales.shape[0]
    padded = np.zeros(nb * block, np.int8)
    padded[:codes.size] = codes
    out = padded.reshape(nb, block).astype(np.float32) * scales[:, None]
    return out.ravel()[:n].reshape(shape).astype(np.float32)
