"""Activation blobs: the reference's ``HiddenBlob`` (`SP/wire.py:73-139`) with
an optional device-resident payload.

``HiddenBlob`` keeps the reference's fields (rows, cols, data, quant,
synthetic, quantize_flag), its ``nbytes()`` formula (byte counters must not
change, `SP/wire.py:105-111`) and its byte encoding.  A blob produced by the
B200 engine keeps its f32 rows, or its int8 codes + f32 scales, in HBM; the
host copy is made only when ``.data`` / ``.quant`` / ``.array()`` is read, so
span->span relays move device buffers and never touch the host.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np

from .errors import ProtocolError

BLOCK_SIZE = 64
_BLOB_HEADER = struct.Struct("<BII")     # encoding, rows, cols   (SP/wire.py:66)
_QUANT_HEADER = struct.Struct("<II")     # block_size, n_blocks   (SP/wire.py:67)
ENC_RAW = 0
ENC_QUANT = 1


@dataclass
class QuantizedHidden:
    """Blockwise-quantised activations (`SP/quantize.py:18-33`)."""

    shape: tuple
    block_size: int
    scales: np.ndarray
    codes: np.ndarray

    @property
    def n_blocks(self) -> int:
        return self.scales.shape[0]

    def encoded_nbytes(self) -> int:
        return 4 * self.n_blocks + self.codes.size


class HiddenBlob:
    """Activation matrix: raw f32, int8-coded, or shape-only — host or device."""

    def __init__(self, rows: int, cols: int, data=None, quant=None, synthetic: bool = False,
                 quantize_flag: bool = False, *, dev=None, dev_codes=None, dev_scales=None):
        self.rows = int(rows)
        self.cols = int(cols)
        self._data = data
        self._quant = quant
        self.synthetic = synthetic
        self.quantize_flag = quantize_flag
        self.dev = dev                   # torch f32 [rows, cols] on the GPU
        self.dev_codes = dev_codes       # torch int8 [rows*cols]
        self.dev_scales = dev_scales     # torch f32 [ceil(rows*cols/64)]

    # -- constructors (SP/wire.py:84-95) ----------------------------------------
    @classmethod
    def from_array(cls, a: np.ndarray, quantized: bool = False) -> "HiddenBlob":
        """Host rows -> blob.  Quantisation always runs on the GPU codec
        (bit-exact with SP/quantize.py:36-49); the codes stay in HBM."""
        a2 = np.ascontiguousarray(a, dtype=np.float32)
        if a2.ndim != 2:
            a2 = a2.reshape(-1, a2.shape[-1])
        if quantized:
            from . import codec
            codes, scales = codec.quantize_device(codec.to_device(a2))
            return cls(a2.shape[0], a2.shape[1], dev_codes=codes, dev_scales=scales)
        return cls(a2.shape[0], a2.shape[1], data=a2)

    @classmethod
    def shape_only(cls, rows: int, cols: int, quantized: bool = False) -> "HiddenBlob":
        return cls(rows, cols, synthetic=True, quantize_flag=quantized)

    @classmethod
    def from_device(cls, y, codes=None, scales=None) -> "HiddenBlob":
        rows, cols = int(y.shape[0]), int(y.shape[1])
        if codes is not None:
            return cls(rows, cols, dev_codes=codes, dev_scales=scales)
        return cls(rows, cols, dev=y)

    # -- views ---------------------------------------------------------------------
    @property
    def is_quantized(self) -> bool:
        return self._quant is not None or self.dev_codes is not None

    @property
    def data(self):
        if self._data is None and self.dev is not None:
            self._data = self.dev.detach().to("cpu").numpy().astype(np.float32, copy=False)
        return self._data

    @data.setter
    def data(self, v):
        self._data = v

    @property
    def quant(self):
        if self._quant is None and self.dev_codes is not None:
            self._quant = QuantizedHidden((self.rows, self.cols), BLOCK_SIZE,
                                          self.dev_scales.to("cpu").numpy(),
                                          self.dev_codes.to("cpu").numpy())
        return self._quant

    @quant.setter
    def quant(self, v):
        self._quant = v

    def array(self) -> np.ndarray:
        """Decode to f32 [rows, cols] (SP/wire.py:97-103)."""
        if self.synthetic:
            raise ProtocolError("synthetic blob carries no data")
        if self.is_quantized:
            # dequantisation runs on the GPU codec even for host-held codes
            codes, scales = self.device_codes()
            from . import codec
            return codec.dequantize_device(codes, scales, self.rows * self.cols).to(
                "cpu").numpy().reshape(self.rows, self.cols)
        return self.data

    def array_async(self, out=None) -> "PendingRows":
        """Start the device->host copy of the decoded rows without waiting for
        the stream: the copy lands in pinned memory behind the kernels already
        queued, and ``.result()`` waits for it (an extension of `array()` for
        callers that pipeline several sessions, e.g. the multi-GPU ring).
        ``out``: a pinned f32 [rows, cols] host tensor to copy into (reused
        buffers avoid a pinned allocation per call)."""
        if self.synthetic:
            raise ProtocolError("synthetic blob carries no data")
        if self.dev is None and self.dev_codes is None:
            return PendingRows(self.array(), None)
        import torch
        if self.dev is not None:
            src = self.dev
        else:
            from . import codec
            src = codec.dequantize_device(self.dev_codes, self.dev_scales, self.rows * self.cols)
        host = out if out is not None else torch.empty((self.rows, self.cols),
                                                       dtype=torch.float32, pin_memory=True)
        host.copy_(src.reshape(self.rows, self.cols), non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(src.device))
        return PendingRows(host, ev)

    def device_codes(self, device=None):
        """(codes, scales) as device tensors (uploaded if host-held)."""
        if self.dev_codes is None:
            import torch
            from . import codec
            dev = device or codec.default_device()
            q = self._quant
            self.dev_codes = torch.from_numpy(np.ascontiguousarray(q.codes, np.int8)).to(dev)
            self.dev_scales = torch.from_numpy(np.ascontiguousarray(q.scales, np.float32)).to(dev)
        return self.dev_codes, self.dev_scales

    def device_rows(self, device=None):
        """f32 [rows, cols] device tensor (uploaded if host-held); not for coded blobs."""
        if self.dev is None:
            import torch
            from . import codec
            dev = device or codec.default_device()
            self.dev = torch.from_numpy(np.ascontiguousarray(self.data, np.float32)).to(dev)
        return self.dev

    def nbytes(self) -> int:
        """Encoded payload size — the formula of SP/wire.py:105-111."""
        n = self.rows * self.cols
        if self.is_quantized or (self.synthetic and self.quantize_flag):
            n_blocks = (n + BLOCK_SIZE - 1) // BLOCK_SIZE
            return _BLOB_HEADER.size + _QUANT_HEADER.size + 4 * n_blocks + n
        return _BLOB_HEADER.size + 4 * n

    def encode(self) -> bytes:
        """Byte encoding of SP/wire.py:113-122."""
        if self.synthetic:
            raise ProtocolError("synthetic blob cannot be encoded")
        if self.is_quantized:
            q = self.quant
            return (_BLOB_HEADER.pack(ENC_QUANT, self.rows, self.cols)
                    + _QUANT_HEADER.pack(q.block_size, q.n_blocks)
                    + q.scales.astype("<f4").tobytes() + q.codes.tobytes())
        return (_BLOB_HEADER.pack(ENC_RAW, self.rows, self.cols)
                + np.ascontiguousarray(self.data, dtype="<f4").tobytes())

    def __repr__(self) -> str:
        where = "device" if (self.dev is not None or self.dev_codes is not None) else "host"
        kind = "synthetic" if self.synthetic else ("int8" if self.is_quantized else "f32")
        return f"HiddenBlob({self.rows}x{self.cols}, {kind}, {where})"


class PendingRows:
    """A device->host read in flight (`HiddenBlob.array_async`)."""

    def __init__(self, host, event):
        self._host, self._event = host, event

    def result(self) -> np.ndarray:
        if self._event is None:
            return self._host
        self._event.synchronize()
        return self._host.numpy()
