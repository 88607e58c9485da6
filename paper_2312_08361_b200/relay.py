"""Relay checksums on the span-to-span wire of the multi-process paths.

The reference stamps relayed activations with a content checksum and the
receiving server refuses a step whose payload does not match
(`SP/server.py:388-393` check, `:413-426` stamp; `Error("desync", "relay
checksum mismatch")`).  Here the wire is a device buffer moved by NCCL, so the
stamp and the check run on the GPU in the stream (`sp_content_hash`,
`sp_content_hash_verify`; definition in `csrc/hash.cu`): no host round trip per
hop.  A mismatch sets a sticky device flag; `raise_if_mismatch()` reads it (one
device->host read) and raises `ProtocolError` with the reference's message.

Wire layout of one hop (rows x d hidden values, SP/quantize.py codes):
``[int8 codes: n][f32 scales: 4*ceil(n/64)][zero pad to 8][u64 hash]`` — the
hash trailer covers the codes and scales.
"""

from __future__ import annotations

import torch

from . import _lib
from .errors import ProtocolError

TRAILER = 8


def wire_layout(rows: int, d: int, checksum: bool = True) -> tuple[int, int, int]:
    """(payload bytes, hash offset, total bytes) of one hop's wire."""
    n = rows * d
    payload = n + 4 * ((n + 63) // 64)
    if not checksum:
        return payload, payload, payload
    off = (payload + 7) // 8 * 8
    return payload, off, off + TRAILER


def split_wire(w: torch.Tensor, rows: int, d: int):
    """(codes int8 [n], scales f32 [ceil(n/64)]) views of a wire buffer."""
    n = rows * d
    n_sc = (n + 63) // 64
    return w[:n].view(torch.int8), w[n:n + 4 * n_sc].view(torch.float32)


class WireCheck:
    """GPU relay checksum: `stamp` writes the payload hash into the trailer,
    `verify` checks a received wire against its trailer (device flag)."""

    def __init__(self, device: torch.device):
        if device.type != "cuda":
            raise ProtocolError("the relay checksum runs on the GPU (no CPU fallback)")
        self.lib = _lib.load()
        self.dev = device
        self.mismatch = torch.zeros(1, dtype=torch.int32, device=device)
        self.stamped = 0
        self.verified = 0

    def _stream(self) -> int:
        return torch.cuda.current_stream(self.dev).cuda_stream

    def stamp(self, wire: torch.Tensor, payload: int, off: int) -> None:
        _lib.check(self.lib.sp_content_hash(wire.data_ptr(), payload, wire.data_ptr() + off,
                                            self._stream()))
        self.stamped += 1

    def verify(self, wire: torch.Tensor, payload: int, off: int) -> None:
        _lib.check(self.lib.sp_content_hash_verify(wire.data_ptr(), payload,
                                                   wire.data_ptr() + off,
                                                   self.mismatch.data_ptr(), self._stream()))
        self.verified += 1

    def raise_if_mismatch(self) -> None:
        if int(self.mismatch.item()):
            raise ProtocolError("desync: relay checksum mismatch")
