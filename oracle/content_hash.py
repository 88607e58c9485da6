"""Device content hash of wire payloads — CPU restatement (test infrastructure).

The builder's own format (parity unpinned by the reference, which has no
device hash): SURVEY.md §8f item 4 asks for a GPU-side content hash over the
int8 codes that cross span boundaries; the reference's relay checksum is
FNV-1a 64 on the host (`SP/wire.py:39-44`, stamped / checked at
`SP/server.py:388-393, 413-426`), which `fnv1a64` below restates and which the
engine's `blob_checksum` keeps.  Definition (`csrc/hash.cu`):

    w_i = little-endian u32 of bytes [4i, 4i+4) (zero-padded), m = ceil(n/4)
    H   = (n + sum_{i<m} (w_i + 1) * r^(i+1)) mod (2^61 - 1)

Two independent formulations (power sum and Horner) are kept so the tests can
pin one against the other.
"""

from __future__ import annotations

import numpy as np

P = (1 << 61) - 1
RADIX = 0x0A3B1C5D7E9F2468 % P


def _words(data: bytes) -> np.ndarray:
    n = len(data)
    pad = (-n) % 4
    return np.frombuffer(bytes(data) + b"\0" * pad, dtype="<u4").astype(object)


def content_hash(data: bytes) -> int:
    """Power-sum form (the GPU's decomposition: any order of the terms)."""
    h = len(data) % P
    pw = RADIX
    for w in _words(data):
        h = (h + (int(w) + 1) * pw) % P
        pw = pw * RADIX % P
    return h


def content_hash_horner(data: bytes) -> int:
    """The same polynomial evaluated by Horner's rule from the last word."""
    acc = 0
    for w in reversed(list(_words(data))):
        acc = (acc + int(w) + 1) * RADIX % P
    return (acc + len(data)) % P


def fnv1a64(data: bytes) -> int:
    """`SP/wire.py:39-44`."""
    h = 0xCBF29CE484222325
    for b in data:
        h ^= b
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h
