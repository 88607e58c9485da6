"""CPU stand-in for `relay.WireCheck` (test infrastructure): the same stamp /
verify / raise_if_mismatch protocol over the oracle restatement of the device
content hash (oracle/content_hash.py), so the gloo tests exercise the
pipeline's and the failover ring's checksum plumbing on CPU.  `corrupt` =
indices of stamp calls after which one payload byte is flipped (a corrupted
hop, detected by the receiver)."""

import numpy as np
import torch

from oracle.content_hash import content_hash
from paper_2312_08361_b200.errors import ProtocolError


class OracleWireCheck:
    def __init__(self, corrupt=()):
        self.corrupt = set(corrupt)
        self.stamped = 0
        self.verified = 0
        self.bad = False

    @staticmethod
    def _hash(wire, payload):
        return content_hash(wire[:payload].numpy().tobytes())

    def stamp(self, wire, payload, off):
        h = self._hash(wire, payload)
        wire[off:off + 8] = torch.from_numpy(np.frombuffer(h.to_bytes(8, "little"), np.uint8).copy())
        if self.stamped in self.corrupt:
            wire[payload // 2] ^= 0x10
        self.stamped += 1

    def verify(self, wire, payload, off):
        want = int.from_bytes(wire[off:off + 8].numpy().tobytes(), "little")
        if self._hash(wire, payload) != want:
            self.bad = True
        self.verified += 1

    def raise_if_mismatch(self):
        if self.bad:
            raise ProtocolError("desync: relay checksum mismatch")
