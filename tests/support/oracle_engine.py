"""TEST-ONLY: engine / client head backed by the CPU oracle, used to check the
host-side mirror (server/client/router/balancer) against the reference's
golden traces on machines without a GPU.  Never imported by product code."""

from __future__ import annotations

import numpy as np
import torch

from oracle import codec as oc
from oracle import model as om


class OracleEngine:
    """The engine protocol of SP/server.py:77-142 over oracle.model."""

    def __init__(self, cfg):
        self.config = cfg
        self.blocks = {b: om.init_block(cfg, b) for b in range(cfg.n_blocks)}
        self.tables = om.Tables(cfg)

    def make_caches(self, start, end, width):
        return [om.KVCache(self.config, width) for _ in range(start, end)]

    def cache_length(self, caches):
        lengths = {c.length for c in caches}
        assert len(lengths) == 1
        return lengths.pop()

    def run_cached(self, start, end, caches, blob, width, n_new, quantized):
        from paper_2312_08361_b200.blob import HiddenBlob
        x = blob.array().reshape(width, n_new, self.config.hidden_dim)
        for b, c in zip(range(start, end), caches):
            x, kn, vn = om.block_forward_batched(self.config, self.blocks[b], x, c.keys, c.values,
                                                 self.tables)
            c.append(kn, vn)
        return HiddenBlob.from_array(x.reshape(width * n_new, -1), quantized)

    def reorder(self, caches, parents0):
        for c in caches:
            c.gather(parents0)

    def blob_checksum(self, blob):
        return 0


class OracleHead:
    def __init__(self, cfg):
        self.emb = om.init_embedding(cfg)

    def embed_array(self, tokens):
        return self.emb[np.asarray(tokens, dtype=np.intp)].copy()

    def pick(self, rows):
        return om.greedy_pick(om.logits_for(self.emb, np.asarray(rows)[-1]))


def install_host_codec(monkeypatch):
    """Route the blob codec through the oracle codec on CPU tensors (test only)."""
    from paper_2312_08361_b200 import codec

    def to_device(a, device=None):
        return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32))

    def quantize_device(x):
        c, s = oc.quantize(x.numpy())
        return torch.from_numpy(c), torch.from_numpy(s)

    def dequantize_device(codes, scales, n):
        return torch.from_numpy(oc.dequantize(codes.numpy(), scales.numpy(), (n,)))

    monkeypatch.setattr(codec, "to_device", to_device)
    monkeypatch.setattr(codec, "quantize_device", quantize_device)
    monkeypatch.setattr(codec, "dequantize_device", dequantize_device)
    monkeypatch.setattr(codec, "default_device", lambda: torch.device("cpu"))
