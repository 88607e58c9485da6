"""TEST-ONLY: the engine protocol of SP/server.py:77-142 over the oracle
restatement (oracle/model.py), returning the reference's own HiddenBlob.  Run
inside the reference's BlockServer it reproduces the reference's golden failover
traces, which pins the oracle engine before the GPU engine is compared with it.
Never imported by product code."""

from __future__ import annotations

from oracle import model as om


class OracleEngine:
    def __init__(self, cfg, blocks=None):
        import swarmpipe.wire as wire
        self._blob = wire.HiddenBlob
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
        x = blob.array().reshape(width, n_new, self.config.hidden_dim)
        for b, c in zip(range(start, end), caches):
            x, kn, vn = om.block_forward_batched(self.config, self.blocks[b], x, c.keys, c.values,
                                                 self.tables)
            c.append(kn, vn)
        return self._blob.from_array(x.reshape(width * n_new, -1), quantized)

    def reorder(self, caches, parents0):
        for c in caches:
            c.gather(parents0)

    def blob_checksum(self, blob):
        return 0
