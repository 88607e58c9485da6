"""B200-native span-forward hot path of Petals / swarmpipe (arXiv 2312.08361).

Public surface (mirrors the reference engine protocol, SP/server.py:77-186):

* :class:`B200ServerEngine` — drop-in for ``RealServerEngine``
* :class:`HiddenBlob`       — ``SP/wire.py`` blob with a device-resident payload
* :mod:`.config`            — model shapes (toy / Llama / BLOOM)
* :class:`.head.ClientHead` — the client payload (embedding, tied logits, pick)
* :mod:`.codec`             — GPU hidden-state codec
* :mod:`.pipeline`          — one span per GPU, int8 codes over NCCL send/recv
* :mod:`.placement`         — the even span split of the bench / pipeline

The session, dual-cache and block-assignment layers are the reference's own
(BlockServer, SwarmClient, balancer): the engine plugs into them unchanged.
"""

from .config import SpanConfig, bloom_176b, from_reference, llama2_7b, llama2_70b, toy  # noqa: F401

__all__ = ["SpanConfig", "toy", "llama2_7b", "llama2_70b", "bloom_176b", "from_reference",
           "B200ServerEngine", "HiddenBlob"]


def __getattr__(name):
    # the engine needs the CUDA library; import it lazily so pure-host modules
    # (config, balancer) stay importable in CPU-only tooling
    if name == "B200ServerEngine":
        from .engine import B200ServerEngine
        return B200ServerEngine
    if name == "HiddenBlob":
        from .blob import HiddenBlob
        return HiddenBlob
    raise AttributeError(name)
