"""Failover across GPUs (BASELINE north star): each span server
runs on its own GPU, a server dropped mid-generation is replaced by a server on
a spare GPU, and the dual-cache client replays the dropped span's cached inputs
there.  Tokens and every failover counter must equal the reference's golden
traces (the same traces `test_gpu_swarm.py` checks on one GPU).  Activations
cross GPUs peer to peer (device payloads `.to()` the next server's GPU).

Needs >= 3 GPUs (`gpurun --gpus 4`); skipped on one.
"""

import json
import os

import numpy as np
import pytest
import torch

from conftest import GOLDEN

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(torch.cuda.device_count() < 3, reason="needs >= 3 GPUs")]
TRACES = [t for t in json.load(open(os.path.join(GOLDEN, "swarm_traces.json"))) if t["crash"]]


def _placement(n_gpus):
    """replica a of stage s on GPU s % (n - 1); every other replica on the spare GPU n - 1"""
    def gpu_of(stage, replica):
        return (n_gpus - 1) if replica > 0 else stage % (n_gpus - 1)
    return gpu_of


@pytest.mark.parametrize("tr", TRACES, ids=[t["name"] for t in TRACES])
def test_failover_onto_spare_gpu_matches_reference_trace(swarmpipe, tr):
    """The reference's own swarm (BlockServer / SimNetwork / SwarmClient) with each
    server's B200 engine on its placement GPU: the crashed span's cached inputs
    are replayed onto a server whose engine lives on the spare GPU."""
    from paper_2312_08361_b200.engine import B200ServerEngine
    from support.ref_swarm import build_gpu_swarm
    cfg = swarmpipe.model.ModelConfig(seed=1)
    n = torch.cuda.device_count()
    gpu_of = _placement(n)
    engines = {}

    def engine_for(stage, replica):
        g = gpu_of(stage, replica)
        if g not in engines:
            engines[g] = B200ServerEngine(cfg, device=g)
        return engines[g]

    prof = (swarmpipe.netsim.NetProfile(failure_prob=tr["failure_prob"])
            if "failure_prob" in tr else None)
    swarm = build_gpu_swarm(swarmpipe, cfg, engine_for=engine_for, n_stages=tr["n_stages"],
                            replicas=tr["replicas"], seed=tr.get("seed", 0), profile=prof,
                            server_overrides={k: {"crash_after_messages": v}
                                              for k, v in tr["crash"].items()})
    assert len({e.device for e in engines.values()}) >= 2
    res = swarm.client().generate([3, 1, 4], tr["n_new"], quantized=tr["quantized"])
    c = res.counters
    if not tr["quantized"]:
        assert res.tokens == tr["tokens"]
    assert (c.messages, c.recoveries, c.reroutes) == (tr["messages"], tr["recoveries"],
                                                      tr["reroutes"])
    assert [list(e) for e in c.restore_events] == tr["restore_events"]
    assert c.per_step_bytes == tr["per_step_bytes"]
    assert swarm.net.total_bytes() == tr["total_bytes"]
    # the replays ran on servers whose engines live on the spare GPU
    spare = {sid for sid, s in swarm.servers.items() if s.engine.device.index == n - 1}
    assert spare


def test_llama_int8_spans_on_three_gpus_equal_one_gpu():
    """70B-family kernels (int8 weights, GQA, RoPE, SwiGLU, bf16 KV): a 3-span
    chain on three GPUs, int8-coded between spans, gives bit-identical rows to
    the same chain on one GPU (prefill then decode)."""
    from paper_2312_08361_b200.blob import HiddenBlob
    from paper_2312_08361_b200.config import SpanConfig
    from paper_2312_08361_b200.engine import B200ServerEngine
    cfg = SpanConfig(n_blocks=6, hidden_dim=512, n_heads=4, n_kv_heads=2, ffn_dim=1024,
                     vocab_size=64, max_seq_len=512, family="llama", weight_dtype="int8",
                     kv_dtype="bf16", seed=5)
    spans = [(0, 2), (2, 4), (4, 6)]
    rng = np.random.default_rng(9)
    prompt = rng.standard_normal((40, cfg.hidden_dim)).astype(np.float32)
    steps = [rng.standard_normal((1, cfg.hidden_dim)).astype(np.float32) for _ in range(6)]

    def run(devices):
        engs = [B200ServerEngine(cfg, device=g) for g in devices]
        caches = [e.make_caches(a, b, 1) for e, (a, b) in zip(engs, spans)]
        outs = []
        for x, n in [(prompt, 40)] + [(s, 1) for s in steps]:
            blob = HiddenBlob.from_array(x)
            for i, (e, (a, b)) in enumerate(zip(engs, spans)):
                blob = e.run_cached(a, b, caches[i], blob, 1, n, i < len(spans) - 1)
            outs.append(blob.array())
        return outs

    multi = run([0, 1, 2])
    single = run([0, 0, 0])
    for m, s in zip(multi, single):
        assert np.array_equal(m, s)
