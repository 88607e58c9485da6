"""The dual-cache failover path on the GPU: span servers backed by the B200
engine, the client head on the GPU, crash injection — tokens and every
failover counter must equal the reference's golden traces (SURVEY.md §0.10:
these integer counters are engine-independent)."""

import json
import os
import sys

import numpy as np
import pytest

from conftest import GOLDEN, ROOT

pytestmark = pytest.mark.gpu
TRACES = json.load(open(os.path.join(GOLDEN, "swarm_traces.json")))


def test_client_head_matches_reference(golden_toy):
    from oracle import model as om
    from paper_2312_08361_b200.config import toy
    from paper_2312_08361_b200.head import ClientHead
    head = ClientHead(toy(seed=1))
    emb = head.embedding()
    assert np.array_equal(emb, golden_toy["default__embedding"])
    assert np.array_equal(head.embed_array([3, 1, 4]), emb[[3, 1, 4]])
    rng = np.random.default_rng(0)
    for _ in range(50):
        row = rng.standard_normal((2, 64)).astype(np.float32)
        assert head.pick(row) == om.greedy_pick(om.logits_for(emb, row[-1]))


@pytest.mark.parametrize("tr", TRACES, ids=[t["name"] for t in TRACES])
def test_gpu_failover_trace(tr):
    from paper_2312_08361_b200.client import SwarmClient, build_swarm
    from paper_2312_08361_b200.config import toy
    from paper_2312_08361_b200.engine import B200ServerEngine
    from paper_2312_08361_b200.head import ClientHead
    cfg = toy(seed=1)
    eng = B200ServerEngine(cfg)
    net, servers, routes = build_swarm(lambda: eng, cfg, tr["n_stages"], tr["replicas"],
                                       crash=tr["crash"])
    res = SwarmClient("client1", cfg, net, routes, ClientHead(cfg)).generate(
        [3, 1, 4], tr["n_new"], quantized=tr["quantized"])
    c = res.counters
    assert res.tokens == tr["tokens"]
    assert (c.messages, c.recoveries, c.reroutes) == (tr["messages"], tr["recoveries"], tr["reroutes"])
    assert [list(e) for e in c.restore_events] == tr["restore_events"]
    assert c.per_step_bytes == tr["per_step_bytes"]


def _reference_importable():
    for p in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(p, "swarmpipe")):
            return p
    return None


@pytest.mark.skipif(_reference_importable() is None, reason="reference package not installed")
def test_dropin_inside_reference_block_server():
    """The engine plugged into the reference's OWN BlockServer / SimNetwork /
    SwarmClient (rebinding RealServerEngine): greedy
    tokens equal the oracle through a crash + restore."""
    sys.path.insert(0, _reference_importable())
    import swarmpipe
    import swarmpipe.server
    import swarmpipe.swarm
    from swarmpipe.model import ModelConfig, reference_generate
    from paper_2312_08361_b200.engine import B200ServerEngine
    orig = swarmpipe.swarm.RealServerEngine
    swarmpipe.swarm.RealServerEngine = B200ServerEngine
    swarmpipe.server.RealServerEngine = B200ServerEngine
    try:
        cfg = ModelConfig(seed=1)
        swarm = swarmpipe.swarm.build_sim_swarm(
            cfg, n_stages=1, replicas=2, seed=0,
            server_overrides={"s0a": {"crash_after_messages": 6}})
        assert isinstance(swarm.servers["s0a"].engine, B200ServerEngine)
        res = swarm.client().generate([3, 1, 4], 32)
        assert res.tokens == reference_generate(cfg, [3, 1, 4], 32)
        assert res.counters.recoveries == 1
        assert [tuple(e) for e in res.counters.restore_events] == [(0, 8, 7, 1792)]
        swarm = swarmpipe.swarm.build_sim_swarm(cfg, n_stages=4, replicas=2, seed=3,
                                                profile=swarmpipe.netsim.NetProfile(failure_prob=1e-2))
        res = swarm.client().generate([3, 1, 4], 64, quantized=True)
        assert len(res.tokens) == 67
    finally:
        swarmpipe.swarm.RealServerEngine = orig
        swarmpipe.server.RealServerEngine = orig


@pytest.mark.skipif(_reference_importable() is None, reason="reference package not installed")
def test_dropin_beam_search_matches_reference_oracle():
    """§8f item 2, T/test_beam.py:21-44 with the GPU engine inside the reference's
    own swarm: k = 4 beams (reorder = page-table permutation with copy-on-write
    tails) give the local beam oracle's hypotheses and scores, also through a
    crashed server, and k = 1 degenerates to greedy."""
    sys.path.insert(0, _reference_importable())
    import swarmpipe.server
    import swarmpipe.swarm
    from swarmpipe.model import ModelConfig, reference_beam, reference_generate
    from paper_2312_08361_b200.engine import B200ServerEngine
    orig = swarmpipe.swarm.RealServerEngine
    swarmpipe.swarm.RealServerEngine = B200ServerEngine
    swarmpipe.server.RealServerEngine = B200ServerEngine
    try:
        cfg = ModelConfig(seed=1)
        swarm = swarmpipe.swarm.build_sim_swarm(cfg, seed=0)
        assert swarm.client().beam_generate([4, 2], 16, k=1).tokens == \
            reference_generate(cfg, [4, 2], 16)
        want = reference_beam(cfg, [4, 2], 24, k=4)
        res = swarmpipe.swarm.build_sim_swarm(cfg, seed=0).client().beam_generate([4, 2], 24, k=4)
        assert [h for h, _ in res.beams] == [h for h, _ in want]
        for (_, sa), (_, sb) in zip(res.beams, want):
            assert sa == pytest.approx(sb, abs=1e-4)
        want = reference_beam(cfg, [4, 2], 16, k=4)
        swarm = swarmpipe.swarm.build_sim_swarm(
            cfg, seed=0, server_overrides={"s2a": {"crash_after_messages": 10}})
        res = swarm.client().beam_generate([4, 2], 16, k=4)
        assert [h for h, _ in res.beams] == [h for h, _ in want]
        assert res.counters.recoveries >= 1
    finally:
        swarmpipe.swarm.RealServerEngine = orig
        swarmpipe.server.RealServerEngine = orig


@pytest.mark.parametrize("quantized", [False, True])
def test_llama_int8_failover_greedy_tokens_match_oracle(quantized):
    """BASELINE north star on the 70B kernel family (int8 weights, GQA, RoPE,
    SwiGLU, bf16 KV): 2 stages x 2 replicas, a stage-1 server crashes
    mid-generation, the client replays its cached inputs onto the replica —
    greedy tokens equal the CPU oracle's (reference_generate restated)."""
    from oracle import model as om
    from paper_2312_08361_b200.client import SwarmClient, build_swarm
    from paper_2312_08361_b200.config import SpanConfig
    from paper_2312_08361_b200.engine import B200ServerEngine
    from paper_2312_08361_b200.head import ClientHead
    cfg = SpanConfig(n_blocks=4, hidden_dim=512, n_heads=4, n_kv_heads=2, ffn_dim=1024,
                     vocab_size=64, max_seq_len=512, family="llama", weight_dtype="int8",
                     kv_dtype="bf16", seed=5)
    eng = B200ServerEngine(cfg)
    net, servers, routes = build_swarm(lambda: eng, cfg, 2, 2, crash={"s1a": 9})
    res = SwarmClient("client1", cfg, net, routes, ClientHead(cfg)).generate(
        [3, 1, 4], 24, quantized=quantized)
    assert res.counters.recoveries >= 1 and res.counters.restore_events
    if not quantized:
        assert res.tokens == om.reference_generate(cfg, [3, 1, 4], 24)
    else:
        # stage boundary coded: the oracle applies the same codec round trip
        from oracle import codec as oc
        emb = om.init_embedding(cfg)
        r0, r1 = om.SpanRunner(cfg, 0, 2), om.SpanRunner(cfg, 2, 4)
        toks = [3, 1, 4]
        x = emb[toks]
        for _ in range(24):
            h = r0.step(x[None])[0]
            codes, scales = oc.quantize(h)
            h = oc.dequantize(codes, scales, h.shape)
            y = r1.step(h[None])[0]
            t = om.greedy_pick(om.logits_for(emb, y[-1]))
            toks.append(t)
            x = emb[[t]]
        assert res.tokens == toks
