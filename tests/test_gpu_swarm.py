"""The B200 engine inside the reference's OWN host layer on the GPU: the
reference's BlockServer / SimNetwork / DirectoryBoard / SwarmClient (installed
unmodified in baseline/_ref) with `B200ServerEngine` as every server's payload
engine and the GPU client head as the client's (SURVEY.md §7 step 2 swap recipe,
tests/support/ref_swarm.py).

Pinned: tokens and every failover counter (messages, recoveries, reroutes,
restore_events, per-step bytes, virtual elapsed time, total bytes on the wire)
equal the traces the reference itself produced (tests/golden/make_golden.py);
SURVEY.md §0.10: these are engine-independent, so a drop-in must reproduce them
exactly."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu
TRACES = json.load(open(os.path.join(GOLDEN, "swarm_traces.json")))


def _swarm(swarmpipe, tr, model=None):
    from support.ref_swarm import build_gpu_swarm
    prof = (swarmpipe.netsim.NetProfile(failure_prob=tr["failure_prob"])
            if "failure_prob" in tr else None)
    return build_gpu_swarm(swarmpipe, model or swarmpipe.model.ModelConfig(seed=1),
                           n_stages=tr["n_stages"], replicas=tr["replicas"],
                           seed=tr.get("seed", 0), profile=prof,
                           server_overrides={k: {"crash_after_messages": v}
                                             for k, v in tr["crash"].items()})


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
    rows = rng.standard_normal((5, 64)).astype(np.float32)
    got = head.logits(rows)
    want = rows @ emb.T
    err = np.abs(got - want).max()
    print(f"head logits max-abs err {err:.3g}")
    assert err <= 1e-5
    # sampling: GPU logits, the reference's float64 draw -> same tokens for one rng stream
    from paper_2312_08361_b200.head import sample_pick
    r1, r2 = np.random.default_rng(7), np.random.default_rng(7)
    for _ in range(20):
        row = rng.standard_normal((1, 64)).astype(np.float32)
        assert head.pick(row, "sample", r1, 5) == sample_pick(row[0] @ emb.T, r2, 5)


@pytest.mark.parametrize("tr", TRACES, ids=[t["name"] for t in TRACES])
def test_failover_trace_inside_reference_swarm(swarmpipe, tr):
    from paper_2312_08361_b200.engine import B200ServerEngine
    swarm = _swarm(swarmpipe, tr)
    assert all(isinstance(s.engine, B200ServerEngine) for s in swarm.servers.values())
    res = swarm.client().generate([3, 1, 4], tr["n_new"], quantized=tr["quantized"])
    c = res.counters
    assert (c.messages, c.recoveries, c.reroutes) == (tr["messages"], tr["recoveries"],
                                                      tr["reroutes"])
    assert [list(e) for e in c.restore_events] == tr["restore_events"]
    assert c.step_activation_bytes == tr["step_activation_bytes"]
    assert c.per_step_bytes == tr["per_step_bytes"]
    assert res.elapsed_s == tr["elapsed_s"]
    assert swarm.net.total_bytes() == tr["total_bytes"]
    agree = np.mean(np.array(res.tokens) == np.array(tr["tokens"]))
    print(f"{tr['name']}: tokens agree {agree:.3f}, oracle tokens {tr['tokens'] == tr['oracle']}")
    if not tr["quantized"]:
        assert res.tokens == tr["tokens"] == tr["oracle"]
    else:
        # int8-coded stage boundaries: the reference's own tokens (codec bit-exact,
        # block outputs within 1e-5; T/test_acceptance.py:358-371 allows >= 95 %)
        assert agree >= 0.95


def test_dropin_c1_crash_and_restore(swarmpipe):
    """one stage x 2 replicas, s0a crashes after 6
    messages; tokens == the oracle, one recovery, restore of t = 7 rows."""
    from swarmpipe.model import ModelConfig, reference_generate
    from support.ref_swarm import build_gpu_swarm
    cfg = ModelConfig(seed=1)
    swarm = build_gpu_swarm(swarmpipe, cfg, n_stages=1, replicas=2, seed=0,
                            server_overrides={"s0a": {"crash_after_messages": 6}})
    res = swarm.client().generate([3, 1, 4], 32)
    assert res.tokens == reference_generate(cfg, [3, 1, 4], 32)
    assert res.counters.recoveries == 1
    assert [tuple(e) for e in res.counters.restore_events] == [(0, 8, 7, 1792)]


def test_dropin_other_strategies(swarmpipe):
    """T/test_client.py:24-28: RESTART and CACHELESS generation through the GPU
    engine equal the oracle too."""
    from swarmpipe.client import Strategy
    from swarmpipe.model import ModelConfig, reference_generate
    from support.ref_swarm import build_gpu_swarm
    cfg = ModelConfig(seed=1)
    want = reference_generate(cfg, [5, 9], 12)
    for strat in (Strategy.RESTART, Strategy.CACHELESS):
        swarm = build_gpu_swarm(swarmpipe, cfg, n_stages=2, replicas=2, seed=1)
        assert swarm.client().generate([5, 9], 12, strategy=strat).tokens == want


def test_dropin_beam_search_matches_reference_oracle(swarmpipe):
    """§8f item 2, T/test_beam.py:21-44 inside the reference's swarm: k = 4 beams
    (reorder = page-table permutation with copy-on-write tails, logits on the
    GPU head) give the local beam oracle's hypotheses and scores, also through a
    crashed server, and k = 1 degenerates to greedy."""
    from swarmpipe.model import ModelConfig, reference_beam, reference_generate
    from support.ref_swarm import build_gpu_swarm
    cfg = ModelConfig(seed=1)
    assert build_gpu_swarm(swarmpipe, cfg, seed=0).client().beam_generate(
        [4, 2], 16, k=1).tokens == reference_generate(cfg, [4, 2], 16)
    want = reference_beam(cfg, [4, 2], 24, k=4)
    res = build_gpu_swarm(swarmpipe, cfg, seed=0).client().beam_generate([4, 2], 24, k=4)
    assert [h for h, _ in res.beams] == [h for h, _ in want]
    for (_, sa), (_, sb) in zip(res.beams, want):
        assert sa == pytest.approx(sb, abs=1e-4)
    want = reference_beam(cfg, [4, 2], 16, k=4)
    swarm = build_gpu_swarm(swarmpipe, cfg, seed=0,
                            server_overrides={"s2a": {"crash_after_messages": 10}})
    res = swarm.client().beam_generate([4, 2], 16, k=4)
    assert [h for h, _ in res.beams] == [h for h, _ in want]
    assert res.counters.recoveries >= 1


def test_gpu_beam_select_matches_reference(swarmpipe):
    """§8f item 2: beam_select (SP/model.py:470-491) on the GPU — float64
    log-softmax, candidate ranking by (score desc, parent asc, token asc) — gives
    the reference's parents and tokens, scores to 1e-12, also with exact ties."""
    from swarmpipe.model import beam_select as ref_select
    from paper_2312_08361_b200.head import beam_select
    rng = np.random.default_rng(3)
    for w, vocab, k in ((1, 256, 4), (4, 32000, 4), (3, 1000, 16), (8, 250, 8)):
        logits = (rng.standard_normal((w, vocab)) * 3).astype(np.float32)
        scores = rng.standard_normal(w) * 2
        p, t, s = beam_select(scores, logits, k)
        rp, rt, rs = ref_select(scores, logits, k)
        assert p == list(rp) and t == list(rt)
        assert np.allclose(s, rs, rtol=0, atol=1e-12)
    # ties: equal scores and repeated logits -> parent asc, then token asc
    logits = np.tile(np.round(rng.standard_normal((1, 64)), 0).astype(np.float32), (4, 1))
    scores = np.zeros(4)
    p, t, s = beam_select(scores, logits, 12)
    rp, rt, rs = ref_select(scores, logits, 12)
    assert p == list(rp) and t == list(rt)


def test_dropin_beam_search_with_gpu_beam_select(swarmpipe, monkeypatch):
    """The reference's own SwarmClient.beam_generate with its selection step
    swapped for the GPU one (and the GPU engine / head): hypotheses and scores of
    the local beam oracle (T/test_beam.py:21-44)."""
    import swarmpipe.client as rc
    from swarmpipe.model import ModelConfig, reference_beam
    from paper_2312_08361_b200.head import beam_select
    from support.ref_swarm import build_gpu_swarm
    cfg = ModelConfig(seed=1)
    want = reference_beam(cfg, [4, 2], 20, k=4)        # the oracle, before the swap
    monkeypatch.setattr(rc.M, "beam_select", beam_select)
    res = build_gpu_swarm(swarmpipe, cfg, seed=0).client().beam_generate([4, 2], 20, k=4)
    assert [h for h, _ in res.beams] == [h for h, _ in want]
    for (_, sa), (_, sb) in zip(res.beams, want):
        assert sa == pytest.approx(sb, abs=1e-4)


@pytest.mark.parametrize("quantized", [False, True])
def test_llama_int8_failover_greedy_tokens_match_oracle(swarmpipe, quantized):
    """The 70B kernel family (int8 weights, GQA, RoPE, SwiGLU, bf16 KV) at a small
    width, inside the reference's swarm: 2 stages x 2 replicas, s1a crashes
    mid-generation, the reference client replays its cached inputs onto s1b —
    greedy tokens equal the CPU oracle's (the same codec round trip at the coded
    stage boundary when quantized, SP/client.py:280-287)."""
    from oracle import codec as oc
    from oracle import model as om
    from paper_2312_08361_b200.config import SpanConfig
    from support.ref_swarm import build_gpu_swarm
    cfg = SpanConfig(n_blocks=4, hidden_dim=512, n_heads=4, n_kv_heads=2, ffn_dim=1024,
                     vocab_size=64, max_seq_len=512, family="llama", weight_dtype="int8",
                     kv_dtype="bf16", seed=5)
    swarm = build_gpu_swarm(swarmpipe, cfg, n_stages=2, replicas=2, seed=0,
                            server_overrides={"s1a": {"crash_after_messages": 9}})
    res = swarm.client().generate([3, 1, 4], 24, quantized=quantized)
    assert res.counters.recoveries >= 1 and res.counters.restore_events
    emb = om.init_embedding(cfg)
    r0, r1 = om.SpanRunner(cfg, 0, 2), om.SpanRunner(cfg, 2, 4)
    toks = [3, 1, 4]
    x = emb[toks]
    margins = []
    for _ in range(24):
        h = r0.step(x[None])[0]
        if quantized:
            codes, scales = oc.quantize(h)
            h = oc.dequantize(codes, scales, h.shape)
        y = r1.step(h[None])[0]
        lg = om.logits_for(emb, y[-1])
        top2 = np.sort(lg)[-2:]
        margins.append(float(top2[1] - top2[0]))
        t = om.greedy_pick(lg)
        toks.append(t)
        x = emb[[t]]
    print(f"oracle min top1-top2 margin {min(margins):.4g}")
    assert res.tokens == toks
