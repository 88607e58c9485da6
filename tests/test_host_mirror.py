"""Host-side mirror of the session / dual-cache / routing / assignment layers
vs the reference (golden traces from tests/golden/make_golden.py, and the
live reference when /root/reference is importable).  CPU only: the payload
engine here is the test-only oracle engine."""

import json
import os
import sys

import numpy as np
import pytest

from conftest import GOLDEN, REFERENCE_SRC, reference_available
from paper_2312_08361_b200 import balancer as B
from paper_2312_08361_b200.client import SwarmClient, build_swarm
from paper_2312_08361_b200.config import toy
from paper_2312_08361_b200.router import RoutingGraph, ServerRoute
from support.oracle_engine import OracleEngine, OracleHead, install_host_codec

TRACES = json.load(open(os.path.join(GOLDEN, "swarm_traces.json")))


def _run_trace(tr, engine_factory, head):
    cfg = toy(seed=1)
    net, servers, routes = build_swarm(engine_factory, cfg, tr["n_stages"], tr["replicas"],
                                       crash=tr["crash"])
    cl = SwarmClient("client1", cfg, net, routes, head)
    return cl.generate([3, 1, 4], tr["n_new"], quantized=tr["quantized"])


@pytest.mark.parametrize("tr", TRACES, ids=[t["name"] for t in TRACES])
def test_failover_trace_matches_reference(tr, monkeypatch):
    install_host_codec(monkeypatch)
    cfg = toy(seed=1)
    eng = OracleEngine(cfg)
    res = _run_trace(tr, lambda: eng, OracleHead(cfg))
    c = res.counters
    assert res.tokens == tr["tokens"] == tr["oracle"]
    assert c.messages == tr["messages"]
    assert c.recoveries == tr["recoveries"]
    assert c.reroutes == tr["reroutes"]
    assert [list(e) for e in c.restore_events] == tr["restore_events"]
    assert c.step_activation_bytes == tr["step_activation_bytes"]
    assert c.per_step_bytes == tr["per_step_bytes"]


def test_assignment_golden():
    g = json.load(open(os.path.join(GOLDEN, "assignment.json")))
    for k, v in g["stage_intervals"].items():
        nb, ns = map(int, k.split("_"))
        assert [list(x) for x in B.stage_intervals(nb, ns)] == v
    for nb, cap, loads, want in g["choose_start"]:
        assert B.choose_start(nb, cap, loads) == want
    for nb, caps, assign, value in g["greedy_join"]:
        got, val = B.greedy_join_assignment([(c, 1.0) for c in caps], nb)
        assert [list(got[i]) for i in range(len(caps))] == assign and val == value


def test_gpu_span_plans():
    """70B spans at 1/2/4/8 GPUs equal stage_intervals."""
    assert B.gpu_span_plan(80, 8) == [(10 * i, 10 * i + 10) for i in range(8)]
    assert B.gpu_span_plan(70, 8) == [(0, 9), (9, 18), (18, 27), (27, 36), (36, 45), (45, 54),
                                      (54, 62), (62, 70)]
    plan = B.gpu_span_plan(80, 4, "greedy")
    assert sorted(plan) == [(0, 20), (20, 40), (40, 60), (60, 80)]


@pytest.mark.skipif(not reference_available(), reason="reference not mounted")
def test_balancer_and_router_vs_live_reference():
    sys.path.insert(0, REFERENCE_SRC)
    from swarmpipe import balancer as RB
    from swarmpipe.directory import ServerInfo as RSI
    from swarmpipe.router import RoutingGraph as RG, ServerRoute as RSR
    rng = np.random.default_rng(3)
    for _ in range(60):
        nb = int(rng.integers(2, 30))
        servers = []
        for i in range(int(rng.integers(1, 8))):
            cap = int(rng.integers(1, nb + 1))
            st = int(rng.integers(0, nb - cap + 1))
            servers.append((f"s{i:02d}", st, st + cap, float(rng.integers(1, 5))))
        snap_r = [RSI(s, s, a, b, t) for s, a, b, t in servers]
        snap_m = [B.ServerInfo(s, s, a, b, t) for s, a, b, t in servers]
        assert RB.swarm_throughput(snap_r, nb) == B.swarm_throughput(snap_m, nb)
        fr = sorted((r.server_id, r.start, r.end) for r in RB.greedy_fixpoint(snap_r, nb))
        fm = sorted((r.server_id, r.start, r.end) for r in B.greedy_fixpoint(snap_m, nb))
        assert fr == fm
        for s, a, b, t in servers:
            assert RB.propose_rebalance(s, snap_r, nb, RB.RebalanceConfig()) == \
                B.propose_rebalance(s, snap_m, nb, B.RebalanceConfig())
        rg, mg = RG(nb), RoutingGraph(nb)
        rr = [RSR(s, a, b, t * 50, float(rng.integers(0, 20))) for s, a, b, t in servers]
        rg.sync(rr)
        mg.sync([ServerRoute(r.server_id, r.start, r.end, r.throughput, r.rtt_ms) for r in rr])
        try:
            want = rg.find_best_chain(0, nb)
        except Exception:
            with pytest.raises(Exception):
                mg.find_best_chain(0, nb)
            continue
        got = mg.find_best_chain(0, nb)
        assert [(h.server_id, h.start, h.end) for h in want.hops] == \
            [(h.server_id, h.start, h.end) for h in got.hops]


@pytest.mark.parametrize("batch,tokens,mbt", [(32, 132, 1024), (3, 6, 12), (5, 3000, 1024),
                                              (1, 1, 1024), (17, 100, 64)])
def test_device_micro_batches(batch, tokens, mbt):
    """The GPU forward's whole-sequence chunks: cover every sequence once, in
    order, never split a sequence, never exceed max(micro_batch_tokens, device
    cap) tokens unless a single sequence is longer (SP/server.py:189-194), and
    are balanced (sizes differ by at most one sequence)."""
    from paper_2312_08361_b200.engine import device_micro_batches
    cap = 2048
    chunks = list(device_micro_batches(batch, tokens, mbt, cap))
    assert [i for c in chunks for i in range(c.start, c.stop)] == list(range(batch))
    sizes = [c.stop - c.start for c in chunks]
    assert max(sizes) - min(sizes) <= 1
    for n in sizes:
        assert n == 1 or n * tokens <= max(mbt, cap)
    if batch * tokens <= max(mbt, cap):
        assert len(chunks) == 1
