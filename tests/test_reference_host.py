"""CPU checks of everything around the kernels that the reference's host layer
sees: the device blob's byte accounting (SP/wire.py:105-122), the oracle engine
inside the reference's own swarm (pins tests/golden/swarm_traces.json and the
oracle before the GPU engine is compared with them), the span placement the
bench uses, and the engine's micro-batch chunking."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import codec as oc
from paper_2312_08361_b200.blob import HiddenBlob, QuantizedHidden
from paper_2312_08361_b200.placement import stage_intervals

TRACES = json.load(open(os.path.join(GOLDEN, "swarm_traces.json")))
BLOBS = json.load(open(os.path.join(GOLDEN, "blob.json")))


def _fnv(b: bytes) -> int:
    h = 0xCBF29CE484222325
    for c in b:
        h = ((h ^ c) * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h


def _host_blob(a, quantized):
    """Our HiddenBlob with a host payload (raw rows, or the codec's codes +
    scales as the GPU codec produces them bit for bit, tests/test_gpu_codec.py)."""
    if not quantized:
        return HiddenBlob.from_array(a)
    codes, scales = oc.quantize(a)
    return HiddenBlob(a.shape[0], a.shape[1],
                      quant=QuantizedHidden(a.shape, 64, scales.reshape(-1), codes.reshape(-1)))


def test_blob_bytes_match_reference_golden():
    """nbytes() and encode() of raw / coded / shape-only blobs equal the
    reference's (tests/golden/blob.json, made by the reference's HiddenBlob)."""
    rng = np.random.default_rng(21)
    it = iter(BLOBS)
    for rows, cols in ((1, 64), (3, 64), (7, 100), (1, 4096), (2, 8192), (1, 14336), (0, 64),
                       (5, 1)):
        a = (rng.standard_normal((rows, cols)) * rng.uniform(0.1, 30)).astype(np.float32)
        for q in (False, True):
            g = next(it)
            b = _host_blob(a, q)
            assert (g["rows"], g["cols"], g["quantized"]) == (rows, cols, q)
            assert b.nbytes() == g["nbytes"], (rows, cols, q)
            assert _fnv(b.encode()) == g["fnv"], (rows, cols, q)
            g = next(it)
            s = HiddenBlob.shape_only(rows, cols, q)
            assert g["synthetic"] and s.nbytes() == g["nbytes"]


def test_blob_bytes_match_live_reference(swarmpipe):
    """Same, against the reference's HiddenBlob live, plus the reference decodes
    our encoding to the same matrix."""
    from swarmpipe.wire import HiddenBlob as RefBlob
    rng = np.random.default_rng(4)
    for rows, cols in ((1, 64), (4, 8192), (3, 130), (2, 1), (0, 16)):
        a = (rng.standard_normal((rows, cols)) * 7).astype(np.float32)
        for q in (False, True):
            ours, ref = _host_blob(a, q), RefBlob.from_array(a, q)
            assert ours.nbytes() == ref.nbytes()
            assert ours.encode() == ref.encode()
            dec, _ = RefBlob.decode(ours.encode())
            assert np.array_equal(dec.array(), ref.array())
        for q in (False, True):
            assert HiddenBlob.shape_only(rows, cols, q).nbytes() == \
                RefBlob.shape_only(rows, cols, q).nbytes()


@pytest.mark.parametrize("tr", TRACES, ids=[t["name"] for t in TRACES])
def test_oracle_engine_reproduces_reference_trace(swarmpipe, tr):
    """The oracle engine (test infrastructure) inside the reference's own
    BlockServer/SimNetwork/SwarmClient reproduces the reference's traces."""
    from paper_2312_08361_b200.config import from_reference
    from support.oracle_engine import OracleEngine
    from support.ref_swarm import rebound
    cfg = swarmpipe.model.ModelConfig(seed=1)
    shared = OracleEngine(from_reference(cfg))
    prof = (swarmpipe.netsim.NetProfile(failure_prob=tr["failure_prob"])
            if "failure_prob" in tr else None)
    with rebound(swarmpipe, lambda config, blocks=None: shared, client_engine=False):
        swarm = swarmpipe.swarm.build_sim_swarm(
            cfg, n_stages=tr["n_stages"], replicas=tr["replicas"], seed=tr.get("seed", 0),
            profile=prof, server_overrides={k: {"crash_after_messages": v}
                                            for k, v in tr["crash"].items()})
    res = swarm.client().generate([3, 1, 4], tr["n_new"], quantized=tr["quantized"])
    c = res.counters
    assert res.tokens == tr["tokens"]
    assert (c.messages, c.recoveries, c.reroutes) == (tr["messages"], tr["recoveries"],
                                                      tr["reroutes"])
    assert [list(e) for e in c.restore_events] == tr["restore_events"]
    assert c.per_step_bytes == tr["per_step_bytes"]
    assert res.elapsed_s == tr["elapsed_s"]
    assert swarm.net.total_bytes() == tr["total_bytes"]


def test_stage_intervals_golden():
    """The bench's per-rank spans equal the reference's stage_intervals
    (tests/golden/assignment.json, SP/swarm.py:40-49), including the 70B plans at
    1/2/4/8 GPUs and BLOOM's 9,9,9,9,9,9,8,8."""
    g = json.load(open(os.path.join(GOLDEN, "assignment.json")))
    for k, v in g["stage_intervals"].items():
        nb, ns = map(int, k.split("_"))
        assert [list(x) for x in stage_intervals(nb, ns)] == v
    assert stage_intervals(80, 8) == [(10 * i, 10 * i + 10) for i in range(8)]


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
