"""The multi-process failover ring (`paper_2312_08361_b200/failover.py`) on CPU:
3 and 4 processes over gloo — N span ranks + 1 spare — with the oracle as every
rank's span engine and client head.  A span rank is dropped mid-generation (it
stops posting heartbeats); the client (rank 0) detects the missing heartbeat,
sends the spare the span's cached int8 inputs, the spare replays them as one
prefill per session, and the ring resumes.

Pinned: every session's greedy tokens equal (a) the same ring without a
failure and (b) a single-process oracle run of the same pipeline (span by span
with the codec round trip at every stage boundary, SP/client.py:280-287); the
replay ran on the spare with the expected history lengths.  The schedule, wire
format, control plane and replay are the ones the GPU runs over NCCL
(tests/test_gpu_failover.py); only the span engine and head are swapped.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import codec as oc
from oracle import model as om
from paper_2312_08361_b200.blob import HiddenBlob
from paper_2312_08361_b200.config import toy
from paper_2312_08361_b200.errors import ProtocolError
from paper_2312_08361_b200.placement import stage_intervals
from support.wirecheck import OracleWireCheck

P, T = 3, 10


class OracleSpanEngine:
    """run_cached / make_caches over the oracle, on CPU torch tensors."""

    def __init__(self, cfg):
        self.cfg = cfg
        self.blocks = {b: om.init_block(cfg, b) for b in range(cfg.n_blocks)}

    def make_caches(self, a, b, width):
        return om.SpanRunner(self.cfg, a, b, blocks=self.blocks, width=width)

    def run_cached(self, a, b, runner, blob, width, n_new, quantized):
        d = self.cfg.hidden_dim
        if blob.dev_codes is not None:
            x = oc.dequantize(blob.dev_codes.numpy(), blob.dev_scales.numpy(), (width * n_new, d))
        else:
            x = blob.dev.numpy()
        y = runner.step(np.ascontiguousarray(x, np.float32).reshape(width, n_new, d))
        y = y.reshape(width * n_new, d)
        if quantized:
            c, s = oc.quantize(y)
            return HiddenBlob(width * n_new, d, dev_codes=torch.from_numpy(c),
                              dev_scales=torch.from_numpy(s))
        return HiddenBlob.from_device(torch.from_numpy(np.ascontiguousarray(y)))


class OracleHead:
    def __init__(self, cfg):
        self.emb = om.init_embedding(cfg)

    def embed_device(self, tokens):
        return torch.from_numpy(self.emb[np.asarray(tokens, dtype=np.intp)].copy())

    def pick_device(self, row):
        return om.greedy_pick(om.logits_for(self.emb, row.numpy()))


def _prefixes(n, vocab):
    rng = np.random.default_rng(17)
    return [[int(t) for t in rng.integers(0, vocab, P)] for _ in range(n)]


def _worker(rank, world, port, out_dir, drop, corrupt=None):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2312_08361_b200.failover import FailoverRing
        cfg = toy(seed=1)
        eng = OracleSpanEngine(cfg)
        head = OracleHead(cfg) if rank == 0 else None
        res = {}
        runs = (("clean", None), ("fail", drop)) if corrupt is None else (("corrupt", None),)
        for tag, dr in runs:
            chk = OracleWireCheck(corrupt[1:] if corrupt and corrupt[0] == rank else ())
            ring = FailoverRing(eng, head, cfg, rank, world, torch.device("cpu"),
                                _prefixes(world - 1, cfg.vocab_size), T, drop=dr,
                                detect_timeout_s=1.0, store_prefix=tag, checksum=chk)
            try:
                toks = ring.run()
            except ProtocolError as e:
                toks = str(e)
            res[tag] = (toks, ring.replays, chk.stamped, chk.verified)
            if corrupt is None:
                dist.barrier()
        np.save(os.path.join(out_dir, f"r{rank}.npy"), np.array(res, dtype=object),
                allow_pickle=True)
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _oracle_tokens(cfg, prefix, n_spans):
    emb = om.init_embedding(cfg)
    runners = [om.SpanRunner(cfg, a, b) for a, b in stage_intervals(cfg.n_blocks, n_spans)]
    toks = list(prefix)
    x = emb[toks]
    for _ in range(T):
        h = x
        for i, r in enumerate(runners):
            h = r.step(h[None])[0]
            if i < n_spans - 1:
                c, s = oc.quantize(h)
                h = oc.dequantize(c, s, h.shape)
        t = om.greedy_pick(om.logits_for(emb, h[-1]))
        toks.append(t)
        x = emb[[t]]
    return toks


@pytest.mark.parametrize("world,drop", [(3, (1, 5)), (4, (1, 7)), (4, (2, 9))],
                         ids=["2spans_drop_last", "3spans_drop_middle", "3spans_drop_last"])
def test_failover_ring_tokens_equal_clean_run_and_oracle(tmp_path, world, drop):
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path), drop), nprocs=world, join=True)
    cfg = toy(seed=1)
    res = [np.load(tmp_path / f"r{r}.npy", allow_pickle=True).item() for r in range(world)]
    clean = res[0]["clean"][0]
    failed, client_replays = res[0]["fail"][:2]
    prefixes = _prefixes(world - 1, cfg.vocab_size)
    for s, p in enumerate(prefixes):
        want = _oracle_tokens(cfg, p, world - 1)
        assert clean[s] == want
        assert failed[s] == want
    # the client shipped the history once; the spare replayed it
    spare = res[world - 1]["fail"][1]
    assert len(client_replays) == 1 and len(spare) == 1
    pos = drop[0]
    assert client_replays[0]["position"] == pos and spare[0]["position"] == pos
    assert spare[0]["rows"] == client_replays[0]["rows"] and sum(spare[0]["rows"]) > 0
    assert res[world - 1]["clean"][1] == []              # the spare idles without a failure
    # relay checksums: hops, relay copies and the replayed history all verified
    assert all(res[r]["fail"][2] > 0 for r in range(world - 2))      # coded senders
    assert all(res[r]["fail"][3] > 0 for r in range(1, world))       # receivers + spare


def test_failover_ring_refuses_corrupted_hop(tmp_path):
    """A byte flipped on the client span's second coded hop (after its stamp):
    the next span refuses it at that tick with the reference's desync error
    (SP/server.py:388-393) and leaves the ring; the client then treats it as
    failed and the spare takes its position (the run completes)."""
    world = 3
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path), None, (0, 1)), nprocs=world,
             join=True)
    res = [np.load(tmp_path / f"r{r}.npy", allow_pickle=True).item() for r in range(world)]
    assert res[1]["corrupt"][0] == "desync: relay checksum mismatch"
    assert isinstance(res[0]["corrupt"][0], list)            # the client finished
    assert [r["position"] for r in res[0]["corrupt"][1]] == [1]   # ... after a failover
