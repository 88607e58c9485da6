"""The N > 1 span pipeline (`paper_2312_08361_b200/pipeline.py`) on CPU: 2 and
4 processes over `gloo`, each serving one stage_intervals() span of the toy
model (the reference model, SP/model.py) with the oracle as the span function,
int8 codes + scales on every stage boundary (SP/quantize.py,
SP/client.py:280-287) and f32 rows from the last rank back to rank 0.  The
schedule, the wire format and the grouped send/recv are the ones the GPU bench
runs over NCCL; only `_forward` is swapped.

Pinned: every output row of the last stage equals a single-process run of the
same session (span 0 -> codec round trip -> ... -> last span -> feedback), bit
for bit, and each rank advances exactly the session the schedule names.  Every
coded hop carries the relay checksum (stamped by the sender, verified by the
receiver — the plumbing of relay.WireCheck with the oracle hash); a corrupted
hop is refused with the reference's "relay checksum mismatch" desync.
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
from paper_2312_08361_b200.placement import stage_intervals
from paper_2312_08361_b200.config import toy
from paper_2312_08361_b200.errors import ProtocolError
from paper_2312_08361_b200.pipeline import SpanPipeline
from support.wirecheck import OracleWireCheck


class OraclePipeline(SpanPipeline):
    """SpanPipeline whose span function is the CPU oracle (one SpanRunner per
    session = that session's KV caches on this rank)."""

    def __init__(self, cfg, start, end, rank, world, corrupt=()):
        runners = [om.SpanRunner(cfg, start, end, width=1) for _ in range(max(1, world))]
        super().__init__(None, start, end, runners, rank, world, cfg.hidden_dim,
                         torch.device("cpu"), checksum=OracleWireCheck(corrupt))
        self.log = []          # (tick, session, y) of every forward on this rank

    def _forward(self, session, x, coded_input, quantize_out):
        d = self.d
        if coded_input:
            xin = oc.dequantize(self.in_codes.numpy().copy(), self.in_scales.numpy().copy(), (1, d))
        else:
            xin = x.numpy().reshape(1, d).copy()
        y = self.caches[session].step(xin.reshape(1, 1, d)).reshape(1, d)
        self.y.copy_(torch.from_numpy(np.ascontiguousarray(y, dtype=np.float32)))
        if quantize_out:
            codes, scales = oc.quantize(y)
            self.out_codes.copy_(torch.from_numpy(codes.reshape(-1)))
            self.out_scales.copy_(torch.from_numpy(scales.reshape(-1)))
        self.log.append((self.k, session, y.copy()))


def _worker(rank, world, ticks, port, out_dir, corrupt=None):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = toy(seed=1)
        start, end = stage_intervals(cfg.n_blocks, world)[rank]
        bad = corrupt[1:] if corrupt and corrupt[0] == rank else ()
        pipe = OraclePipeline(cfg, start, end, rank, world, bad)
        for _ in range(ticks):
            pipe.step()
        try:
            pipe.verify()
            verdict = "ok"
        except ProtocolError as e:
            verdict = str(e)
        np.save(os.path.join(out_dir, f"check{rank}.npy"),
                np.array([verdict, pipe.check.stamped, pipe.check.verified], dtype=object),
                allow_pickle=True)
        np.save(os.path.join(out_dir, f"log{rank}.npy"),
                np.array([(k, s, y) for k, s, y in pipe.log], dtype=object), allow_pickle=True)
        np.save(os.path.join(out_dir, f"init{rank}.npy"), pipe.init_rows.numpy())
        dist.barrier()
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 4])
def test_pipeline_matches_single_process(tmp_path, world):
    ticks = 2 * world + 3
    mp.spawn(_worker, args=(world, ticks, _free_port(), str(tmp_path)), nprocs=world, join=True)
    cfg = toy(seed=1)
    d = cfg.hidden_dim
    logs = [np.load(tmp_path / f"log{r}.npy", allow_pickle=True) for r in range(world)]
    init = np.load(tmp_path / "init0.npy")
    spans = stage_intervals(cfg.n_blocks, world)
    # schedule: rank r is active from tick r and advances session (k - r) mod N
    for r in range(world):
        assert [(int(k), int(s)) for k, s, _ in logs[r]] == [(k, (k - r) % world)
                                                             for k in range(r, ticks)]
    # single-process replay of every session: span 0 -> codec -> ... -> last span
    # (f32 out) -> feedback to span 0
    last = logs[-1]
    for s in range(world):
        runners = [om.SpanRunner(cfg, a, b) for a, b in spans]
        x = init[s].reshape(1, d)
        got = [y for _, ss, y in last if ss == s]
        assert got
        for g in got:
            h = x
            for i, rn in enumerate(runners):
                h = rn.step(h.reshape(1, 1, d)).reshape(1, d)
                if i < world - 1:
                    codes, scales = oc.quantize(h)
                    h = oc.dequantize(codes, scales, (1, d))
            assert np.array_equal(g, h)
            x = h
    # relay checksums: every coded hop stamped by its sender, verified by its receiver
    checks = [np.load(tmp_path / f"check{r}.npy", allow_pickle=True) for r in range(world)]
    assert all(c[0] == "ok" for c in checks)
    for r in range(world - 1):
        assert checks[r][1] == ticks - r and checks[r + 1][2] == ticks - r


def test_pipeline_refuses_corrupted_hop(tmp_path):
    """A byte flipped on rank 1's third coded hop (after the stamp) is detected by
    rank 2 (SP/server.py:388-393: Error("desync", "relay checksum mismatch"));
    every other receiver stays clean."""
    world, ticks = 4, 9
    mp.spawn(_worker, args=(world, ticks, _free_port(), str(tmp_path), (1, 2)), nprocs=world,
             join=True)
    checks = [np.load(tmp_path / f"check{r}.npy", allow_pickle=True) for r in range(world)]
    assert [c[0] for c in checks] == ["ok", "ok", "desync: relay checksum mismatch", "ok"]


@pytest.mark.parametrize("world", [2, 4, 8])
def test_stage_split_matches_bench_plan(world):
    """The spans the bench gives each rank (stage_intervals) tile [0, 80) for the
    70B shape at every world size the driver runs."""
    iv = stage_intervals(80, world)
    assert iv[0][0] == 0 and iv[-1][1] == 80
    assert all(a[1] == b[0] for a, b in zip(iv, iv[1:]))
    assert {b - a for a, b in iv} == {80 // world}
