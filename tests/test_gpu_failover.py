"""The multi-process failover ring on GPUs over NCCL (BASELINE north star:
"the failover path re-runs a dropped span's cached inputs on a replacement
GPU"): 3 span ranks + 1 spare rank, one process per GPU, the 70B kernel family
(int8 weights, GQA, RoPE, SwiGLU, bf16 KV) at a small width, the client head on
rank 0's GPU.  A span rank is dropped mid-generation; rank 0 detects the
missing heartbeat, sends the spare the span's cached int8 inputs over NCCL, the
spare replays them (tcgen05 prefill) and the ring resumes.

Pinned: greedy tokens of every session equal the same ring without a failure;
the replay ran on the spare; its latency is printed; every coded hop carried a
GPU content hash that its receiver verified, and a hop corrupted after its
stamp is refused with the reference's desync error (SP/server.py:388-393).  The same schedule is
pinned against the oracle on CPU in tests/test_failover_gloo.py.

Needs >= 4 GPUs (`gpurun --gpus 4`); skipped with fewer.
"""

import os
import socket

import numpy as np
import pytest
import torch

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(torch.cuda.device_count() < 4, reason="needs >= 4 GPUs")]

P, T = 24, 16


def _cfg():
    from paper_2312_08361_b200.config import SpanConfig
    return SpanConfig(n_blocks=6, hidden_dim=512, n_heads=4, n_kv_heads=2, ffn_dim=1024,
                      vocab_size=256, max_seq_len=512, family="llama", weight_dtype="int8",
                      kv_dtype="bf16", seed=5)


class _CorruptingCheck:
    """relay.WireCheck that flips one payload byte after its n-th stamp (a hop
    corrupted in transit)."""

    def __init__(self, dev, n):
        from paper_2312_08361_b200.relay import WireCheck
        self.inner, self.n, self.k = WireCheck(dev), n, 0
        self.mismatch = self.inner.mismatch

    def stamp(self, wire, payload, off):
        self.inner.stamp(wire, payload, off)
        if self.k == self.n:
            wire[payload // 2] ^= 0x10
        self.k += 1

    def verify(self, wire, payload, off):
        self.inner.verify(wire, payload, off)

    def raise_if_mismatch(self):
        self.inner.raise_if_mismatch()


def _worker(rank, world, port, out_dir, drop, corrupt=False):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    try:
        from paper_2312_08361_b200.engine import B200ServerEngine
        from paper_2312_08361_b200.failover import FailoverRing
        from paper_2312_08361_b200.head import ClientHead
        cfg = _cfg()
        eng = B200ServerEngine(cfg, device=rank)
        head = ClientHead(cfg, rank) if rank == 0 else None
        rng = np.random.default_rng(5)
        prefixes = [[int(t) for t in rng.integers(0, cfg.vocab_size, P)] for _ in range(world - 1)]
        res = {}
        if corrupt:
            from paper_2312_08361_b200.errors import ProtocolError
            chk = _CorruptingCheck(dev, 1) if rank == 0 else None
            ring = FailoverRing(eng, head, cfg, rank, world, dev, prefixes, T,
                                detect_timeout_s=2.0, store_prefix="corrupt", checksum=chk)
            try:
                toks = ring.run()
            except ProtocolError as e:
                toks = str(e)
            torch.cuda.synchronize()
            res["corrupt"] = (toks, ring.replays, ring.check.inner.stamped if rank == 0
                              else ring.check.verified)
        for tag, dr in (() if corrupt else (("clean", None), ("fail", drop))):
            ring = FailoverRing(eng, head, cfg, rank, world, dev, prefixes, T, drop=dr,
                                detect_timeout_s=2.0, store_prefix=tag)
            toks = ring.run()
            torch.cuda.synchronize()
            res[tag] = (toks, ring.replays, ring.check.stamped, ring.check.verified)
            dist.barrier()
        np.save(os.path.join(out_dir, f"r{rank}.npy"), np.array(res, dtype=object),
                allow_pickle=True)
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("drop", [(1, 7), (2, 10)], ids=["drop_middle", "drop_last"])
def test_gpu_failover_ring_tokens_equal_clean_run(tmp_path, drop):
    import torch.multiprocessing as mp
    world = 4
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path), drop), nprocs=world, join=True)
    res = [np.load(tmp_path / f"r{r}.npy", allow_pickle=True).item() for r in range(world)]
    clean = res[0]["clean"][0]
    failed, client_replays = res[0]["fail"][:2]
    spare = res[world - 1]["fail"][1]
    print(f"\nfailover at position {drop[0]} tick {drop[1]}: replayed rows per session "
          f"{spare[0]['rows']}, spare replay {spare[0]['replay_s'] * 1e3:.2f} ms, "
          f"client history send {client_replays[0]['client_send_s'] * 1e3:.2f} ms")
    assert failed == clean
    assert len(spare) == 1 and spare[0]["position"] == drop[0]
    assert sum(spare[0]["rows"]) > 0
    # relay checksums on the GPU: coded hops stamped by their senders, verified by receivers
    assert res[0]["clean"][2] > 0 and all(res[r]["clean"][3] > 0 for r in (1, 2))


def test_gpu_failover_ring_refuses_corrupted_hop(tmp_path):
    """Rank 0's second coded hop is corrupted after its stamp: rank 1 refuses it
    (relay checksum mismatch) and leaves the ring; the client replaces it with the
    spare and finishes."""
    import torch.multiprocessing as mp
    world = 4
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path), None, True), nprocs=world,
             join=True)
    res = [np.load(tmp_path / f"r{r}.npy", allow_pickle=True).item() for r in range(world)]
    assert res[1]["corrupt"][0] == "desync: relay checksum mismatch"
    assert isinstance(res[0]["corrupt"][0], list)
    assert [r["position"] for r in res[0]["corrupt"][1]] == [1]
