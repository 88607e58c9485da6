"""Failover at the BASELINE shape (config C5): Llama-2-70B int8, 80 blocks over
N span ranks + 1 spare rank (one process per GPU, NCCL), N sessions with a
P-token prompt generating T tokens.  One span rank is dropped mid-generation;
the client (rank 0) detects it and ships the span's cached int8 inputs to the
spare, which replays them (tcgen05 prefill) and joins the ring.

    python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 \\
        tools/failover_bench.py [--prompt 512] [--new 16] [--drop-rank 1]

Rank 0 prints one JSON line: tokens identical to the run without a failure,
the spare's replay time, the client's history send time, ticks/s."""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--prompt", type=int, default=512)
    ap.add_argument("--new", type=int, default=16)
    ap.add_argument("--drop-rank", type=int, default=1)
    ap.add_argument("--blocks", type=int, default=80)
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    from paper_2312_08361_b200.config import llama2_70b
    from paper_2312_08361_b200.engine import B200ServerEngine, DeviceSpan
    from paper_2312_08361_b200.failover import FailoverRing
    from paper_2312_08361_b200.head import ClientHead
    from paper_2312_08361_b200.placement import stage_intervals
    cfg = llama2_70b(n_blocks=args.blocks, max_seq_len=args.prompt + args.new + 64)
    n = world - 1
    a, b = (0, cfg.n_blocks) if rank == n else stage_intervals(cfg.n_blocks, n)[rank]
    span = DeviceSpan(cfg, a, b, device=local, kv_pool_tokens=2 * n * (args.prompt + args.new + 64))
    eng = B200ServerEngine(cfg, span=span)
    head = ClientHead(cfg, local) if rank == 0 else None
    rng = np.random.default_rng(11)
    prefixes = [[int(t) for t in rng.integers(0, cfg.vocab_size, args.prompt)] for _ in range(n)]
    res = {}
    drop_tick = 2 * n + n * (args.new // 2)       # mid-generation
    for tag, drop in (("clean", None), ("fail", (args.drop_rank, drop_tick))):
        ring = FailoverRing(eng, head, cfg, rank, world, dev, prefixes, args.new, drop=drop,
                            detect_timeout_s=2.0, store_prefix=tag)
        ring.warm()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        toks = ring.run()
        torch.cuda.synchronize()
        res[tag] = (toks, ring.replays, time.perf_counter() - t0, ring.n_ticks)
        dist.barrier()
    # gather the spare's replay record on rank 0
    rec = [None] * world
    dist.all_gather_object(rec, res["fail"][1])
    if rank == 0:
        spare = rec[world - 1][0] if rec[world - 1] else {}
        client = res["fail"][1][0] if res["fail"][1] else {}
        print(json.dumps({
            "workload": f"llama2-70b int8, {cfg.n_blocks} blocks over {n} span GPUs + 1 spare, "
                        f"{n} sessions x ({args.prompt} prompt + {args.new} new tokens)",
            "tokens_equal_clean_run": res["fail"][0] == res["clean"][0],
            "dropped_rank": args.drop_rank, "drop_tick": drop_tick,
            "replayed_rows_per_session": spare.get("rows"),
            "spare_replay_ms": 1e3 * spare.get("replay_s", float("nan")),
            "client_history_send_ms": 1e3 * client.get("client_send_s", float("nan")),
            "clean_wall_s": res["clean"][2], "fail_wall_s": res["fail"][2],
            "detect_timeout_s": 2.0,
            "note": "fail_wall_s - clean_wall_s ~ detection timeout + replay",
        }))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
