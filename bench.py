"""Benchmark: Llama-2-70B-shape int8 span decode steps/s and prefill tokens/s
on B200, with the HBM / tensor-core roofline and the reference CPU path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

N=1: all 80 blocks on one GPU (68.5 GB of int8 weights fit).  N>1 (torchrun):
rank r serves span stage_intervals(80, N)[r]; activations move between spans
as int8 codes + f32 scales by NCCL send/recv; N independent sessions are
kept in flight so every GPU works on a different session each tick.
A "step" = one decode token of every in-flight session through all 80 blocks.
Inputs (weights, 68.5 GB) are far larger than L2, so no flush is needed.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "Llama-2-70B-shape decode steps/s and prefill tokens/s, % of HBM/TC roofline"


class _Configs:
    def __getitem__(self, name):
        from paper_2312_08361_b200.config import bloom_176b, llama2_7b, llama2_70b
        return {"llama2-70b": llama2_70b, "llama2-7b": llama2_7b, "bloom-176b": bloom_176b}[name]


CONFIGS = _Configs()
UNIT = "steps/s"


def load_peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        d["_src"] = "measured"
        return d
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
            "_src": "fallback"}


def stage_intervals(n_blocks: int, n_stages: int) -> list[tuple[int, int]]:
    from paper_2312_08361_b200.placement import stage_intervals as si
    return si(n_blocks, n_stages)


# ---------------------------------------------------------------------------
# clocks during the timed region
# ---------------------------------------------------------------------------

class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.path = tempfile.mktemp(suffix=".csv")

    def start(self):
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.f,
                stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.close()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "samples": len(sm), "reasons": sorted(reasons)}


# ---------------------------------------------------------------------------
# CPU baseline: the reference algorithm (oracle port, numpy/OpenBLAS) on host
# ---------------------------------------------------------------------------

_CPU_BLOCK = {}


def cpu_block_decode_seconds(cfg, context: int, reps: int = 3) -> tuple[float, dict]:
    """Time one decode step of one block of the oracle's block forward (the
    reference's SP/model.py:244-280 structure, f32 numpy) at `context`."""
    from oracle import model as om
    d = cfg.hidden_dim
    key = (cfg, context)
    if key not in _CPU_BLOCK:
        p = {}
        for role, a, b in om.block_matrices(cfg):
            p[role] = np.full((a, b), 1e-3, np.float32)   # f32 effective weights (values irrelevant to timing)
        for k in ("ln1_g", "ln2_g"):
            p[k] = np.ones(d, np.float32)
        for k in ("ln1_b", "ln2_b"):
            p[k] = np.zeros(d, np.float32)
        rng = np.random.default_rng(0)
        pk = rng.standard_normal((1, context, cfg.kv_heads, cfg.head_dim)).astype(np.float32)
        pv = rng.standard_normal((1, context, cfg.kv_heads, cfg.head_dim)).astype(np.float32)
        x = rng.standard_normal((1, 1, d)).astype(np.float32)
        _CPU_BLOCK.clear()
        _CPU_BLOCK[key] = (p, pk, pv, x, om.Tables(cfg))
        om.block_forward_batched(cfg, p, x, pk, pv, _CPU_BLOCK[key][4])   # warm
    p, pk, pv, x, tables = _CPU_BLOCK[key]
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        om.block_forward_batched(cfg, p, x, pk, pv, tables)
        ts.append(time.perf_counter() - t0)
    info = {}
    try:
        from threadpoolctl import threadpool_info
        info = {"threadpools": [{k: v for k, v in t.items() if k in ("internal_api", "num_threads")}
                                for t in threadpool_info()]}
    except Exception:
        pass
    return float(np.median(ts)), info


def cpu_threads() -> int:
    try:
        from threadpoolctl import threadpool_info
        n = [t.get("num_threads", 1) for t in threadpool_info()]
        return int(max(n)) if n else 1
    except Exception:
        return os.cpu_count() or 1


# ---------------------------------------------------------------------------
# the reference arm
# ---------------------------------------------------------------------------

def run_reference(args) -> None:
    """The reference's CPU implementation of the path (the oracle port of
    SP/model.py:244-280, f32 numpy/OpenBLAS on every host core), one decode step
    of the whole 80-block span per step.  80 distinct f32 blocks are 274 GB (more
    than host RAM), so every step runs the same 70B-shape block's weights 80
    times: the same arithmetic and the same 3.4 GB weight stream per block."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2312_08361_b200.config import llama2_70b
    # torchrun exports OMP_NUM_THREADS=1; the reference arm uses every host core
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(limits=os.cpu_count())
    except Exception:
        pass
    cfg = llama2_70b()
    context = args.prefill
    n_blocks = args.blocks or cfg.n_blocks

    def step():
        t = 0.0
        for _ in range(n_blocks):
            s, info = cpu_block_decode_seconds(cfg, context, reps=1)
            t += s
        return t, info

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    per = []
    info = {}
    for _ in range(args.steps):
        s, info = step()
        per.append(s)
    wall = time.perf_counter() - t0
    ms_per_step = wall / args.steps * 1e3
    value = args.steps / wall
    cores = cpu_threads()
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"llama2-70b-shape decode, batch 1, context {context}, "
                               f"{n_blocks} blocks",
                   "sample": f"every step = {n_blocks} block decodes (one block's f32 weights "
                             "reused: 80 distinct blocks exceed host RAM)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"oracle block_forward_batched (SP/model.py:244-280 restated, "
                                   f"f32 numpy/OpenBLAS) of a 70B-shape block at context "
                                   f"{context}, x{n_blocks} blocks per step, {args.steps} steps"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": wall, **info,
    }
    print(json.dumps(line))


def self_launch(args) -> bool:
    """`python bench.py --gpus N` with no launcher: re-run this command under
    torch.distributed.run with N ranks (one per GPU) and relay its output.
    Returns True when it launched (the caller exits)."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ or args.impl == "reference":
        return False
    import socket
    env = dict(os.environ)
    # NCCL's init lines (nRanks of every communicator) go to stdout ahead of the
    # JSON line, which is printed last (NCCL's teardown lines are relayed first)
    env["NCCL_DEBUG"] = "INFO"
    env["NCCL_DEBUG_SUBSYS"] = "INIT"
    for _attempt in range(3):
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
               f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
        r = subprocess.run(cmd, env=env, stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                           text=True)
        if r.returncode != 0 and "EADDRINUSE" in r.stderr:
            continue                                   # rendezvous port raced: new port
        break
    lines = r.stdout.splitlines()
    result = [ln for ln in lines if ln.startswith('{"metric"') or ln.startswith('{"impl"')]
    for ln in lines:
        if ln not in result:
            print(ln)
    sys.stderr.write(r.stderr)
    sys.stderr.flush()
    for ln in result:
        print(ln)
    sys.stdout.flush()
    sys.exit(r.returncode)


# ---------------------------------------------------------------------------
# the B200 arm
# ---------------------------------------------------------------------------

def run_b200(args) -> None:
    import torch
    import torch.distributed as dist

    from paper_2312_08361_b200 import _lib
    from paper_2312_08361_b200.blob import HiddenBlob
    from paper_2312_08361_b200.engine import B200ServerEngine, DeviceSpan

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py --gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    peaks = load_peaks()
    cfg = CONFIGS[args.config]()
    if args.weights:
        cfg = cfg.with_(weight_dtype=args.weights)
    B = args.batch                                 # rows per session per step
    n_blocks = args.blocks or cfg.n_blocks
    if args.blocks:
        cfg = cfg.with_(n_blocks=n_blocks)
    start, end = stage_intervals(n_blocks, world)[rank]
    t_gen = time.perf_counter()
    span = DeviceSpan(cfg, start, end, device=local,
                      # sessions in flight (+1 for the N=1 e2e session; the warm-up
                      # prefill's cache is freed before the sessions are created)
                      kv_pool_tokens=(args.prefill + max(args.steps, 50) * 4 + 256) * B
                      * (max(1, world) + (1 if world == 1 else 0)) + 1024)
    torch.cuda.synchronize()
    t_gen = time.perf_counter() - t_gen
    eng = B200ServerEngine(cfg, span=span)
    lib = _lib.load()
    if os.environ.get("SP_PDL") == "0":       # A/B switch: programmatic dependent launch off
        _lib.check(lib.sp_span_set_option(span.handle, 1, 0))
    if os.environ.get("SP_TC_PAIR") == "0":   # A/B switch: single-CTA tcgen05 prefill GEMM
        _lib.check(lib.sp_span_set_option(span.handle, 2, 0))
    if os.environ.get("SP_ATTN_NSUB"):        # A/B switch: decode-attention sub-chunks per CTA
        _lib.check(lib.sp_span_set_option(span.handle, 5, int(os.environ["SP_ATTN_NSUB"])))
    if os.environ.get("SP_ATTN_CLUSTER"):     # A/B switch: decode-attention cluster merge
        _lib.check(lib.sp_span_set_option(span.handle, 6, int(os.environ["SP_ATTN_CLUSTER"])))
    if args.wide_from:                        # option 11 (throughput setting: 3)
        _lib.check(lib.sp_span_set_option(span.handle, 11, args.wide_from))
    d = cfg.hidden_dim
    stream = torch.cuda.current_stream(dev)

    def prof(on: bool):
        _lib.check(lib.sp_span_set_profiling(span.handle, 1 if on else 0))

    def prof_read():
        import ctypes
        n = 5
        ms = (ctypes.c_double * n)()
        by = (ctypes.c_double * n)()
        fl = (ctypes.c_double * n)()
        la = (ctypes.c_int64 * n)()
        _lib.check(lib.sp_span_profile_read(span.handle, n, ms, by, fl, la))
        return [dict(ms=ms[i], bytes=by[i], flops=fl[i], launches=la[i]) for i in range(n)]

    g = torch.Generator(device=dev).manual_seed(1234 + rank)
    sessions = max(1, world)       # sessions in flight (one per pipeline stage)

    # ---- prefill (2048 tokens per session), timed on the device ----
    x_pre = torch.randn(B * args.prefill, d, device=dev, generator=g)
    # untimed warm-up prefill on a throw-away cache: first-call scratch
    # allocations and kernel attribute setup stay out of the timed region
    warm = eng.make_caches(start, end, B)
    eng.run_cached(start, end, warm, HiddenBlob.from_device(x_pre), B, args.prefill, False)
    torch.cuda.synchronize()
    del warm
    caches = [eng.make_caches(start, end, B) for _ in range(sessions)]
    prof(True)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0.record(stream)
    for s in range(sessions):
        eng.run_cached(start, end, caches[s], HiddenBlob.from_device(x_pre), B, args.prefill,
                       False)
    ev1.record(stream)
    torch.cuda.synchronize()
    pre_ms = ev0.elapsed_time(ev1)
    pre_prof = prof_read()
    prof(False)
    pre_ms_t = torch.tensor([pre_ms], device=dev)
    if world > 1:
        dist.all_reduce(pre_ms_t, op=dist.ReduceOp.MAX)
    pre_ms = float(pre_ms_t.item())
    pre_flops = sum(p["flops"] for p in pre_prof)
    prefill_tok_s = sessions * B * args.prefill / (pre_ms / 1e3)

    # ---- C5 prompt-tune forward: the Table 6 shape, 32
    # sequences x (4 prompt + 128) tokens through the span via engine.forward with
    # the reference server's 1024-token micro-batches (SP/server.py:189-194, 216) ----
    pt_b, pt_t = 32, 4 + 128
    x_pt = HiddenBlob.from_device(torch.randn(pt_b * pt_t, d, device=dev, generator=g))
    eng.forward(start, end, x_pt, pt_b, pt_t, 1024, None)              # untimed warm-up
    torch.cuda.synchronize()
    ev0.record(stream)
    eng.forward(start, end, x_pt, pt_b, pt_t, 1024, None)
    ev1.record(stream)
    torch.cuda.synchronize()
    pt_ms = ev0.elapsed_time(ev1)
    del x_pt
    pt_flops = (end - start) * (2 * cfg.block_params() * pt_b * pt_t
                                + pt_b * 2 * cfg.n_heads * cfg.head_dim * pt_t * pt_t)
    pt_ms_t = torch.tensor([pt_ms], device=dev)
    if world > 1:
        dist.all_reduce(pt_ms_t, op=dist.ReduceOp.MAX)
    pt_ms = float(pt_ms_t.item())

    # ---- decode: W warm-up + K timed steps ----
    from paper_2312_08361_b200.pipeline import SpanPipeline
    pipe = SpanPipeline(eng, start, end, caches, rank, world, d, dev, width=B)
    # W warm-up ticks, plus N more for N > 1: the last-to-first ring edge is
    # first used at tick N - 1, and NCCL sets up a p2p connection on first use
    for _ in range(args.warmup + (world if world > 1 else 0)):
        pipe.step()
    torch.cuda.synchronize()
    launches0 = lib.sp_kernel_launches()
    clocks = ClockSampler(local).start()
    time.sleep(0.3)
    # the barrier comes after the clock sampler's start-up (a subprocess: its
    # duration differs per rank), so every rank enters the timed ticks together;
    # otherwise the first rank's events also time its wait for the last one
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        pipe.step()
    e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk = clocks.stop()
    launches = lib.sp_kernel_launches() - launches0
    dec_ms = e0.elapsed_time(e1)
    t = torch.tensor([dec_ms], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dec_ms = float(t.item())
    # every tick each rank advances one session by its span; a full token of a
    # session needs `world` ticks, `world` sessions are in flight
    ticks = args.steps
    steps_done = ticks * sessions / max(1, world)          # full-model tokens, all sessions
    value = steps_done / (dec_ms / 1e3)

    # ---- per-class breakdown: a second pass of K steps with CUDA events around
    # every launch (events add ~2-3 us each, so this pass is slower than the
    # timed one and only apportions the step) ----
    if world > 1:
        dist.barrier()
    prof(True)
    for _ in range(args.steps):
        pipe.step()
    torch.cuda.synchronize()
    dec_prof = prof_read()
    prof(False)

    # ---- the dominant kernel timed back to back: the decode GEMVs of every
    # block of the span (4 per block), CUDA events on the launching stream ----
    import ctypes
    wbytes = ctypes.c_double()
    reps = 3
    _lib.check(lib.sp_span_decode_gemv_only(span.handle, caches[0].handle, start, end,
                                            pipe.y.data_ptr(), B, stream.cuda_stream,
                                            ctypes.byref(wbytes)))
    g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    g0.record(stream)
    for _ in range(reps):
        _lib.check(lib.sp_span_decode_gemv_only(span.handle, caches[0].handle, start, end,
                                                pipe.y.data_ptr(), B, stream.cuda_stream,
                                                ctypes.byref(wbytes)))
    g1.record(stream)
    torch.cuda.synchronize()
    gemv_ms = g0.elapsed_time(g1) / reps
    gemv_launches = 4 * (end - start)

    # ---- end to end through the public API (host buffers, H2D + D2H per step) ----
    e2e = None
    if world == 1:
        c_e2e = eng.make_caches(start, end, B)
        eng.run_cached(start, end, c_e2e, HiddenBlob.from_array(
            np.random.default_rng(0).standard_normal((B * args.prefill, d)).astype(np.float32)),
            B, args.prefill, False)
        # at least 50 steps (as the N > 1 e2e ticks): a host-clocked loop of 20
        # ~12 ms steps is noisy at the percent level
        e2e_steps = max(args.steps, 50)
        rows = torch.from_numpy(np.random.default_rng(1).standard_normal(
            (e2e_steps + args.warmup, B, d)).astype(np.float32)).pin_memory().numpy()
        for i in range(args.warmup):
            eng.run_cached(start, end, c_e2e, HiddenBlob.from_array(rows[i]), B, 1, False).array()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i in range(args.warmup, args.warmup + e2e_steps):
            out = eng.run_cached(start, end, c_e2e, HiddenBlob.from_array(rows[i]), B, 1, False)
            out.array()
        e2e_s = time.perf_counter() - t0
        e2e = {"value": e2e_steps / e2e_s, "unit": UNIT, "h2d_bytes_per_step": 4 * B * d,
               "d2h_bytes_per_step": 4 * B * d, "steps": e2e_steps}
        del c_e2e
    else:
        # N > 1: every rank's span call goes through B200ServerEngine.run_cached;
        # rank 0 uploads its session's input row from pinned host memory, the
        # last rank reads its output row back to the host, every tick
        host_rows = torch.randn(sessions, B, d, generator=torch.Generator().manual_seed(3)
                                ).pin_memory().numpy()
        for _ in range(args.warmup):
            pipe.step_api(host_rows)
        pipe.finish_api()
        torch.cuda.synchronize()
        dist.barrier()
        torch.cuda.synchronize()
        # at least 50 ticks: a wall-clock window of a few milliseconds per rank
        # would let one host hiccup (GC, a page fault) decide the max over ranks
        e2e_ticks = max(args.steps, 50)
        t0 = time.perf_counter()
        for _ in range(e2e_ticks):
            pipe.step_api(host_rows)
        pipe.finish_api()          # the last tick's result read to the host (last rank)
        torch.cuda.synchronize()
        dist.barrier()
        e2e_t = torch.tensor([time.perf_counter() - t0], device=dev)
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
        e2e_s = float(e2e_t.item())
        pipe.verify()          # every received hop passed its relay checksum (raises if not)
        e2e = {"value": e2e_ticks * sessions / max(1, world) / e2e_s, "unit": UNIT,
               "ticks": e2e_ticks,
               "h2d_bytes_per_step": 4 * B * d, "d2h_bytes_per_step": 4 * B * d,
               "note": "per tick: rank 0 H2D of one input row, last rank D2H of one output "
                       "row (HiddenBlob.array_async, collected at the next tick; all inside "
                       "the timed region); wall clock max over ranks"}

    # ---- roofline of the dominant kernel (decode GEMV) ----
    achieved = wbytes.value / (gemv_ms / 1e3) / 1e9
    step_bytes = sum(p["bytes"] for p in dec_prof[:3])
    rank_ms_per_tick = dec_ms / ticks
    line = None
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu:
            t_block, info = cpu_block_decode_seconds(cfg, args.prefill, reps=3)
            cpu = {"value": 1.0 / (t_block * n_blocks), "unit": UNIT, "cores": cpu_threads(),
                   "kind": "port",
                   "sample": f"oracle block_forward_batched (f32 numpy/OpenBLAS) of one "
                             f"{args.config}-shape block, batch 1, context {args.prefill}, "
                             f"median of 3, scaled to {n_blocks} blocks"}
        peak = peaks["hbm_gbs"]
        # DRAM traffic per GEMV launch (dram__bytes_read.sum + dram__bytes_write.sum)
        # from the committed ncu --set full capture of one block's 4 GEMVs
        traffic, traffic_src = None, None
        try:
            if args.config != "llama2-70b" or args.batch != 1 or args.weights:
                raise ValueError("the committed capture is of the 70B batch-1 GEMVs")
            tj = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                             "profiles", "gemv_traffic.json")))
            traffic, traffic_src = tj["dram_bytes_per_launch"], tj["source"]
        except Exception:
            pass
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dec_ms / max(steps_done, 1e-9) * (sessions / max(1, world)) * world
            if world > 1 else dec_ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": ("int8 (weights x 15-bit int digit activations, exact int32 tensor-core MMA; "
                      "f32 residual)") if cfg.weight_dtype == "int8" else
                     ("nf4 (4-bit codes -> 7-bit levels x uint8 block scales, 23-bit int digit "
                      "activations, exact int32 MMA / int64 sums; f32 residual)")
                     if cfg.weight_dtype == "nf4" else
                     "bf16 (weights; activations split hi+lo bf16, f32 accumulate)",
            "data": "synthetic (splitmix64 random-init weights per SP/model.py:55-60, N(0,1) "
                    "hidden rows)",
            "config": {"workload": f"{args.config}-shape {cfg.weight_dtype} span decode, batch "
                                   f"{B}, context {args.prefill}+, {n_blocks} blocks over "
                                   f"{world} GPU(s), {sessions} session(s) in flight",
                       "span_per_gpu": [start, end], "prefill_tokens": args.prefill,
                       "batch": B, "wide_from": args.wide_from or 3,
                       "wire": ({"bytes_per_hop": pipe.wire_bytes_per_token,
                                 "relay_checksum": pipe.check is not None,
                                 "codec": "int8 codes + f32 scales per 64 (SP/quantize.py)"}
                                if world > 1 else None),
                       "l2": f"inputs larger than L2 ({span.weight_bytes / 1e9:.1f} GB weights "
                             f"per GPU)"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "traffic_src": traffic_src,
                         "kernel": f"gemv3_kernel<{cfg.weight_dtype}> (decode QKV/O/gate-up/"
                                   "down GEMVs, norm folded in)",
                         "peak_src": peaks["_src"], "launches": gemv_launches,
                         "avg_launch_us": gemv_ms / gemv_launches * 1e3,
                         "bytes_per_launch": wbytes.value / gemv_launches,
                         "how": f"{gemv_launches} launches (4 per block) back to back x {reps}, "
                                "CUDA events on the launching stream",
                         "note": (None if B < (args.wide_from or 3) else
                                  "at this batch the decode linears run on the weight-side "
                                  "tcgen05 GEMM (option 11); this GEMV-only figure is not the "
                                  "step's kernel — see step_roofline")},
            "step_roofline": {"bytes_per_tick": step_bytes / ticks,
                              "achieved_gbs": step_bytes / ticks / (rank_ms_per_tick / 1e3) / 1e9,
                              "note": "all algorithmic bytes of a step (weights+KV+activations) "
                                      "over the timed step time",
                              "frac": step_bytes / ticks / (rank_ms_per_tick / 1e3) / 1e9 / peak},
            "prefill": {"tokens_per_s": prefill_tok_s, "ms": pre_ms, "tokens": args.prefill,
                        "sessions": sessions, "tflops": pre_flops / (pre_ms / 1e3) / 1e12,
                        "tc_frac": pre_flops / (pre_ms / 1e3) / 1e12 / peaks["bf16_tflops"],
                        "gemm_ms": pre_prof[1]["ms"], "attn_ms": pre_prof[3]["ms"],
                        "gemm_tflops": pre_prof[1]["flops"] / max(pre_prof[1]["ms"], 1e-9) / 1e9},
            "prompt_tune_forward": {"sequences": pt_b, "tokens_per_seq": pt_t,
                                    "micro_batch_tokens": 1024, "ms": pt_ms,
                                    "tokens_per_s": pt_b * pt_t / (pt_ms / 1e3),
                                    "tflops": pt_flops / (pt_ms / 1e3) / 1e12,
                                    "tc_frac": pt_flops / (pt_ms / 1e3) / 1e12 / peaks["bf16_tflops"],
                                    "note": "C5: engine.forward, Table 6 shape (PAPER.md:611-628)"},
            "decode_breakdown_ms_per_tick_evented": {k: dec_prof[i]["ms"] / ticks for i, k in
                                                     enumerate(["gemv", "gemm", "attn_decode",
                                                                "attn_prefill", "other"])},
            "decode_breakdown_note": "a second pass with CUDA events around every launch "
                                     "(event-inflated: the sum exceeds ms_per_step; it only "
                                     "apportions the step)",
            "e2e": e2e, "cpu_baseline": cpu, "clocks": clk, "gpu_launches": int(launches),
            "weight_gen_s": t_gen, "weight_bytes_per_gpu": span.weight_bytes,
        }
        print(json.dumps(line))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference", "ours"])
    ap.add_argument("--prefill", type=int, default=2048)
    ap.add_argument("--blocks", type=int, default=0, help="override n_blocks (debug only)")
    ap.add_argument("--config", default="llama2-70b", choices=["bloom-176b", "llama2-70b",
                                                                "llama2-7b"],
                    help="model shape (BASELINE.json configs; the metric is quoted on llama2-70b)")
    ap.add_argument("--batch", type=int, default=1, help="rows per session per step")
    ap.add_argument("--weights", default="", choices=["", "int8", "nf4", "bf16"],
                    help="override the config's weight format (nf4: the paper's 4-bit format)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--wide-from", type=int, default=0,
                    help="option 11: decode rows per step from which the linears run on the "
                         "weight-side tcgen05 GEMM (0 = library default 3)")
    args = ap.parse_args()
    self_launch(args)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
