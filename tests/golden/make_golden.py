"""Generate the golden vectors that pin the oracle (and the GPU path) to the
reference implementation.  Run in the build container, where the reference is
importable:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Everything written here comes from calling the reference's own public API
(`swarmpipe.quantize`, `swarmpipe.model`, `swarmpipe.swarm`); nothing from
this repo's product code is involved.  The outputs are small .npz/.json files
committed next to this script so the GPU box (which has no /root/reference)
can check against them.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from swarmpipe import model as M                    # noqa: E402
from swarmpipe.netsim import NetProfile             # noqa: E402
from swarmpipe.quantize import dequantize_hidden, quantize_hidden  # noqa: E402
from swarmpipe.swarm import build_sim_swarm, stage_intervals        # noqa: E402
from swarmpipe.balancer import choose_start, greedy_join_assignment  # noqa: E402
from swarmpipe.client import Strategy               # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def codec_vectors() -> None:
    """Codec KATs: T/test_quantize_wire.py:16-58 and T/test_acceptance.py:343-357
    style inputs (N(0,1) x U(0.1, 30)) at every hidden width of the configs."""
    rng = np.random.default_rng(11)
    cases = {}
    shapes = [(1, 64), (7, 64), (64, 64), (129,), (4096,), (1, 4096), (2, 8192),
              (1, 14336), (3, 100), (1,), (63,), (65,)]
    for i, shape in enumerate(shapes):
        h = (rng.standard_normal(shape) * rng.uniform(0.1, 30)).astype(np.float32)
        cases[f"h{i}"] = h
    z = np.zeros((4, 64), np.float32)
    cases["zeros"] = z
    hot = np.ones(128, np.float32)
    hot[7] = 127.0
    cases["hot"] = hot
    # ties: exact .5 multiples of the scale exercise round-half-even
    tie = (np.arange(-64, 64, dtype=np.float32) * 0.5).astype(np.float32)
    cases["ties"] = tie
    arrays = {}
    for k, h in cases.items():
        q = quantize_hidden(h)
        arrays[f"{k}__in"] = h
        arrays[f"{k}__codes"] = q.codes
        arrays[f"{k}__scales"] = q.scales
        arrays[f"{k}__deq"] = dequantize_hidden(q)
    np.savez_compressed(os.path.join(OUT, "codec.npz"), **arrays)


def toy_model_vectors() -> None:
    """Weights samples, block forward I/O and greedy tokens for the reference
    default config (`T/conftest.py:7-9`, ModelConfig(seed=1)) and the tiny one."""
    arrays = {}
    for name, cfg in (("default", M.ModelConfig(seed=1)),
                      ("tiny", M.ModelConfig(n_blocks=2, hidden_dim=8, n_heads=2,
                                             vocab_size=16, max_seq_len=64, seed=3))):
        blocks, client = M.init_model(cfg)
        for role in ("wq", "wk", "wv", "wo", "w1", "w2"):
            for b in (0, cfg.n_blocks - 1):
                arrays[f"{name}__w_{role}_{b}"] = getattr(blocks[b], role)
        arrays[f"{name}__embedding"] = client.embedding
        rng = np.random.default_rng(5)
        d, H, hd = cfg.hidden_dim, cfg.n_heads, cfg.head_dim
        for tag, (B, n, t0) in {"prefill": (2, 5, 3), "decode": (1, 1, 7),
                                "fresh": (3, 4, 0)}.items():
            x = rng.standard_normal((B, n, d)).astype(np.float32)
            pk = rng.standard_normal((B, t0, H, hd)).astype(np.float32)
            pv = rng.standard_normal((B, t0, H, hd)).astype(np.float32)
            y, kn, vn = M.block_forward_batched(blocks[0], x, pk, pv)
            for k, v in dict(x=x, pk=pk, pv=pv, y=y, kn=kn, vn=vn).items():
                arrays[f"{name}__{tag}_{k}"] = v
        toks = M.reference_generate(cfg, [3, 1, 4] if cfg.vocab_size > 4 else [1, 2, 3], 32)
        arrays[f"{name}__greedy32"] = np.asarray(toks, np.int64)
        # whole-model stepping: prefill 3 rows then 6 decode rows, final-block outputs
        runner = M._LocalRunner(cfg, blocks)
        xs = rng.standard_normal((9, d)).astype(np.float32)
        outs = [runner.step(xs[None, :3])[0]]
        for i in range(3, 9):
            outs.append(runner.step(xs[None, i:i + 1])[0])
        arrays[f"{name}__stack_in"] = xs
        arrays[f"{name}__stack_out"] = np.concatenate(outs, axis=0)
    # beam gather example, T/test_model.py:222-234
    np.savez_compressed(os.path.join(OUT, "toy_model.npz"), **arrays)


def swarm_traces() -> None:
    """Failover counters of the reference swarm under deterministic crash
    injection (no random drops), SURVEY.md Appendix A.  These integer
    counters are engine-independent and must be reproduced
    exactly by the host mirror + GPU engine."""
    cfg = M.ModelConfig(seed=1)
    scenarios = [
        dict(name="c1_one_stage", n_stages=1, replicas=2, crash={"s0a": 6}, n_new=32,
             quantized=False),
        dict(name="two_stage_crash_s1a", n_stages=2, replicas=2, crash={"s1a": 9}, n_new=32,
             quantized=False),
        dict(name="four_stage_crash_s2a_q", n_stages=4, replicas=2, crash={"s2a": 14},
             n_new=24, quantized=True),
        dict(name="four_stage_two_crashes", n_stages=4, replicas=2,
             crash={"s0a": 5, "s3a": 20}, n_new=24, quantized=False),
        dict(name="no_failure_q", n_stages=4, replicas=1, crash={}, n_new=16, quantized=True),
        # random message drops, SURVEY.md 0.10 (seeds 3, 5, 11, p = 0.01, 128 tokens):
        # the counters depend only on the seeded drop stream and the byte sizes
        dict(name="drops_p01_seed3", n_stages=4, replicas=2, crash={}, n_new=128,
             quantized=False, seed=3, failure_prob=1e-2),
        dict(name="drops_p01_seed5_q", n_stages=4, replicas=2, crash={}, n_new=128,
             quantized=True, seed=5, failure_prob=1e-2),
        dict(name="drops_p01_seed11", n_stages=2, replicas=2, crash={"s0b": 40}, n_new=128,
             quantized=False, seed=11, failure_prob=1e-2),
    ]
    out = []
    for sc in scenarios:
        prof = NetProfile(failure_prob=sc["failure_prob"]) if "failure_prob" in sc else None
        swarm = build_sim_swarm(cfg, n_stages=sc["n_stages"], replicas=sc["replicas"],
                                seed=sc.get("seed", 0), profile=prof,
                                server_overrides={k: {"crash_after_messages": v}
                                                  for k, v in sc["crash"].items()})
        res = swarm.client().generate([3, 1, 4], sc["n_new"], strategy=Strategy.DUAL_CACHE,
                                      quantized=sc["quantized"])
        c = res.counters
        out.append(dict(sc, tokens=res.tokens, messages=c.messages, recoveries=c.recoveries,
                        reroutes=c.reroutes, restore_events=[list(e) for e in c.restore_events],
                        step_activation_bytes=c.step_activation_bytes,
                        per_step_bytes=c.per_step_bytes, elapsed_s=res.elapsed_s,
                        total_bytes=swarm.net.total_bytes(),
                        oracle=M.reference_generate(cfg, [3, 1, 4], sc["n_new"])))
    with open(os.path.join(OUT, "swarm_traces.json"), "w") as f:
        json.dump(out, f, indent=1)


def assignment_vectors() -> None:
    """Block-assignment KATs (bit-exact): stage_intervals and greedy placement
    for the 70B / BLOOM configs plus random windows."""
    rng = np.random.default_rng(14)
    out = {"stage_intervals": {}, "choose_start": [], "greedy_join": []}
    for nb, ns in ((80, 1), (80, 2), (80, 4), (80, 8), (70, 8), (70, 2), (32, 1), (8, 4), (8, 3)):
        out["stage_intervals"][f"{nb}_{ns}"] = stage_intervals(nb, ns)
    for _ in range(200):
        nb = int(rng.integers(1, 40))
        cap = int(rng.integers(1, nb + 1))
        loads = [float(v) for v in rng.integers(0, 5, nb)]
        out["choose_start"].append([nb, cap, loads, choose_start(nb, cap, loads)])
    for nb, caps in ((80, [10] * 8), (70, [9] * 8), (70, [9] * 8 + [9] * 8), (80, [20] * 4)):
        servers = [(c, 1.0) for c in caps]
        assign, value = greedy_join_assignment(servers, nb)
        out["greedy_join"].append([nb, caps, [list(assign[i]) for i in range(len(caps))], value])
    with open(os.path.join(OUT, "assignment.json"), "w") as f:
        json.dump(out, f)


def backward_vectors() -> None:
    """Prompt-tuning backward (SP/model.py:320-381, SP/server.py:106-139): one
    block's input gradient, and the engine-level forward(record) + backward of a
    span with micro-batching, from the reference's RealServerEngine."""
    from swarmpipe.server import RealServerEngine
    from swarmpipe.wire import HiddenBlob
    cfg = M.ModelConfig(seed=1)
    blocks, _ = M.init_model(cfg)
    rng = np.random.default_rng(31)
    arrays = {}
    x = rng.standard_normal((2, 7, cfg.hidden_dim)).astype(np.float32)
    dy = rng.standard_normal((2, 7, cfg.hidden_dim)).astype(np.float32)
    arrays["block_x"], arrays["block_dy"] = x, dy
    for b in (0, 5):
        arrays[f"block{b}_dx"] = M.block_backward(blocks[b], M.HiddenStates(x), M.HiddenStates(dy),
                                                  cfg.n_heads).data
    eng = RealServerEngine(cfg, blocks)
    batch, tokens = 3, 6
    xs = rng.standard_normal((batch * tokens, cfg.hidden_dim)).astype(np.float32)
    gs = rng.standard_normal((batch * tokens, cfg.hidden_dim)).astype(np.float32)
    record: list = []
    y = eng.forward(2, 6, HiddenBlob.from_array(xs), batch, tokens, 12, record)
    gx = eng.backward(2, 6, HiddenBlob.from_array(gs), batch, tokens, record)
    arrays["span_x"], arrays["span_g"] = xs, gs
    arrays["span_y"], arrays["span_dx"] = y.array(), gx.array()
    np.savez_compressed(os.path.join(OUT, "backward.npz"), **arrays)


def blob_vectors() -> None:
    """HiddenBlob byte accounting (SP/wire.py:105-122): nbytes() and the FNV-1a
    of encode() for raw / int8-coded / shape-only blobs (inputs: the rng stream
    below, regenerated by tests/test_reference_host.py).  These byte counts drive
    SimNetwork's timing and drop budget, so the device blob must reproduce them."""
    from swarmpipe.wire import HiddenBlob, fnv1a64
    rng = np.random.default_rng(21)
    out = []
    for rows, cols in ((1, 64), (3, 64), (7, 100), (1, 4096), (2, 8192), (1, 14336), (0, 64),
                       (5, 1)):
        a = (rng.standard_normal((rows, cols)) * rng.uniform(0.1, 30)).astype(np.float32)
        for q in (False, True):
            b = HiddenBlob.from_array(a, q)
            out.append(dict(rows=rows, cols=cols, quantized=q, nbytes=b.nbytes(),
                            fnv=fnv1a64(b.encode())))
            s = HiddenBlob.shape_only(rows, cols, q)
            out.append(dict(rows=rows, cols=cols, quantized=q, synthetic=True,
                            nbytes=s.nbytes()))
    with open(os.path.join(OUT, "blob.json"), "w") as f:
        json.dump(out, f)


if __name__ == "__main__":
    only = sys.argv[1:]
    for fn in (codec_vectors, toy_model_vectors, swarm_traces, assignment_vectors,
               backward_vectors, blob_vectors):
        if not only or fn.__name__ in only:
            fn()
    print("golden vectors written to", OUT)
