"""Span forward on the GPU vs the CPU oracle (and the reference's golden
vectors) through the engine protocol of SP/server.py:77-142.

Tolerances (written here):
* toy family (f32 end to end): max-abs 1e-5 — the reference's own bound
  (T/test_server.py:42-58, :123-136);
* interleaving / micro-batching: array_equal (T/test_server.py:91-119, :247-255);
* bf16/int8-weight Llama/BLOOM shapes: decode max-abs <= 2e-3 * max|y|
  (f32-class hi/lo tensor-core GEMV), prefill <= 2e-2 * max|y| (f32 SIMT
  GEMM with bf16 KV), measured against the oracle on the same rounded weights.
"""

import numpy as np
import pytest

from oracle import model as om
from paper_2312_08361_b200.config import SpanConfig, toy

pytestmark = pytest.mark.gpu


def _engine(cfg):
    from paper_2312_08361_b200.engine import B200ServerEngine
    return B200ServerEngine(cfg)


def _blob(a, quantized=False):
    from paper_2312_08361_b200.blob import HiddenBlob
    return HiddenBlob.from_array(a, quantized)


def _errs(got, want):
    """(max-abs / max|y|, p99 of the per-element relative error with a 1e-3*max|y|
    floor): the second shows what the max-abs ratio can hide in small outputs."""
    s = np.abs(want).max()
    rel = np.abs(got - want) / (np.abs(want) + 1e-3 * s)
    return float(np.abs(got - want).max() / s), float(np.percentile(rel, 99))


def test_toy_stack_matches_reference_golden(golden_toy):
    """prefill 3 rows then 6 decode rows through all 8 blocks (reference run)."""
    eng = _engine(toy(seed=1))
    xs = golden_toy["default__stack_in"]
    want = golden_toy["default__stack_out"]
    caches = eng.make_caches(0, 8, 1)
    outs = [eng.run_cached(0, 8, caches, _blob(xs[:3]), 1, 3, False).array()]
    for i in range(3, 9):
        outs.append(eng.run_cached(0, 8, caches, _blob(xs[i:i + 1]), 1, 1, False).array())
    got = np.concatenate(outs)
    assert eng.cache_length(caches) == 9
    assert np.abs(got - want).max() < 1e-5


def test_toy_greedy_tokens_match_reference(golden_toy):
    """reference_generate(ModelConfig(seed=1), [3,1,4], 32) with the GPU span
    and the oracle's tied head (client side stays on the host here)."""
    cfg = toy(seed=1)
    eng = _engine(cfg)
    emb = golden_toy["default__embedding"]
    caches = eng.make_caches(0, 8, 1)
    toks = [3, 1, 4]
    x = emb[toks]
    for _ in range(32):
        y = eng.run_cached(0, 8, caches, _blob(x), 1, x.shape[0], False).array()
        t = om.greedy_pick(om.logits_for(emb, y[-1]))
        toks.append(t)
        x = emb[[t]]
    assert toks == list(golden_toy["default__greedy32"])


def test_five_steps_match_local_stage():
    """T/test_server.py:42-58 on blocks [2, 5)."""
    cfg = toy(seed=1)
    eng = _engine(cfg)
    rng = np.random.default_rng(0)
    x_all = rng.standard_normal((5, 64)).astype(np.float32)
    runner = om.SpanRunner(cfg, 2, 5)
    caches = eng.make_caches(2, 5, 1)
    for i in range(5):
        got = eng.run_cached(2, 5, caches, _blob(x_all[i:i + 1]), 1, 1, False).array()
        want = runner.step(x_all[i:i + 1][None])[0]
        assert np.abs(got - want).max() < 1e-5
    assert eng.cache_length(caches) == 5


def test_interleaved_sessions_bit_identical():
    """T/test_server.py:91-119."""
    eng = _engine(toy(seed=1))
    rng = np.random.default_rng(1)
    xa = rng.standard_normal((6, 64)).astype(np.float32)
    xb = rng.standard_normal((6, 64)).astype(np.float32)

    def serial(xs):
        c = eng.make_caches(0, 4, 1)
        return np.concatenate([eng.run_cached(0, 4, c, _blob(xs[i:i + 1]), 1, 1, False).array()
                               for i in range(6)])

    sa, sb = serial(xa), serial(xb)
    ca, cb = eng.make_caches(0, 4, 1), eng.make_caches(0, 4, 1)
    ia, ib = [], []
    for i in range(6):
        ia.append(eng.run_cached(0, 4, ca, _blob(xa[i:i + 1]), 1, 1, False).array())
        ib.append(eng.run_cached(0, 4, cb, _blob(xb[i:i + 1]), 1, 1, False).array())
    assert np.array_equal(np.concatenate(ia), sa)
    assert np.array_equal(np.concatenate(ib), sb)


def test_restore_then_continue():
    """T/test_server.py:123-136: replay of 10 rows then 1 step == uninterrupted."""
    eng = _engine(toy(seed=1))
    rng = np.random.default_rng(2)
    x = rng.standard_normal((11, 64)).astype(np.float32)
    c1 = eng.make_caches(0, 4, 1)
    direct = [eng.run_cached(0, 4, c1, _blob(x[i:i + 1]), 1, 1, False).array() for i in range(11)]
    c2 = eng.make_caches(0, 4, 1)
    eng.run_cached(0, 4, c2, _blob(x[:10]), 1, 10, False)
    res = eng.run_cached(0, 4, c2, _blob(x[10:11]), 1, 1, False).array()
    assert np.abs(res - direct[10]).max() < 1e-5


def test_reorder_paper_example():
    """T/test_server.py:167-178: new slot i <- old slot idx[i]-1."""
    eng = _engine(toy(seed=1))
    rng = np.random.default_rng(3)
    c = eng.make_caches(0, 4, 5)
    x = rng.standard_normal((5, 64)).astype(np.float32)
    eng.run_cached(0, 4, c, _blob(x), 5, 1, False)
    old = [blk.keys.copy() for blk in c]
    eng.reorder(c, [1, 1, 0, 2, 1])
    for before, blk in zip(old, c):
        keys = blk.keys
        for new_slot, old_slot in enumerate([2, 2, 1, 3, 2]):
            assert np.array_equal(keys[new_slot], before[old_slot - 1])
    # widening from a prefill, then stepping the clones (copy-on-write tail)
    c = eng.make_caches(0, 4, 1)
    eng.run_cached(0, 4, c, _blob(x[:3]), 1, 3, False)
    eng.reorder(c, [0, 0, 0, 0])
    assert c.width == 4 and all(b.width == 4 and b.length == 3 for b in c)
    y = eng.run_cached(0, 4, c, _blob(x[:4]), 4, 1, False).array()
    runner = om.SpanRunner(toy(seed=1), 0, 4)
    runner.step(x[:3][None])
    runner.reorder([0, 0, 0, 0])
    want = runner.step(x[:4][:, None, :])[:, 0]
    assert np.abs(y - want).max() < 1e-5


def test_micro_batch_split_bit_identical():
    """T/test_server.py:247-255: a forward split into micro-batches equals the
    whole batch bit for bit — with a real split (4 chunks vs 1)."""
    eng = _engine(toy(seed=1))
    rng = np.random.default_rng(4)
    x = rng.standard_normal((4, 512, 64)).astype(np.float32)
    blob = _blob(x.reshape(-1, 64))
    eng.stateless_tokens = 4096
    whole = eng.forward(0, 2, blob, 4, 512, micro_batch_tokens=10**9, record=None).array()
    assert eng.last_forward_chunks == 1
    eng.stateless_tokens = 512
    split = eng.forward(0, 2, blob, 4, 512, micro_batch_tokens=512, record=None).array()
    assert eng.last_forward_chunks == 4
    assert np.array_equal(whole, split)
    runner = om.SpanRunner(toy(seed=1), 0, 2, width=4)
    want = runner.step(x)
    err = np.abs(whole.reshape(4, 512, 64) - want).max()
    print(f"toy stateless forward max-abs err vs oracle {err:.3g}")
    assert err < 1e-5


@pytest.mark.parametrize("batch,tokens", [(6, 40), (4, 300)])
def test_micro_batch_split_bit_identical_tensor_core(batch, tokens):
    """The same pin on the int8 tcgen05 path, where the whole batch and the
    one-sequence chunks run different GEMM schedules (CTA-pair tiles vs the
    few-token split-K kernel): exact integer accumulation makes every row
    independent of M, so the results are array_equal."""
    cfg = SMALL["llama_int8"]
    eng = _engine(cfg)
    rng = np.random.default_rng(8)
    x = rng.standard_normal((batch * tokens, cfg.hidden_dim)).astype(np.float32)
    blob = _blob(x)
    eng.stateless_tokens = 4096
    whole = eng.forward(0, cfg.n_blocks, blob, batch, tokens, 10**9, None).array()
    assert eng.last_forward_chunks == 1
    eng.stateless_tokens = tokens
    split = eng.forward(0, cfg.n_blocks, blob, batch, tokens, tokens, None).array()
    assert eng.last_forward_chunks == batch
    assert np.array_equal(whole, split)


def test_quantized_output_equals_codec_of_output():
    eng = _engine(toy(seed=1))
    rng = np.random.default_rng(5)
    x = rng.standard_normal((3, 64)).astype(np.float32)
    c1, c2 = eng.make_caches(0, 8, 1), eng.make_caches(0, 8, 1)
    raw = eng.run_cached(0, 8, c1, _blob(x), 1, 3, False).array()
    q = eng.run_cached(0, 8, c2, _blob(x), 1, 3, True)
    from oracle import codec as oc
    codes, scales = oc.quantize(raw)
    assert np.array_equal(q.quant.codes, codes) and np.array_equal(q.quant.scales, scales)
    # quantized input path: dequant in-kernel == host dequant
    c3, c4 = eng.make_caches(4, 8, 1), eng.make_caches(4, 8, 1)
    a = eng.run_cached(4, 8, c3, q, 1, 3, False).array()
    b = eng.run_cached(4, 8, c4, _blob(oc.dequantize(codes, scales, raw.shape)), 1, 3,
                       False).array()
    assert np.array_equal(a, b)


SMALL = {
    "llama_int8": SpanConfig(n_blocks=3, hidden_dim=512, n_heads=4, n_kv_heads=2, ffn_dim=1024,
                             vocab_size=64, max_seq_len=512, family="llama",
                             weight_dtype="int8", kv_dtype="bf16", seed=5),
    "llama_bf16": SpanConfig(n_blocks=3, hidden_dim=512, n_heads=4, ffn_dim=768,
                             vocab_size=64, max_seq_len=512, family="llama",
                             weight_dtype="bf16", kv_dtype="bf16", seed=6),
    "bloom_int8": SpanConfig(n_blocks=2, hidden_dim=512, n_heads=4, vocab_size=64,
                             max_seq_len=512, family="bloom", weight_dtype="int8",
                             kv_dtype="bf16", seed=7),
    "llama_f32": SpanConfig(n_blocks=2, hidden_dim=256, n_heads=2, n_kv_heads=1, ffn_dim=512,
                            vocab_size=64, max_seq_len=512, family="llama", seed=8),
    # nf4 weights (oracle/model.py quantize_columns_nf4): decode on the exact
    # integer GEMV, prefill on the exact-f32 SIMT GEMM over the same levels
    "llama_nf4": SpanConfig(n_blocks=3, hidden_dim=512, n_heads=4, n_kv_heads=2, ffn_dim=1024,
                            vocab_size=64, max_seq_len=512, family="llama",
                            weight_dtype="nf4", kv_dtype="bf16", seed=10),
    "bloom_nf4": SpanConfig(n_blocks=2, hidden_dim=512, n_heads=4, vocab_size=64,
                            max_seq_len=512, family="bloom", weight_dtype="nf4",
                            kv_dtype="bf16", seed=11),
    # the 70B attention shape: 8 query heads per kv head, head_dim 128
    "llama_g8": SpanConfig(n_blocks=2, hidden_dim=1024, n_heads=8, n_kv_heads=1, ffn_dim=2048,
                           vocab_size=64, max_seq_len=2048, family="llama",
                           weight_dtype="int8", kv_dtype="bf16", seed=9),
}


@pytest.mark.parametrize("name", sorted(SMALL))
def test_extended_families_vs_oracle(name):
    cfg = SMALL[name]
    eng = _engine(cfg)
    rng = np.random.default_rng(11)
    d = cfg.hidden_dim
    t_pre, n_dec = 70, 6        # crosses a 64-position page boundary
    x = rng.standard_normal((t_pre + n_dec, d)).astype(np.float32)
    runner = om.SpanRunner(cfg, 0, cfg.n_blocks)
    c = eng.make_caches(0, cfg.n_blocks, 1)
    got = eng.run_cached(0, cfg.n_blocks, c, _blob(x[:t_pre]), 1, t_pre, False).array()
    want = runner.step(x[None, :t_pre])[0]
    # prefill: tcgen05 GEMMs on 15-bit activation digit planes, tcgen05 attention
    # with hi/lo Q against the bf16 cache (f32 families: exact-f32 SIMT)
    tol = 2e-3 if cfg.weight_dtype != "f32" else 1e-4
    e_pre, r_pre = _errs(got, want)
    errs = []
    for i in range(t_pre, t_pre + n_dec):
        g = eng.run_cached(0, cfg.n_blocks, c, _blob(x[i:i + 1]), 1, 1, False).array()
        w = runner.step(x[None, i:i + 1])[0]
        errs.append(_errs(g, w))
    print(f"{name}: prefill err {e_pre:.2e} (p99 rel {r_pre:.2e}); decode err max "
          f"{max(e for e, _ in errs):.2e} (p99 rel {max(r for _, r in errs):.2e})")
    assert e_pre <= tol
    assert max(e for e, _ in errs) <= tol


def test_engine_blocks_params_hash_matches_reference(golden_toy):
    """`params_hash(engine.blocks)` (T/test_server.py:228) reads the GPU
    weights back; for the toy config they equal the reference arrays."""
    eng = _engine(toy(seed=1))
    arrs = eng.blocks[0].arrays()
    assert np.array_equal(arrs[0], golden_toy["default__w_wq_0"])
    assert np.array_equal(arrs[5], golden_toy["default__w_w2_0"])


def test_tc_prefill_matches_simt_and_is_batch_invariant():
    """tcgen05 int8 prefill GEMM (2 activation digit planes, exact int32
    accumulate) vs the exact-f32 SIMT GEMM on the same weights, and the
    micro-batch invariance of T/test_server.py:247-255 on the tensor-core path."""
    import ctypes
    cfg = SMALL["llama_int8"]
    from paper_2312_08361_b200 import _lib
    from paper_2312_08361_b200.engine import DeviceSpan, B200ServerEngine
    span_tc = DeviceSpan(cfg, 0, cfg.n_blocks)
    span_ref = DeviceSpan(cfg, 0, cfg.n_blocks)
    _lib.check(span_ref.lib.sp_span_set_option(span_ref.handle, 0, 0))
    e_tc, e_ref = B200ServerEngine(cfg, span=span_tc), B200ServerEngine(cfg, span=span_ref)
    rng = np.random.default_rng(21)
    x = rng.standard_normal((3 * 150, cfg.hidden_dim)).astype(np.float32)
    a = e_tc.forward(0, cfg.n_blocks, _blob(x), 3, 150, 10**9, None).array()
    b = e_ref.forward(0, cfg.n_blocks, _blob(x), 3, 150, 10**9, None).array()
    rel = np.abs(a - b).max() / np.abs(b).max()
    assert rel < 2e-3, rel
    split = e_tc.forward(0, cfg.n_blocks, _blob(x), 3, 150, 150, None).array()
    assert np.array_equal(a, split)
    runner = om.SpanRunner(cfg, 0, cfg.n_blocks, width=3)
    want = runner.step(x.reshape(3, 150, -1)).reshape(-1, cfg.hidden_dim)
    assert np.abs(a - want).max() <= 2e-2 * np.abs(want).max()


@pytest.mark.gpu
def test_tc_pair_gemm_equals_single_cta():
    """The CTA-pair tcgen05 GEMM (cta_group::2, M = 256) and the single-CTA one
    accumulate the same exact integers: outputs must be bit-identical, also for
    token counts that are not a multiple of the 256-token pair tile."""
    cfg = SMALL["llama_int8"]
    from paper_2312_08361_b200 import _lib
    from paper_2312_08361_b200.engine import DeviceSpan, B200ServerEngine
    span = DeviceSpan(cfg, 0, cfg.n_blocks)
    eng = B200ServerEngine(cfg, span=span)
    rng = np.random.default_rng(5)
    for batch, tokens in ((1, 300), (2, 129), (1, 512)):
        x = rng.standard_normal((batch * tokens, cfg.hidden_dim)).astype(np.float32)
        _lib.check(span.lib.sp_span_set_option(span.handle, 2, 1))
        pair = eng.forward(0, cfg.n_blocks, _blob(x), batch, tokens, 10**9, None).array()
        _lib.check(span.lib.sp_span_set_option(span.handle, 2, 0))
        single = eng.forward(0, cfg.n_blocks, _blob(x), batch, tokens, 10**9, None).array()
        _lib.check(span.lib.sp_span_set_option(span.handle, 2, 1))
        assert np.array_equal(pair, single), (batch, tokens, float(np.abs(pair - single).max()),
                                              float(np.abs(single).max()))


@pytest.mark.parametrize("name", ["llama_int8", "bloom_int8", "llama_bf16", "llama_g8",
                                  "llama_nf4", "bloom_nf4"])
def test_extended_families_greedy_tokens_match_oracle(name):
    """BASELINE north star: identical greedy tokens to the CPU oracle and
    max-abs logits diff <= 1e-2 — prompt through the prefill path (tcgen05 for
    int8), then 24 decode steps (tensor-core GEMV + fused attention), GPU head."""
    from paper_2312_08361_b200.head import ClientHead
    cfg = SMALL[name]
    eng = _engine(cfg)
    head = ClientHead(cfg)
    emb = om.init_embedding(cfg)
    runner = om.SpanRunner(cfg, 0, cfg.n_blocks)
    c = eng.make_caches(0, cfg.n_blocks, 1)
    toks_gpu, toks_cpu = [3, 1, 4], [3, 1, 4]
    xg = head.embed_array(toks_gpu)
    xc = emb[toks_cpu]
    assert np.array_equal(xg, xc)
    worst = 0.0
    for _ in range(24):
        yg = eng.run_cached(0, cfg.n_blocks, c, _blob(xg), 1, xg.shape[0], False).array()
        yc = runner.step(xc[None])[0]
        lg, lc = om.logits_for(emb, yg[-1]), om.logits_for(emb, yc[-1])
        worst = max(worst, float(np.abs(lg - lc).max()))
        tg, tc = head.pick(yg), om.greedy_pick(lc)
        toks_gpu.append(tg)
        toks_cpu.append(tc)
        xg = head.embed_array([tg])
        xc = emb[[tc]]
    assert toks_gpu == toks_cpu
    assert worst <= 1e-2, worst


@pytest.mark.parametrize("name", ["llama_int8", "bloom_int8", "llama_g8"])
def test_wide_gemm_equals_gemv(name):
    """Option 11: a 5-row step on the decode GEMV (option 11 = 9) and on the
    weight-side tcgen05 GEMM (the default, from 3 rows) give the same rows bit for
    bit — the GEMM path restates the GEMV's statistics, activation code, scale and
    epilogue — and both match the oracle."""
    from paper_2312_08361_b200 import _lib
    cfg = SMALL[name]
    eng = _engine(cfg)
    rng = np.random.default_rng(61)
    d = cfg.hidden_dim
    x = rng.standard_normal((5, 30 + 2, d)).astype(np.float32)
    outs = {}
    try:
        for wf in (9, 3):
            _lib.check(eng.lib.sp_span_set_option(eng.span.handle, 11, wf))
            c = eng.make_caches(0, cfg.n_blocks, 5)
            eng.run_cached(0, cfg.n_blocks, c, _blob(x[:, :30].reshape(-1, d)), 5, 30, False)
            outs[wf] = [eng.run_cached(0, cfg.n_blocks, c, _blob(x[:, i]), 5, 1, False).array()
                        for i in (30, 31)]
    finally:
        _lib.check(eng.lib.sp_span_set_option(eng.span.handle, 11, 3))
    for a, b in zip(outs[9], outs[3]):
        assert np.array_equal(a, b)
    runner = om.SpanRunner(cfg, 0, cfg.n_blocks, width=5)
    runner.step(x[:, :30])
    for j, i in enumerate((30, 31)):
        w = runner.step(x[:, i:i + 1])[:, 0]
        assert np.abs(outs[3][j] - w).max() <= 2e-3 * np.abs(w).max()


@pytest.mark.parametrize("name,width", [("llama_int8", 12), ("bloom_int8", 16), ("llama_int8", 32)])
def test_wide_decode_token_tile_gemm(name, width):
    """The token-tile wide GEMM (option 10 off: tokens padded to M = 128,
    normalise-then-code digit planes) against the default weight-side path
    (the GEMV's numerics) and the oracle: equal to the decode tolerance."""
    from paper_2312_08361_b200 import _lib
    cfg = SMALL[name]
    rng = np.random.default_rng(53)
    d = cfg.hidden_dim
    x = rng.standard_normal((width, 30 + 2, d)).astype(np.float32)
    outs = {}
    eng = _engine(cfg)
    try:
        for v in (1, 0):
            _lib.check(eng.lib.sp_span_set_option(eng.span.handle, 10, v))
            c = eng.make_caches(0, cfg.n_blocks, width)
            eng.run_cached(0, cfg.n_blocks, c, _blob(x[:, :30].reshape(-1, d)), width, 30, False)
            outs[v] = [eng.run_cached(0, cfg.n_blocks, c, _blob(x[:, i]), width, 1, False).array()
                       for i in (30, 31)]
    finally:
        _lib.check(eng.lib.sp_span_set_option(eng.span.handle, 10, 1))
    runner = om.SpanRunner(cfg, 0, cfg.n_blocks, width=width)
    runner.step(x[:, :30])
    for j, i in enumerate((30, 31)):
        w = runner.step(x[:, i:i + 1])[:, 0]
        sc = np.abs(w).max()
        assert np.abs(outs[0][j] - w).max() <= 2e-3 * sc
        assert np.abs(outs[0][j] - outs[1][j]).max() <= 2e-3 * sc


@pytest.mark.parametrize("name,width", [("llama_int8", 9), ("bloom_int8", 16), ("llama_g8", 12),
                                        ("llama_int8", 24), ("bloom_int8", 32), ("llama_int8", 40)])
def test_wide_decode_vs_oracle(name, width):
    """Decode with >= 3 rows per step (option 11) runs its linears on the tcgen05 GEMM
    (one pass over the weights for all rows: weight-side up to 32 rows, the
    token-tile split-K GEMM beyond) and attention on the fused decode kernel;
    every row vs the oracle at the decode tolerance."""
    cfg = SMALL[name]
    eng = _engine(cfg)
    rng = np.random.default_rng(13)
    d = cfg.hidden_dim
    x = rng.standard_normal((width, 40 + 4, d)).astype(np.float32)
    runner = om.SpanRunner(cfg, 0, cfg.n_blocks, width=width)
    c = eng.make_caches(0, cfg.n_blocks, width)
    eng.run_cached(0, cfg.n_blocks, c, _blob(x[:, :40].reshape(-1, d)), width, 40, False)
    runner.step(x[:, :40])
    for i in range(40, 44):
        g = eng.run_cached(0, cfg.n_blocks, c, _blob(x[:, i]), width, 1, False).array()
        w = runner.step(x[:, i:i + 1])[:, 0]
        s = np.abs(w).max()
        assert np.abs(g - w).max() <= 2e-3 * s, (i, np.abs(g - w).max() / s)
    assert eng.cache_length(c) == 44


@pytest.mark.parametrize("name", ["llama_int8", "bloom_int8", "llama_g8", "llama_bf16"])
def test_decode_width_invariant(name):
    """Decode numerics do not depend on the width of the step (
    T/test_server.py:247-255 pins the same for forward): slot r of a width-3, 8,
    12 and 24 session equals a width-1 session on the same rows, bit for bit —
    across the switch from the decode GEMV (1-2 rows) to the weight-side tcgen05
    GEMM (3-32 rows), which codes, scales and reduces every row exactly like the
    GEMV (one 15-bit activation code, exact integer products, the GEMV's
    statistics and epilogue order, per-row attention)."""
    cfg = SMALL[name]
    eng = _engine(cfg)
    rng = np.random.default_rng(31)
    d = cfg.hidden_dim
    widths = (3, 8, 12, 24)
    x = rng.standard_normal((max(widths), 70 + 3, d)).astype(np.float32)
    single = []
    for r in range(max(widths)):
        c1 = eng.make_caches(0, cfg.n_blocks, 1)
        eng.run_cached(0, cfg.n_blocks, c1, _blob(x[r, :70]), 1, 70, False)
        single.append([eng.run_cached(0, cfg.n_blocks, c1, _blob(x[r, i:i + 1]), 1, 1,
                                      False).array()[0] for i in range(70, 73)])
    for width in widths:
        cw = eng.make_caches(0, cfg.n_blocks, width)
        eng.run_cached(0, cfg.n_blocks, cw, _blob(x[:width, :70].reshape(-1, d)), width, 70,
                       False)
        for j, i in enumerate(range(70, 73)):
            out = eng.run_cached(0, cfg.n_blocks, cw, _blob(x[:width, i]), width, 1,
                                 False).array()
            for r in range(width):
                assert np.array_equal(out[r], single[r][j]), (width, r, i)


@pytest.mark.parametrize("name", ["bloom_int8", "llama_int8"])
def test_decode_attention_streamed_subchunks(name):
    """Decode attention streaming several 128-position sub-chunks per CTA with
    a running online softmax (the MHA/BLOOM launch shape) equals the one-sub-
    chunk-per-CTA launch to f32 rounding, across page and chunk boundaries."""
    from paper_2312_08361_b200 import _lib
    cfg = SMALL[name]
    rng = np.random.default_rng(17)
    d = cfg.hidden_dim
    x = rng.standard_normal((2, 300 + 5, d)).astype(np.float32)
    outs = []
    eng = _engine(cfg)
    _lib.check(eng.lib.sp_span_set_option(eng.span.handle, 7, 0))   # round-1 kernel
    for nsub in (1, 3):
        eng = _engine(cfg)
        _lib.check(eng.lib.sp_span_set_option(eng.span.handle, 5, nsub))
        c = eng.make_caches(0, cfg.n_blocks, 2)
        eng.run_cached(0, cfg.n_blocks, c, _blob(x[:, :300].reshape(-1, d)), 2, 300, False)
        outs.append([eng.run_cached(0, cfg.n_blocks, c, _blob(x[:, i]), 2, 1, False).array()
                     for i in range(300, 305)])
        _lib.check(eng.lib.sp_span_set_option(eng.span.handle, 5, 0))
    _lib.check(eng.lib.sp_span_set_option(eng.span.handle, 7, 1))
    # f32-rounding differences in ctx, seen through the next GEMV's 15-bit
    # activation code (resolution 2^-14 of the row maximum)
    for a, b in zip(*outs):
        assert np.abs(a - b).max() <= 2e-4 * np.abs(b).max()


def test_decode_attention_cluster_merge():
    """70B attention shape (8 query heads per kv head): the DSMEM cluster merge
    (8 and 16 CTAs per kv head) equals the global last-CTA merge to f32
    rounding, below and above 1 K positions and across chunk boundaries."""
    from paper_2312_08361_b200 import _lib
    cfg = SMALL["llama_g8"]
    rng = np.random.default_rng(19)
    d = cfg.hidden_dim
    x = rng.standard_normal((2, 1100 + 4, d)).astype(np.float32)
    outs = {}
    eng = _engine(cfg)
    _lib.check(eng.lib.sp_span_set_option(eng.span.handle, 7, 0))   # round-1 kernel
    try:
        for cl in (-1, 8, 16):
            eng = _engine(cfg)
            _lib.check(eng.lib.sp_span_set_option(eng.span.handle, 6, cl))
            c = eng.make_caches(0, cfg.n_blocks, 2)
            got = [eng.run_cached(0, cfg.n_blocks, c, _blob(x[:, :t0].reshape(-1, d)), 2, t0, False)
                   .array() for t0 in (200,)]
            got += [eng.run_cached(0, cfg.n_blocks, c, _blob(x[:, i]), 2, 1, False).array()
                    for i in range(200, 203)]
            eng.run_cached(0, cfg.n_blocks, c, _blob(x[:, 203:1100].reshape(-1, d)), 2, 897, False)
            got += [eng.run_cached(0, cfg.n_blocks, c, _blob(x[:, i]), 2, 1, False).array()
                    for i in range(1100, 1104)]
            outs[cl] = got
    finally:
        _lib.check(eng.lib.sp_span_set_option(eng.span.handle, 6, -1))
        _lib.check(eng.lib.sp_span_set_option(eng.span.handle, 7, 1))
    for cl in (8, 16):
        for a, b in zip(outs[cl], outs[-1]):
            assert np.abs(a - b).max() <= 2e-4 * np.abs(b).max()


@pytest.mark.parametrize("name,t_pre", [("llama_g8", 70), ("llama_g8", 2040),
                                        ("llama_int8", 300), ("bloom_int8", 130),
                                        ("llama_bf16", 65), ("llama_g8_long", 3300)])
def test_decode_attention_cluster_kernel(name, t_pre):
    """The default decode attention (8-CTA cluster per kv head, every warp
    32 positions in parallel, DSMEM merge: attn_decode_cl.cu) against the
    round-1 kernel (global last-CTA merge, option 7 = 0) and the oracle: the
    new token's K/V append, page boundaries, GQA 8/2/1, ALiBi, bf16 weights, and
    more positions than one pass of the cluster holds (> 3072: two passes)."""
    from paper_2312_08361_b200 import _lib
    cfg = SMALL[name] if name in SMALL else SMALL["llama_g8"].with_(max_seq_len=4096)
    rng = np.random.default_rng(23)
    d = cfg.hidden_dim
    x = rng.standard_normal((t_pre + 3, d)).astype(np.float32)
    outs = {}
    eng = _engine(cfg)
    try:
        for v2 in (1, 0):
            _lib.check(eng.lib.sp_span_set_option(eng.span.handle, 7, v2))
            c = eng.make_caches(0, cfg.n_blocks, 1)
            eng.run_cached(0, cfg.n_blocks, c, _blob(x[:t_pre]), 1, t_pre, False)
            outs[v2] = [eng.run_cached(0, cfg.n_blocks, c, _blob(x[i:i + 1]), 1, 1,
                                       False).array() for i in range(t_pre, t_pre + 3)]
    finally:
        _lib.check(eng.lib.sp_span_set_option(eng.span.handle, 7, 1))
    runner = om.SpanRunner(cfg, 0, cfg.n_blocks)
    runner.step(x[None, :t_pre])
    for j, i in enumerate(range(t_pre, t_pre + 3)):
        w = runner.step(x[None, i:i + 1])[0]
        s = np.abs(w).max()
        e_new, e_old = np.abs(outs[1][j] - w).max() / s, np.abs(outs[0][j] - w).max() / s
        print(f"{name} T={i + 1}: cluster kernel err {e_new:.2e}, round-1 kernel err {e_old:.2e} "
              f"(max-abs / max|y|)")
        assert e_new <= 2e-3
        assert np.abs(outs[1][j] - outs[0][j]).max() <= 2e-3 * s


@pytest.mark.parametrize("name,t_pre", [("bloom_int8", 70), ("bloom_int8", 450),
                                         ("llama_bf16", 300), ("bloom_long", 2040),
                                         ("bloom_long", 4100)])
def test_decode_attention_mha_kernel(name, t_pre):
    """Multi-head decode attention (one query head per kv head: attn_decode_mha.cu,
    option 9) against the MMA / cluster kernels (option 9 off) and the oracle:
    one chunk (T <= 512), 3 and 4 chunks merged by the last CTA, 1024-position
    chunks past 4 K, ALiBi and RoPE, the new token's K/V append."""
    from paper_2312_08361_b200 import _lib
    cfg = SMALL[name] if name in SMALL else SMALL["bloom_int8"].with_(max_seq_len=4608, seed=12)
    rng = np.random.default_rng(29)
    d = cfg.hidden_dim
    x = rng.standard_normal((t_pre + 3, d)).astype(np.float32)
    outs = {}
    eng = _engine(cfg)
    try:
        for v in (1, 0):
            _lib.check(eng.lib.sp_span_set_option(eng.span.handle, 9, v))
            c = eng.make_caches(0, cfg.n_blocks, 1)
            eng.run_cached(0, cfg.n_blocks, c, _blob(x[:t_pre]), 1, t_pre, False)
            outs[v] = [eng.run_cached(0, cfg.n_blocks, c, _blob(x[i:i + 1]), 1, 1,
                                      False).array() for i in range(t_pre, t_pre + 3)]
    finally:
        _lib.check(eng.lib.sp_span_set_option(eng.span.handle, 9, 1))
    runner = om.SpanRunner(cfg, 0, cfg.n_blocks)
    runner.step(x[None, :t_pre])
    for j, i in enumerate(range(t_pre, t_pre + 3)):
        w = runner.step(x[None, i:i + 1])[0]
        s = np.abs(w).max()
        e_new, e_old = np.abs(outs[1][j] - w).max() / s, np.abs(outs[0][j] - w).max() / s
        print(f"{name} T={i + 1}: mha kernel err {e_new:.2e}, mma kernel err {e_old:.2e} "
              f"(max-abs / max|y|)")
        assert e_new <= 2e-3
        assert np.abs(outs[1][j] - outs[0][j]).max() <= 2e-3 * s


def test_decode_attention_mha_batch_rows_independent():
    """The batched MHA decode (many (row, head) pairs per step) gives every row
    exactly what it gets stepped alone (width 8: the widest step whose linears
    run on the decode GEMV; wider steps switch the linears to the tcgen05 GEMM)."""
    cfg = SMALL["bloom_int8"]
    eng = _engine(cfg)
    rng = np.random.default_rng(41)
    d = cfg.hidden_dim
    x = rng.standard_normal((8, 400 + 2, d)).astype(np.float32)
    cw = eng.make_caches(0, cfg.n_blocks, 8)
    eng.run_cached(0, cfg.n_blocks, cw, _blob(x[:, :400].reshape(-1, d)), 8, 400, False)
    outs = [eng.run_cached(0, cfg.n_blocks, cw, _blob(x[:, i]), 8, 1, False).array()
            for i in (400, 401)]
    for r in (0, 3, 7):
        c1 = eng.make_caches(0, cfg.n_blocks, 1)
        eng.run_cached(0, cfg.n_blocks, c1, _blob(x[r, :400]), 1, 400, False)
        for j, i in enumerate((400, 401)):
            one = eng.run_cached(0, cfg.n_blocks, c1, _blob(x[r, i:i + 1]), 1, 1, False).array()
            assert np.array_equal(one[0], outs[j][r]), (r, i)


@pytest.mark.parametrize("name", ["llama_g8", "llama_int8", "bloom_int8", "llama_bf16"])
def test_prefill_attention_tcgen05(name):
    """Prefill / replay attention on tcgen05 + TMEM (attn_prefill_tc.cu, the
    default for bf16 KV, hd 128) against the mma.sync FlashAttention kernel
    with hi/lo Q and P (option 8 off, option 3 on) and the oracle: a 100-token
    prefill then a 200-token chunk on top of the cache (t0 > 0, causal mask
    across the page boundary), ragged last query tile."""
    from paper_2312_08361_b200 import _lib
    cfg = SMALL[name]
    rng = np.random.default_rng(37)
    d = cfg.hidden_dim
    x = rng.standard_normal((300, d)).astype(np.float32)
    outs = {}
    eng = _engine(cfg)
    try:
        for tc in (1, 0):
            _lib.check(eng.lib.sp_span_set_option(eng.span.handle, 8, tc))
            _lib.check(eng.lib.sp_span_set_option(eng.span.handle, 3, 1 - tc))
            c = eng.make_caches(0, cfg.n_blocks, 1)
            a = eng.run_cached(0, cfg.n_blocks, c, _blob(x[:100]), 1, 100, False).array()
            b = eng.run_cached(0, cfg.n_blocks, c, _blob(x[100:]), 1, 200, False).array()
            outs[tc] = np.concatenate([a, b])
    finally:
        _lib.check(eng.lib.sp_span_set_option(eng.span.handle, 8, 1))
        _lib.check(eng.lib.sp_span_set_option(eng.span.handle, 3, 0))
    runner = om.SpanRunner(cfg, 0, cfg.n_blocks)
    want = np.concatenate([runner.step(x[None, :100])[0], runner.step(x[None, 100:])[0]])
    s = np.abs(want).max()
    e_tc = np.abs(outs[1] - want).max() / s
    e_mma = np.abs(outs[0] - want).max() / s
    rel = np.abs(outs[1] - want) / (np.abs(want) + 1e-3 * s)
    print(f"{name} prefill: tcgen05 err {e_tc:.2e}, mma.sync hi/lo err {e_mma:.2e} "
          f"(max-abs / max|y|); tcgen05 per-element relative p99 {np.percentile(rel, 99):.2e}")
    assert e_tc <= 2e-3
    assert np.abs(outs[1] - outs[0]).max() <= 2e-3 * s


def test_bf16_tc_prefill_matches_simt():
    """bf16 weights (Llama-2-7B family) on the tcgen05 GEMM (kind::f16, hi/lo
    bf16 activation planes, f32 accumulation) vs the exact-f32 SIMT GEMM, and
    the micro-batch invariance of T/test_server.py:247-255."""
    from paper_2312_08361_b200 import _lib
    from paper_2312_08361_b200.engine import DeviceSpan, B200ServerEngine
    cfg = SMALL["llama_bf16"]
    span_tc = DeviceSpan(cfg, 0, cfg.n_blocks)
    span_ref = DeviceSpan(cfg, 0, cfg.n_blocks)
    _lib.check(span_ref.lib.sp_span_set_option(span_ref.handle, 0, 0))
    e_tc, e_ref = B200ServerEngine(cfg, span=span_tc), B200ServerEngine(cfg, span=span_ref)
    rng = np.random.default_rng(23)
    x = rng.standard_normal((2 * 150, cfg.hidden_dim)).astype(np.float32)
    a = e_tc.forward(0, cfg.n_blocks, _blob(x), 2, 150, 10**9, None).array()
    b = e_ref.forward(0, cfg.n_blocks, _blob(x), 2, 150, 10**9, None).array()
    rel = np.abs(a - b).max() / np.abs(b).max()
    assert rel < 2e-3, rel
    split = e_tc.forward(0, cfg.n_blocks, _blob(x), 2, 150, 150, None).array()
    assert np.array_equal(a, split)


def test_nf4_decode_rows_independent():
    """nf4 decode GEMV (one row per launch): a width-3 decode equals three
    width-1 sessions bit for bit, and the oracle within the decode tolerance."""
    cfg = SMALL["llama_nf4"]
    eng = _engine(cfg)
    rng = np.random.default_rng(29)
    d = cfg.hidden_dim
    x = rng.standard_normal((3, 40 + 3, d)).astype(np.float32)
    c3 = eng.make_caches(0, cfg.n_blocks, 3)
    eng.run_cached(0, cfg.n_blocks, c3, _blob(x[:, :40].reshape(-1, d)), 3, 40, False)
    wide = [eng.run_cached(0, cfg.n_blocks, c3, _blob(x[:, i]), 3, 1, False).array()
            for i in range(40, 43)]
    for r in range(3):
        c1 = eng.make_caches(0, cfg.n_blocks, 1)
        eng.run_cached(0, cfg.n_blocks, c1, _blob(x[r, :40]), 1, 40, False)
        runner = om.SpanRunner(cfg, 0, cfg.n_blocks)
        runner.step(x[None, r, :40])
        for j, i in enumerate(range(40, 43)):
            one = eng.run_cached(0, cfg.n_blocks, c1, _blob(x[r, i:i + 1]), 1, 1, False).array()
            assert np.array_equal(one[0], wide[j][r])
            w = runner.step(x[None, r, i:i + 1])[0]
            assert np.abs(one - w).max() <= 2e-3 * np.abs(w).max()


@pytest.mark.parametrize("name", ["llama_nf4", "bloom_nf4"])
def test_nf4_tc_prefill_matches_simt(name):
    """nf4 prefill on the tcgen05 GEMM (levels split exactly into two int8
    planes, hi * 128 + lo) vs the exact-f32 SIMT GEMM over the same levels, and
    micro-batch invariance on the tensor-core path."""
    from paper_2312_08361_b200 import _lib
    from paper_2312_08361_b200.engine import DeviceSpan, B200ServerEngine
    cfg = SMALL[name]
    span_tc = DeviceSpan(cfg, 0, cfg.n_blocks)
    span_ref = DeviceSpan(cfg, 0, cfg.n_blocks)
    _lib.check(span_ref.lib.sp_span_set_option(span_ref.handle, 0, 0))
    e_tc, e_ref = B200ServerEngine(cfg, span=span_tc), B200ServerEngine(cfg, span=span_ref)
    rng = np.random.default_rng(31)
    x = rng.standard_normal((2 * 150, cfg.hidden_dim)).astype(np.float32)
    a = e_tc.forward(0, cfg.n_blocks, _blob(x), 2, 150, 10**9, None).array()
    b = e_ref.forward(0, cfg.n_blocks, _blob(x), 2, 150, 10**9, None).array()
    rel = np.abs(a - b).max() / np.abs(b).max()
    assert rel < 2e-3, rel
    split = e_tc.forward(0, cfg.n_blocks, _blob(x), 2, 150, 150, None).array()
    assert np.array_equal(a, split)
