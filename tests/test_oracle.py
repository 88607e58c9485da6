"""The oracle is pinned before it is trusted: bit-exact against the
reference's golden vectors (tests/golden/make_golden.py) and, when
/root/reference is importable, against the live reference."""

import json
import os
import sys

import numpy as np
import pytest

from conftest import GOLDEN, REFERENCE_SRC, reference_available
from oracle import codec as oc
from oracle import model as om
from paper_2312_08361_b200.config import SpanConfig, toy


def test_codec_golden_bit_exact(golden_codec):
    keys = sorted({k.split("__")[0] for k in golden_codec.files})
    for k in keys:
        h = golden_codec[f"{k}__in"]
        codes, scales = oc.quantize(h)
        assert np.array_equal(codes, golden_codec[f"{k}__codes"]), k
        assert np.array_equal(scales, golden_codec[f"{k}__scales"]), k
        assert np.array_equal(oc.dequantize(codes, scales, h.shape), golden_codec[f"{k}__deq"]), k


def test_codec_kats():
    """T/test_quantize_wire.py:16-29."""
    codes, scales = oc.quantize(np.zeros((4, 64), np.float32))
    assert (scales == 0).all() and (codes == 0).all()
    h = np.ones(128, np.float32)
    h[7] = 127.0
    codes, scales = oc.quantize(h, block=128)
    assert scales[0] == pytest.approx(1.0)
    assert np.abs(oc.dequantize(codes, scales, h.shape, block=128) - h).max() <= 1.0


@pytest.mark.parametrize("name,cfg", [("default", toy(seed=1)),
                                      ("tiny", SpanConfig(n_blocks=2, hidden_dim=8, n_heads=2,
                                                          vocab_size=16, max_seq_len=64, seed=3))])
def test_toy_weights_and_forward_golden(golden_toy, name, cfg):
    g = golden_toy
    for role in ("wq", "wk", "wv", "wo", "w1", "w2"):
        for b in (0, cfg.n_blocks - 1):
            w = om.init_block(cfg, b)[role]
            assert np.array_equal(w, g[f"{name}__w_{role}_{b}"]), (role, b)
    assert np.array_equal(om.init_embedding(cfg), g[f"{name}__embedding"])
    p0 = om.init_block(cfg, 0)
    for tag in ("prefill", "decode", "fresh"):
        y, kn, vn = om.block_forward_batched(cfg, p0, g[f"{name}__{tag}_x"], g[f"{name}__{tag}_pk"],
                                             g[f"{name}__{tag}_pv"])
        assert np.array_equal(y, g[f"{name}__{tag}_y"]), tag
        assert np.array_equal(kn, g[f"{name}__{tag}_kn"]), tag
        assert np.array_equal(vn, g[f"{name}__{tag}_vn"]), tag
    prefix = [3, 1, 4] if cfg.vocab_size > 4 else [1, 2, 3]
    assert om.reference_generate(cfg, prefix, 32) == list(g[f"{name}__greedy32"])


def test_toy_stack_golden(golden_toy):
    cfg = toy(seed=1)
    r = om.SpanRunner(cfg)
    xs = golden_toy["default__stack_in"]
    outs = [r.step(xs[None, :3])[0]] + [r.step(xs[None, i:i + 1])[0] for i in range(3, 9)]
    assert np.array_equal(np.concatenate(outs), golden_toy["default__stack_out"])


def test_kv_gather_example():
    """T/test_model.py:222-234: new slot i <- old slot idx[i]."""
    cfg = toy(seed=1)
    c = om.KVCache(cfg, 5)
    k = np.arange(5 * 2 * 4 * 16, dtype=np.float32).reshape(5, 2, 4, 16)
    c.append(k, -k)
    c.gather([1, 1, 0, 2, 1])
    for i, j in enumerate([1, 1, 0, 2, 1]):
        assert np.array_equal(c.keys[i], k[j])


def test_extension_families_consistent():
    """Unpinned extensions: stepwise == full prefill (KV-equivalence, the
    property of T/test_model.py:103-135) for llama/bloom restatements."""
    for cfg in (SpanConfig(n_blocks=2, hidden_dim=64, n_heads=4, n_kv_heads=2, ffn_dim=96,
                           family="llama", seed=2, max_seq_len=64),
                SpanConfig(n_blocks=2, hidden_dim=64, n_heads=4, family="bloom", seed=2,
                           max_seq_len=64)):
        rng = np.random.default_rng(0)
        x = rng.standard_normal((1, 9, 64)).astype(np.float32)
        full = om.SpanRunner(cfg).step(x)
        r = om.SpanRunner(cfg)
        step = np.concatenate([r.step(x[:, i:i + 1]) for i in range(9)], axis=1)
        assert np.abs(full - step).max() < 1e-5


def test_int8_weight_rounding_is_codec_per_column():
    rng = np.random.default_rng(1)
    w = rng.uniform(-1, 1, (256, 32)).astype(np.float32)
    codes, scales = om.quantize_columns_int8(w)
    for j in range(32):
        c2, s2 = oc.quantize(w[:, j], block=256)
        assert np.array_equal(codes[j], c2) and scales[j] == s2[0]


@pytest.mark.skipif(not reference_available(), reason="reference not mounted")
def test_live_reference_matches_oracle():
    sys.path.insert(0, REFERENCE_SRC)
    import swarmpipe.model as R
    import swarmpipe.quantize as Q
    rc = R.ModelConfig(seed=4)
    cfg = toy(seed=4)
    blocks, client = R.init_model(rc)
    for b in range(rc.n_blocks):
        p = om.init_block(cfg, b)
        for k in ("wq", "wk", "wv", "wo", "w1", "w2"):
            assert np.array_equal(p[k], getattr(blocks[b], k))
    assert R.reference_generate(rc, [5, 9], 24) == om.reference_generate(cfg, [5, 9], 24)
    rng = np.random.default_rng(9)
    for n in (1, 63, 64, 65, 1000):
        h = (rng.standard_normal(n) * 3).astype(np.float32)
        q = Q.quantize_hidden(h)
        c, s = oc.quantize(h)
        assert np.array_equal(q.codes, c) and np.array_equal(q.scales, s)


def test_swarm_trace_fixture_is_self_consistent():
    with open(os.path.join(GOLDEN, "swarm_traces.json")) as f:
        traces = json.load(f)
    for t in traces:
        # raw stage boundaries reproduce the oracle; int8-coded ones may drift
        # (T/test_acceptance.py:358-371 allows >= 95 % matched-context agreement)
        if not t["quantized"]:
            assert t["tokens"] == t["oracle"]
        for (_, _, tt, nbytes) in t["restore_events"]:
            assert nbytes == tt * 64 * 4


def test_oracle_block_backward_matches_reference_golden():
    """oracle.block_backward restates SP/model.py:320-381 bit for bit
    (golden vectors from the reference, tests/golden/backward.npz)."""
    g = np.load(os.path.join(GOLDEN, "backward.npz"))
    cfg = toy(seed=1)
    for b in (0, 5):
        got = om.block_backward(cfg, om.init_block(cfg, b), g["block_x"], g["block_dy"])
        assert np.array_equal(got, g[f"block{b}_dx"])


def test_oracle_span_forward_backward_matches_reference_golden():
    """forward(record) with whole-sequence micro-batches then backward block by
    block in reverse (SP/server.py:106-139), on the oracle."""
    g = np.load(os.path.join(GOLDEN, "backward.npz"))
    cfg = toy(seed=1)
    d, batch, tokens = cfg.hidden_dim, 3, 6
    x = g["span_x"].reshape(batch, tokens, d)
    gr = g["span_g"].reshape(batch, tokens, d)
    blocks = {b: om.init_block(cfg, b) for b in range(2, 6)}
    tables = om.Tables(cfg)
    per_chunk = max(1, 12 // tokens)
    ys, dxs = [], []
    for lo in range(0, batch, per_chunk):
        h = x[lo:lo + per_chunk]
        rec = []
        for b in range(2, 6):
            rec.append(h)
            empty = np.zeros((h.shape[0], 0, cfg.kv_heads, cfg.head_dim), np.float32)
            h, _, _ = om.block_forward_batched(cfg, blocks[b], h, empty, empty, tables)
        ys.append(h)
        gc = gr[lo:lo + per_chunk]
        for i, b in enumerate(reversed(range(2, 6))):
            gc = om.block_backward(cfg, blocks[b], rec[len(rec) - 1 - i], gc)
        dxs.append(gc)
    assert np.array_equal(np.concatenate(ys).reshape(-1, d), g["span_y"])
    assert np.array_equal(np.concatenate(dxs).reshape(-1, d), g["span_dx"])


def test_nf4_format_properties():
    """The nf4 weight format (oracle/model.py quantize_columns_nf4; builder's
    format, parity unpinned): 4-bit codes, uint8 block scales, all-zero
    channels and blocks map to the zero level, and every weight lands on the
    nearest level of its block (|w - w_eff| <= half the widest level gap)."""
    from oracle import model as om
    rng = np.random.default_rng(3)
    w = rng.standard_normal((256, 96)).astype(np.float32)
    w[:, 5] = 0.0                                  # an all-zero channel
    w[64:128, 7] = 0.0                             # an all-zero block
    codes, q, s = om.quantize_columns_nf4(w)
    assert codes.shape == (96, 256) and q.shape == (96, 4) and s.shape == (96,)
    assert codes.max() <= 15 and q.max() == 255
    assert (codes[5] == om.NF4_ZERO).all() and s[5] == 0
    assert q[7, 1] == 0 and (codes[7, 64:128] == om.NF4_ZERO).all()

    class C:
        weight_dtype = "nf4"
    eff = om.effective_weight(C, w)
    assert (eff[:, 5] == 0).all() and (eff[64:128, 7] == 0).all()
    gap = np.diff(om.CB7).max() / 2 + 0.5           # levels in units of q * s, + rounding
    bound = (gap * np.repeat(q.astype(np.float32), 64, axis=1) * s[:, None]).T
    assert (np.abs(eff - w) <= bound * 1.0001 + 1e-12).all()
    assert list(om.CB7) == [-63, -44, -33, -25, -18, -12, -6, 0, 5, 10, 16, 21, 28, 35, 46, 63]


def test_content_hash_restatement_forms_agree():
    """oracle/content_hash.py: the power-sum form (the GPU's decomposition) equals
    Horner's rule; length is part of the hash (zero padding is not a collision);
    FNV-1a 64 restatement equals the reference vectors (SP/wire.py:39-44)."""
    import os
    from oracle.content_hash import content_hash, content_hash_horner, fnv1a64
    for n in (0, 1, 3, 4, 5, 17, 64, 1000):
        d = os.urandom(n)
        assert content_hash(d) == content_hash_horner(d)
    assert content_hash(b"\0") != content_hash(b"\0\0") != content_hash(b"")
    assert fnv1a64(b"") == 0xCBF29CE484222325
    assert fnv1a64(b"a") == 0xAF63DC4C8601EC8C
