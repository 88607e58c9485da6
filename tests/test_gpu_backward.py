"""Prompt-tuning backward on the GPU: `block_backward`
(SP/model.py:320-381) and the engine protocol's `backward`
(SP/server.py:127-139), float64 recompute like the reference.

Pinned against golden vectors produced by the reference itself
(tests/golden/make_golden.py: backward.npz) and, through the reference's own
FinetuneSession/BlockServer with the GPU engine plugged in, against the
reference engine's soft-prompt gradient."""

import os
import sys

import numpy as np
import pytest

from conftest import GOLDEN, ROOT

pytestmark = pytest.mark.gpu
G = np.load(os.path.join(GOLDEN, "backward.npz"))


def _blob(a):
    from paper_2312_08361_b200.blob import HiddenBlob
    return HiddenBlob.from_array(a)


def test_block_backward_matches_reference_golden():
    import torch
    from paper_2312_08361_b200 import _lib
    from paper_2312_08361_b200.config import toy
    from paper_2312_08361_b200.engine import B200ServerEngine
    eng = B200ServerEngine(toy(seed=1))
    x = torch.from_numpy(G["block_x"].reshape(14, 64)).cuda()
    dy = torch.from_numpy(G["block_dy"].reshape(14, 64)).cuda()
    for b in (0, 5):
        dx = torch.empty_like(x)
        _lib.check(eng.lib.sp_span_block_backward(eng.span.handle, b, x.data_ptr(), dy.data_ptr(),
                                                  dx.data_ptr(), 2, 7, 0))
        torch.cuda.synchronize()
        want = G[f"block{b}_dx"].reshape(14, 64)
        got = dx.cpu().numpy()
        # float64 on both sides, rounded to f32 once: at most an ulp apart
        assert np.abs(got - want).max() <= 1e-6 * np.abs(want).max()


def test_span_forward_record_backward_matches_reference_golden():
    """RealServerEngine.forward(record) + backward over blocks [2, 6) with
    micro-batches of 12 tokens (whole 6-token sequences, SP/server.py:189-194)."""
    from paper_2312_08361_b200.config import toy
    from paper_2312_08361_b200.engine import B200ServerEngine
    eng = B200ServerEngine(toy(seed=1))
    record: list = []
    y = eng.forward(2, 6, _blob(G["span_x"]), 3, 6, 12, record)
    assert np.abs(y.array() - G["span_y"]).max() < 1e-5
    dx = eng.backward(2, 6, _blob(G["span_g"]), 3, 6, record).array()
    want = G["span_dx"]
    assert np.abs(dx - want).max() <= 1e-5 * np.abs(want).max()


def test_backward_rejects_other_families():
    """block_backward is the reference's, defined for its own family only
    (SP/model.py:320): a recording forward on another family is refused up
    front (its records could never be used), and the C ABI refuses the backward."""
    import ctypes
    import torch
    from paper_2312_08361_b200._lib import SpanPipeError, check
    from paper_2312_08361_b200.config import SpanConfig
    from paper_2312_08361_b200.engine import B200ServerEngine
    from paper_2312_08361_b200.errors import ProtocolError
    cfg = SpanConfig(n_blocks=2, hidden_dim=512, n_heads=4, n_kv_heads=2, ffn_dim=1024,
                     vocab_size=64, max_seq_len=256, family="llama", weight_dtype="int8",
                     kv_dtype="bf16", seed=5)
    eng = B200ServerEngine(cfg)
    x = np.ones((4, 512), np.float32)
    with pytest.raises(ProtocolError):
        eng.forward(0, 2, _blob(x), 1, 4, 10**9, [])
    eng.forward(0, 2, _blob(x), 1, 4, 10**9, None)           # non-recording is fine
    xd = torch.ones((4, 512), device="cuda")
    with pytest.raises(SpanPipeError):
        check(eng.lib.sp_span_block_backward(eng.span.handle, 0, xd.data_ptr(), xd.data_ptr(),
                                             xd.data_ptr(), 1, 4, ctypes.c_void_p(0)))


def test_dropin_finetune_session(swarmpipe):
    """The reference's own FinetuneSession over its own swarm, every server's
    engine the B200 engine: the soft-prompt and head gradients of one pass equal
    the reference engine's, and the copy task's loss decreases."""
    import swarmpipe.server
    import swarmpipe.swarm
    from swarmpipe.client import FinetuneSession
    from swarmpipe.model import ModelConfig
    from paper_2312_08361_b200.engine import B200ServerEngine
    cfg = ModelConfig(seed=1)
    rng = np.random.default_rng(0)
    batch = rng.integers(0, 256, (3, 4))
    labels = (batch[:, -1] % 8).astype(np.intp)

    def one_pass():
        swarm = swarmpipe.swarm.build_sim_swarm(cfg, seed=0)
        ft = FinetuneSession(swarm.client(), n_labels=8, prompt_len=2, lr=0.0, init_seed=1)
        return ft._one_pass(batch, labels, req_id=999)

    loss_ref, gp_ref, gh_ref = one_pass()                       # reference CPU engine
    orig = swarmpipe.swarm.RealServerEngine
    swarmpipe.swarm.RealServerEngine = B200ServerEngine
    swarmpipe.server.RealServerEngine = B200ServerEngine
    try:
        loss, gp, gh = one_pass()
        assert abs(loss - loss_ref) <= 1e-5 * abs(loss_ref)
        assert np.abs(gp - gp_ref).max() <= 1e-4 * np.abs(gp_ref).max()
        assert np.abs(gh - gh_ref).max() <= 1e-4 * np.abs(gh_ref).max()
        swarm = swarmpipe.swarm.build_sim_swarm(cfg, seed=0)
        ft = FinetuneSession(swarm.client(), n_labels=8, prompt_len=4, lr=0.3, init_seed=0)
        r2 = np.random.default_rng(0)
        b2 = r2.integers(0, 256, (24, 6))
        l2 = (b2[:, -1] % 8).astype(np.intp)
        for _ in range(30):
            ft.step(b2, l2)
        assert ft.loss_curve[-1] < ft.loss_curve[0]
    finally:
        swarmpipe.swarm.RealServerEngine = orig
        swarmpipe.server.RealServerEngine = orig


def _gpu_block_backward(eng, b, x, dy):
    """sp_span_block_backward on [batch, t, d] f32 arrays -> dx (numpy)."""
    import torch
    from paper_2312_08361_b200 import _lib
    batch, t, d = x.shape
    xd = torch.from_numpy(np.ascontiguousarray(x.reshape(-1, d))).cuda()
    dyd = torch.from_numpy(np.ascontiguousarray(dy.reshape(-1, d))).cuda()
    dx = torch.empty_like(xd)
    _lib.check(eng.lib.sp_span_block_backward(eng.span.handle, b, xd.data_ptr(), dyd.data_ptr(),
                                              dx.data_ptr(), batch, t, 0))
    torch.cuda.synchronize()
    return dx.cpu().numpy().reshape(batch, t, d)


def test_block_backward_zero_grad_out():
    """T/test_model.py:151-156: a zero output gradient gives exactly zero."""
    from paper_2312_08361_b200.config import toy
    from paper_2312_08361_b200.engine import B200ServerEngine
    eng = B200ServerEngine(toy(seed=3))
    x = np.random.default_rng(0).standard_normal((2, 4, 64)).astype(np.float32)
    dx = _gpu_block_backward(eng, 1, x, np.zeros_like(x))
    assert not dx.any()


def test_block_backward_params_untouched():
    """T/test_model.py:158-164: the backward only reads the block's weights."""
    from paper_2312_08361_b200.config import toy
    from paper_2312_08361_b200.engine import B200ServerEngine
    cfg = toy(seed=3)
    eng = B200ServerEngine(cfg)
    roles = [r for r, _, _ in cfg.block_matrices()]
    before = {r: eng.span.read_weight(0, r).copy() for r in roles}
    rng = np.random.default_rng(1)
    x = rng.standard_normal((1, 6, 64)).astype(np.float32)
    _gpu_block_backward(eng, 0, x, rng.standard_normal(x.shape).astype(np.float32))
    for r in roles:
        assert np.array_equal(eng.span.read_weight(0, r), before[r]), r


def _forward_f64(p, x, n_heads):
    """The toy block (SP/model.py:244-280) in float64 on [1, t, d] — the
    finite-difference loss of T/test_model.py:166-192."""
    import oracle.model as om
    f8 = {k: np.asarray(v, np.float64) for k, v in p.items()}
    t, d = x.shape[1], x.shape[2]
    hd = d // n_heads
    h = om.ln(x, f8["ln1_g"], f8["ln1_b"])
    q, k, v = (om._split_heads(h @ f8[w], n_heads) for w in ("wq", "wk", "wv"))
    s = np.einsum("bhid,bhjd->bhij", q, k) / np.sqrt(hd)
    s = np.where(np.triu(np.ones((t, t), bool), 1), -1e30, s)
    e = np.exp(s - s.max(axis=-1, keepdims=True))
    x1 = x + om._merge_heads((e / e.sum(axis=-1, keepdims=True)) @ v) @ f8["wo"]
    return x1 + om.gelu(om.ln(x1, f8["ln2_g"], f8["ln2_b"]) @ f8["w1"]) @ f8["w2"]


def test_block_backward_matches_finite_differences():
    """T/test_model.py:166-192: the GPU gradient against central differences
    (eps 1e-3) of a float64 forward, worst relative error <= 1e-4 over trials."""
    sys.path.insert(0, ROOT)
    import oracle.model as om
    from paper_2312_08361_b200.config import toy
    from paper_2312_08361_b200.engine import B200ServerEngine
    eps, worst = 1e-3, 0.0
    for trial in range(4):
        cfg = toy(seed=trial, n_blocks=1)
        eng = B200ServerEngine(cfg)
        p = om.init_block(cfg, 0)
        rng = np.random.default_rng(100 + trial)
        x = rng.standard_normal((1, 4, 64)).astype(np.float32)
        gy = rng.standard_normal((1, 4, 64)).astype(np.float32)
        got = _gpu_block_backward(eng, 0, x, gy)
        g8 = gy.astype(np.float64)
        fd = np.zeros(x.shape)
        for i in range(4):
            for j in range(64):
                up = x.astype(np.float64)
                dn = up.copy()
                up[0, i, j] += eps
                dn[0, i, j] -= eps
                fd[0, i, j] = ((g8 * _forward_f64(p, up, cfg.n_heads)).sum()
                               - (g8 * _forward_f64(p, dn, cfg.n_heads)).sum()) / (2 * eps)
        worst = max(worst, np.abs(got - fd).max() / max(np.abs(fd).max(), 1e-12))
    print(f"worst relative gradient error vs finite differences {worst:.3g}")
    assert worst <= 1e-4, worst
