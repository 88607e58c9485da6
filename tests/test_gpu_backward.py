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
