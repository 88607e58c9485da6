"""Error behaviour of the C ABI on the GPU (the engine raises
ProtocolError-class errors, the ABI returns status codes): every rejected call
leaves the span and its sessions usable, and a session continues bit-exactly
after the rejected call."""

import subprocess
import sys
import textwrap

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_rejected_calls_leave_state_intact():
    from paper_2312_08361_b200._lib import SpanPipeError
    from paper_2312_08361_b200.blob import HiddenBlob
    from paper_2312_08361_b200.config import toy
    from paper_2312_08361_b200.engine import B200ServerEngine
    from paper_2312_08361_b200.errors import ProtocolError
    cfg = toy(seed=1)
    eng = B200ServerEngine(cfg)
    rng = np.random.default_rng(0)
    x = rng.standard_normal((4, cfg.hidden_dim)).astype(np.float32)
    ref = eng.make_caches(0, 8, 1)
    want = [eng.run_cached(0, 8, ref, HiddenBlob.from_array(x[i:i + 1]), 1, 1, False).array()
            for i in range(4)]
    c = eng.make_caches(0, 8, 1)
    got = [eng.run_cached(0, 8, c, HiddenBlob.from_array(x[:1]), 1, 1, False).array()]
    with pytest.raises((SpanPipeError, ProtocolError)):            # width mismatch
        eng.run_cached(0, 8, c, HiddenBlob.from_array(x[:2]), 2, 1, False)
    with pytest.raises((SpanPipeError, ProtocolError)):            # beyond max_seq_len
        eng.run_cached(0, 8, c, HiddenBlob.from_array(
            np.zeros((cfg.max_seq_len, cfg.hidden_dim), np.float32)), 1, cfg.max_seq_len, False)
    with pytest.raises((SpanPipeError, ProtocolError)):            # reorder out of range
        eng.reorder(c, [3])
    assert eng.cache_length(c) == 1
    for i in range(1, 4):
        got.append(eng.run_cached(0, 8, c, HiddenBlob.from_array(x[i:i + 1]), 1, 1, False).array())
    for g, w in zip(got, want):
        assert np.array_equal(g, w)


def test_process_exits_cleanly_after_errors():
    """A fresh interpreter that hits rejected calls and then exits with live
    sessions and spans must not corrupt the heap on teardown."""
    code = textwrap.dedent("""
        import numpy as np
        from paper_2312_08361_b200.blob import HiddenBlob
        from paper_2312_08361_b200.config import SpanConfig
        from paper_2312_08361_b200.engine import B200ServerEngine
        cfg = SpanConfig(n_blocks=2, hidden_dim=512, n_heads=4, n_kv_heads=2, ffn_dim=1024,
                         vocab_size=64, max_seq_len=256, family="llama", weight_dtype="int8",
                         kv_dtype="bf16", seed=5)
        eng = B200ServerEngine(cfg)
        c = eng.make_caches(0, 2, 1)
        x = np.ones((200, 512), np.float32)
        eng.run_cached(0, 2, c, HiddenBlob.from_array(x), 1, 200, False)
        for bad in ((x, 1, 200), (x[:2], 2, 1)):
            try:
                eng.run_cached(0, 2, c, HiddenBlob.from_array(bad[0]), bad[1], bad[2], False)
            except Exception:
                pass
        keep = [eng.make_caches(0, 2, 3) for _ in range(3)]
        y = eng.run_cached(0, 2, c, HiddenBlob.from_array(x[:1]), 1, 1, True)
        print("ok", y.array().shape)
    """)
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "ok (1, 512)" in r.stdout
