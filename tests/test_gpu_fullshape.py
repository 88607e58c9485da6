"""One block at the BASELINE shapes themselves (Llama-2-70B int8 and
nf4, BLOOM-176B int8, Llama-2-7B bf16), checked against the oracle's block forward
(SP/model.py:244-280 restated) on the weights the GPU generated — whose bit-exactness
against the reference recipe is pinned at small shapes (tests/test_gpu_weights.py) —
plus batch invariance of the decode path at full width."""

import numpy as np
import pytest

from oracle import model as om

pytestmark = pytest.mark.gpu


def _cfg(name):
    from paper_2312_08361_b200.config import bloom_176b, llama2_7b, llama2_70b
    return {"llama2-70b-int8": lambda: llama2_70b(n_blocks=1),
            "llama2-70b-nf4": lambda: llama2_70b(n_blocks=1, weight_dtype="nf4"),
            "bloom-176b-int8": lambda: bloom_176b(n_blocks=1),
            "llama2-7b-bf16": lambda: llama2_7b(n_blocks=1)}[name]()


def _blob(a):
    from paper_2312_08361_b200.blob import HiddenBlob
    return HiddenBlob.from_array(np.ascontiguousarray(a, dtype=np.float32))


@pytest.mark.parametrize("name", ["llama2-70b-int8", "llama2-70b-nf4", "bloom-176b-int8",
                                  "llama2-7b-bf16"])
def test_full_shape_block_vs_oracle(name):
    from paper_2312_08361_b200.engine import B200ServerEngine, DeviceSpan
    cfg = _cfg(name)
    span = DeviceSpan(cfg, 0, 1, kv_pool_tokens=4096)
    eng = B200ServerEngine(cfg, span=span)
    d = cfg.hidden_dim
    p = {role: span.read_weight(0, role) for role, _, _ in cfg.block_matrices()}
    p.update(ln1_g=np.ones(d, np.float32), ln1_b=np.zeros(d, np.float32),
             ln2_g=np.ones(d, np.float32), ln2_b=np.zeros(d, np.float32))
    runner = om.SpanRunner(cfg, 0, 1, blocks={0: p})
    rng = np.random.default_rng(41)
    t_pre, n_dec = 40, 3
    x = rng.standard_normal((t_pre + n_dec, d)).astype(np.float32)
    c = eng.make_caches(0, 1, 1)
    got = eng.run_cached(0, 1, c, _blob(x[:t_pre]), 1, t_pre, False).array()
    want = runner.step(x[None, :t_pre])[0]
    s = np.abs(want).max()
    e_pre = np.abs(got - want).max() / s
    e_dec = []
    for i in range(t_pre, t_pre + n_dec):
        g = eng.run_cached(0, 1, c, _blob(x[i:i + 1]), 1, 1, False).array()
        w = runner.step(x[None, i:i + 1])[0]
        e_dec.append(np.abs(g - w).max() / np.abs(w).max())
    print(f"{name}: prefill err {e_pre:.2e}, decode err max {max(e_dec):.2e} (max-abs / max|y|)")
    assert e_pre <= 2e-3
    assert max(e_dec) <= 2e-3


def test_full_shape_decode_rows_independent():
    """70B int8 block: a width-2 decode equals two width-1 decodes bit for bit
    (exact integer GEMV partials, fixed-order merges; one 15-bit activation code
    for every width)."""
    from paper_2312_08361_b200.engine import B200ServerEngine, DeviceSpan
    cfg = _cfg("llama2-70b-int8")
    eng = B200ServerEngine(cfg, span=DeviceSpan(cfg, 0, 1, kv_pool_tokens=4096))
    d = cfg.hidden_dim
    rng = np.random.default_rng(43)
    x = rng.standard_normal((2, 33, d)).astype(np.float32)
    c2 = eng.make_caches(0, 1, 2)
    eng.run_cached(0, 1, c2, _blob(x[:, :32].reshape(-1, d)), 2, 32, False)
    wide = eng.run_cached(0, 1, c2, _blob(x[:, 32]), 2, 1, False).array()
    for r in range(2):
        c1 = eng.make_caches(0, 1, 1)
        eng.run_cached(0, 1, c1, _blob(x[r, :32]), 1, 32, False)
        one = eng.run_cached(0, 1, c1, _blob(x[r, 32:33]), 1, 1, False).array()
        assert np.array_equal(one[0], wide[r])
