"""GPU hidden-state codec vs the reference's golden vectors and the oracle —
bit-exact codes, scales and dequantised values (SP/quantize.py:36-58)."""

import numpy as np
import pytest

from oracle import codec as ocodec

pytestmark = pytest.mark.gpu


def _gpu_roundtrip(h):
    import torch
    from paper_2312_08361_b200 import codec
    x = torch.from_numpy(np.ascontiguousarray(h, np.float32).ravel()).cuda()
    c, s = codec.quantize_device(x)
    back = codec.dequantize_device(c, s, x.numel())
    torch.cuda.synchronize()
    return c.cpu().numpy(), s.cpu().numpy(), back.cpu().numpy().reshape(np.shape(h))


def test_golden_vectors_bit_exact(golden_codec):
    keys = sorted({k.split("__")[0] for k in golden_codec.files})
    assert len(keys) >= 12
    for k in keys:
        h = golden_codec[f"{k}__in"]
        c, s, back = _gpu_roundtrip(h)
        assert np.array_equal(c, golden_codec[f"{k}__codes"]), k
        assert np.array_equal(s.view(np.uint32), golden_codec[f"{k}__scales"].view(np.uint32)), k
        assert np.array_equal(back.view(np.uint32),
                              golden_codec[f"{k}__deq"].astype(np.float32).view(np.uint32)), k


@pytest.mark.parametrize("d", [64, 4096, 8192, 14336])
@pytest.mark.parametrize("rows", [1, 3, 16])
def test_hidden_widths_vs_oracle(d, rows):
    rng = np.random.default_rng(d * 31 + rows)
    h = (rng.standard_normal((rows, d)) * rng.uniform(0.1, 30)).astype(np.float32)
    h[0, :64] = 0.0                      # a scale-0 block
    c, s, back = _gpu_roundtrip(h)
    oc, os_ = ocodec.quantize(h)
    assert np.array_equal(c, oc)
    assert np.array_equal(s, os_)
    assert np.array_equal(back, ocodec.dequantize(oc, os_, h.shape))


def test_ragged_lengths_and_bound():
    # T/test_quantize_wire.py:45-58 property, sizes 1..300
    for n in list(range(1, 70)) + [127, 128, 129, 255, 300, 1000, 4097]:
        h = np.random.default_rng(n).uniform(-50, 50, n).astype(np.float32)
        c, s, back = _gpu_roundtrip(h)
        oc, os_ = ocodec.quantize(h)
        assert np.array_equal(c, oc) and np.array_equal(s, os_), n
        padded = np.zeros(s.size * 64, np.float32)
        padded[:n] = h
        bounds = np.abs(padded.reshape(-1, 64)).max(1) / 127.0
        err = np.abs(back - h)
        for b in range(s.size):
            lo, hi = b * 64, min((b + 1) * 64, n)
            assert err[lo:hi].max() <= bounds[b] + 1e-6


def test_requantize_idempotent():
    """relaying codes == re-quantising the dequantised rows."""
    rng = np.random.default_rng(7)
    h = (rng.standard_normal((4, 8192)) * 5).astype(np.float32)
    c, s, back = _gpu_roundtrip(h)
    c2, s2, _ = _gpu_roundtrip(back)
    assert np.array_equal(c, c2) and np.array_equal(s, s2)


def test_large_roundtrip_size_independent():
    """Full-size property check (no oracle needed): 64M elements."""
    import torch
    from paper_2312_08361_b200 import codec
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randn(64 << 20, device="cuda", generator=g) * 7
    c, s = codec.quantize_device(x)
    back = codec.dequantize_device(c, s, x.numel())
    c2, s2 = codec.quantize_device(back)
    assert torch.equal(c, c2) and torch.equal(s, s2)
    bound = (s / 1.0).repeat_interleave(64)[: x.numel()]
    assert bool(((back - x).abs() <= bound * 0.501 + 1e-6).all())


def test_array_async_equals_array():
    """HiddenBlob.array_async (pinned, non-blocking device->host read) returns
    exactly what array() returns, for raw and int8-coded device blobs."""
    import torch
    from paper_2312_08361_b200 import codec
    from paper_2312_08361_b200.blob import HiddenBlob
    rng = np.random.default_rng(5)
    x = torch.from_numpy(rng.standard_normal((3, 8192)).astype(np.float32)).cuda()
    raw = HiddenBlob.from_device(x)
    assert np.array_equal(raw.array_async().result(), x.cpu().numpy())
    c, s = codec.quantize_device(x)
    coded = HiddenBlob(3, 8192, dev_codes=c, dev_scales=s)
    assert np.array_equal(coded.array_async().result(), coded.array())
