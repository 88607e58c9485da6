"""Device content hash of the span-to-span wire (csrc/hash.cu, relay.py) —
SURVEY.md §8f item 4: the relay checksum of SP/server.py:388-393 / 413-426
computed and verified on the GPU.

Pinned: sp_content_hash equals the CPU restatement (oracle/content_hash.py,
itself pinned power-sum vs Horner in test_oracle.py) for empty, ragged,
unaligned and multi-CTA buffers; sp_content_hash_verify flags a single flipped
bit anywhere in a wire (codes, scales) and nothing else; the flag is sticky."""

import numpy as np
import pytest
import torch

from oracle.content_hash import content_hash

pytestmark = pytest.mark.gpu


def _lib():
    from paper_2312_08361_b200 import _lib
    return _lib.load(), _lib


def _gpu_hash(buf: torch.Tensor, off: int, n: int) -> int:
    lib, L = _lib()
    out = torch.zeros(1, dtype=torch.int64, device=buf.device)
    L.check(lib.sp_content_hash(buf.data_ptr() + off, n, out.data_ptr(),
                                torch.cuda.current_stream().cuda_stream))
    return int(out.item()) & 0xFFFFFFFFFFFFFFFF


@pytest.mark.parametrize("n", [0, 1, 2, 3, 4, 5, 63, 64, 100, 8704, 8712, 65537, 4 * 2048 + 3,
                               (1 << 20) + 3])
def test_content_hash_matches_restatement(n):
    rng = np.random.default_rng(n)
    host = rng.integers(0, 256, n + 8, dtype=np.uint8)
    buf = torch.from_numpy(host).cuda()
    for off in (0, 1, 3) if n < 100000 else (0, 2):
        assert _gpu_hash(buf, off, n) == content_hash(host[off:off + n].tobytes()), (n, off)


def test_content_hash_verify_flags_any_flipped_bit():
    from paper_2312_08361_b200.relay import WireCheck, split_wire, wire_layout
    from paper_2312_08361_b200.errors import ProtocolError
    rows, d = 3, 8192
    payload, off, total = wire_layout(rows, d)
    chk = WireCheck(torch.device("cuda", 0))
    wire = torch.zeros(total, dtype=torch.uint8, device="cuda")
    codes, scales = split_wire(wire, rows, d)
    codes.copy_(torch.randint(-127, 128, (rows * d,), dtype=torch.int8))
    scales.copy_(torch.rand(scales.numel()))
    chk.stamp(wire, payload, off)
    assert int.from_bytes(wire[off:off + 8].cpu().numpy().tobytes(), "little") == \
        content_hash(wire[:payload].cpu().numpy().tobytes())
    chk.verify(wire, payload, off)
    chk.raise_if_mismatch()                                     # clean
    rng = np.random.default_rng(0)
    for pos in list(rng.integers(0, rows * d, 6)) + list(rows * d + rng.integers(0, payload - rows * d, 6)):
        bad = wire.clone()
        bad[int(pos)] ^= 1 << int(rng.integers(0, 8))
        fresh = WireCheck(torch.device("cuda", 0))
        fresh.verify(bad, payload, off)
        with pytest.raises(ProtocolError, match="relay checksum mismatch"):
            fresh.raise_if_mismatch()
        fresh.verify(wire, payload, off)                         # sticky
        with pytest.raises(ProtocolError):
            fresh.raise_if_mismatch()
