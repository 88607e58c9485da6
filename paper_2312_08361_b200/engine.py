"""B200ServerEngine — the drop-in for the reference's server payload engine.

Implements the engine protocol that `BlockServer` calls (`SP/server.py:77-142`,
SURVEY.md §8b): ``config``, ``blocks``, ``make_caches``, ``cache_length``,
``run_cached``, ``reorder``, ``forward``, ``backward``, ``blob_checksum``.
Every arithmetic step runs in libspanpipe.so on the GPU; Python only moves
pointers.  There is no CPU fallback: constructing an engine without a GPU or
without the built library raises.
"""

from __future__ import annotations

import ctypes
import threading

import numpy as np
import torch

from . import _lib
from .blob import HiddenBlob
from .config import SpanConfig, from_reference
from .errors import ProtocolError

_SPANS: dict = {}
_SPANS_LOCK = threading.Lock()

# role ids of SP/model.py:32-37 (+13 = SwiGLU up-projection)
_ROLE_IDS = {"wq": 1, "wk": 2, "wv": 3, "wo": 4, "w1": 5, "w2": 6, "w3": 13}


def _stream(device: torch.device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def default_pool_tokens(cfg: SpanConfig, n_blocks: int) -> int:
    """KV pool capacity in positions: 4 GiB of pages, at least 64 full sessions
    for small models."""
    elt = 2 if cfg.kv_dtype == "bf16" else 4
    per_tok = 2 * cfg.kv_heads * cfg.head_dim * elt * max(1, n_blocks)
    tokens = (4 << 30) // per_tok
    return int(max(4096, min(tokens, 64 * cfg.max_seq_len)))


class DeviceSpan:
    """Weights of blocks [start, end) generated on one GPU (bit-identical to
    the reference recipe) plus the span's paged KV pool."""

    def __init__(self, cfg: SpanConfig, start: int = 0, end: int | None = None, device: int = 0,
                 kv_pool_tokens: int | None = None):
        if not torch.cuda.is_available():
            raise RuntimeError("B200 span engine needs a CUDA device (no CPU fallback)")
        self.lib = _lib.load()
        self.cfg = cfg
        self.start = start
        self.end = cfg.n_blocks if end is None else end
        self.device = torch.device("cuda", device)
        self.kv_pool_tokens = kv_pool_tokens or default_pool_tokens(cfg, self.end - self.start)
        self._c = _lib.make_config(cfg)
        h = ctypes.c_void_p()
        _lib.check(self.lib.sp_span_create(ctypes.byref(self._c), self.start, self.end, device,
                                           self.kv_pool_tokens, ctypes.byref(h)))
        self.handle = h

    def __del__(self):
        h = getattr(self, "handle", None)
        if h and h.value:
            try:
                self.lib.sp_span_destroy(h)
            except Exception:
                pass
            self.handle = None

    @property
    def weight_bytes(self) -> int:
        return int(self.lib.sp_span_weight_bytes(self.handle))

    @property
    def free_pages(self) -> int:
        return int(self.lib.sp_span_free_pages(self.handle))

    def read_weight(self, block: int, role: str) -> np.ndarray:
        """Effective f32 weight [d_in, d_out] of (block, role) — test access."""
        mats = {r: (a, b) for r, a, b in self.cfg.block_matrices()}
        a, b = mats[role]
        out = np.empty((a, b), np.float32)
        _lib.check(self.lib.sp_span_read_weight(self.handle, block, _ROLE_IDS[role],
                                                out.ctypes.data))
        return out


def shared_span(cfg: SpanConfig, device: int = 0, kv_pool_tokens: int | None = None) -> DeviceSpan:
    """One full-model span per (config, device) per process — the analogue of
    the shared `init_model` blocks of SP/swarm.py:72-74."""
    key = (cfg, device, kv_pool_tokens)
    with _SPANS_LOCK:
        sp = _SPANS.get(key)
        if sp is None:
            sp = _SPANS[key] = DeviceSpan(cfg, 0, cfg.n_blocks, device, kv_pool_tokens)
        return sp


def release_shared_spans() -> None:
    with _SPANS_LOCK:
        _SPANS.clear()


class _BlockView:
    """`BlockParams`-like view (`SP/model.py:89-115`): ``arrays()`` reads the
    effective weights back from the GPU in the reference order."""

    def __init__(self, span: DeviceSpan, block: int):
        self.span, self.block = span, block

    def arrays(self) -> list[np.ndarray]:
        cfg = self.span.cfg
        roles = [r for r, _, _ in cfg.block_matrices()]
        order = [r for r in ("wq", "wk", "wv", "wo", "w1", "w2", "w3") if r in roles]
        d = cfg.hidden_dim
        out = [self.span.read_weight(self.block, r) for r in order]
        out += [np.ones(d, np.float32), np.zeros(d, np.float32),
                np.ones(d, np.float32), np.zeros(d, np.float32)]
        return out

    def n_params(self) -> int:
        return self.span.cfg.block_params()


class _BlockCache:
    """Per-block `KVCache` view (`SP/model.py:139-175`) of a span session."""

    def __init__(self, caches: "SpanCaches", block: int):
        self._c, self.block = caches, block

    @property
    def length(self) -> int:
        return self._c.length

    @property
    def width(self) -> int:
        return self._c.width

    def _read(self):
        cfg = self._c.span.cfg
        t, w = self.length, self.width
        k = np.zeros((w, t, cfg.kv_heads, cfg.head_dim), np.float32)
        v = np.zeros_like(k)
        for s in range(w):
            if t:
                _lib.check(self._c.lib.sp_kv_read(self._c.handle, self.block, s,
                                                  k[s].ctypes.data, v[s].ctypes.data))
        return k, v

    @property
    def keys(self) -> np.ndarray:
        return self._read()[0]

    @property
    def values(self) -> np.ndarray:
        return self._read()[1]


class SpanCaches:
    """The opaque `caches` object of one session over blocks [start, end):
    a paged KV allocation in the span's pool (list-like of per-block views)."""

    def __init__(self, span: DeviceSpan, start: int, end: int, width: int):
        self.span, self.lib = span, span.lib
        self.start, self.end = start, end
        h = ctypes.c_void_p()
        _lib.check(self.lib.sp_kv_create(span.handle, width, ctypes.byref(h)))
        self.handle = h

    def __del__(self):
        h = getattr(self, "handle", None)
        if h and h.value:
            try:
                self.lib.sp_kv_destroy(h)
            except Exception:
                pass
            self.handle = None

    @property
    def length(self) -> int:
        return int(self.lib.sp_kv_length(self.handle))

    @property
    def width(self) -> int:
        return int(self.lib.sp_kv_width(self.handle))

    def __len__(self) -> int:
        return self.end - self.start

    def __getitem__(self, i: int) -> _BlockCache:
        n = len(self)
        if i < 0:
            i += n
        if not 0 <= i < n:
            raise IndexError(i)
        return _BlockCache(self, self.start + i)

    def __iter__(self):
        return (self[i] for i in range(len(self)))


class B200ServerEngine:
    """GPU payload engine with the reference engine protocol."""

    def __init__(self, config, blocks=None, *, device: int = 0, kv_pool_tokens: int | None = None,
                 span: DeviceSpan | None = None):
        self.config = from_reference(config)
        if span is None and isinstance(blocks, _BlockList):
            span = blocks.span
        # `blocks` from the reference (numpy BlockParams) are regenerated on the
        # GPU bit-identically from the seed; they are not uploaded.
        self.span = span or shared_span(self.config, device, kv_pool_tokens)
        self.device = self.span.device
        self.lib = self.span.lib
        self.blocks = _BlockList(self.span)
        # stateless forward chunk (tokens): see device_micro_batches
        self.stateless_tokens = min(2048, self.span.kv_pool_tokens // 2)
        self.last_forward_chunks = 0
        self._staging = []            # pinned host slots for row uploads: [tensor, event]
        self._stage_next = 0
        # block_backward exists for the reference's own family only (SP/model.py:320)
        c = self.config
        self.backward_defined = (c.family == "toy" and c.weight_dtype == "f32"
                                 and c.kv_heads == c.n_heads)

    # -- sessions ---------------------------------------------------------------
    def make_caches(self, start: int, end: int, width: int) -> SpanCaches:
        return SpanCaches(self.span, start, end, width)

    def cache_length(self, caches: SpanCaches) -> int:
        return caches.length

    # -- the hot path ------------------------------------------------------------
    def _input_ptrs(self, blob: HiddenBlob, rows: int):
        """(x_ptr, codes_ptr, scales_ptr, keepalive) for the span kernels."""
        d = self.config.hidden_dim
        if getattr(blob, "synthetic", False):
            raise ProtocolError("synthetic blob carries no data")
        # device payloads produced on another GPU (the previous span's server)
        # move peer to peer over NVLink; same-device payloads are used in place
        here = self.device if isinstance(self.device, torch.device) else torch.device(
            "cuda", self.device)
        if getattr(blob, "dev_codes", None) is not None:
            c, s = blob.dev_codes.to(here), blob.dev_scales.to(here)
            return 0, c.data_ptr(), s.data_ptr(), (c, s)
        if getattr(blob, "dev", None) is not None:
            x = blob.dev.to(here)
            return x.data_ptr(), 0, 0, (x,)
        q = blob.quant
        if q is not None:
            c = torch.from_numpy(np.ascontiguousarray(q.codes, np.int8)).to(self.device)
            s = torch.from_numpy(np.ascontiguousarray(q.scales, np.float32)).to(self.device)
            return 0, c.data_ptr(), s.data_ptr(), (c, s)
        a = np.ascontiguousarray(blob.array(), dtype=np.float32).reshape(rows, d)
        x = self._upload(a)
        return x.data_ptr(), 0, 0, (x,)

    def _upload(self, a: np.ndarray) -> torch.Tensor:
        """Host rows -> HBM without blocking the host on the stream: the rows are
        copied into a pinned staging slot (a ring of 4; a slot is rewritten only
        after its previous copy has completed) and moved by an asynchronous H2D
        copy ordered in the span's stream (a pageable `.to(device)` would wait
        for every kernel already queued — the previous step)."""
        nb = a.nbytes
        if len(self._staging) < 4:
            self._staging.append([None, torch.cuda.Event()])
        slot = self._staging[self._stage_next % len(self._staging)]
        self._stage_next += 1
        if slot[0] is None or slot[0].numel() < nb:
            slot[1].synchronize()
            slot[0] = torch.empty(max(nb, 1 << 16), dtype=torch.uint8, pin_memory=True)
        else:
            slot[1].synchronize()
        host = slot[0][:nb].view(torch.float32).view(a.shape)
        host.numpy()[...] = a
        x = torch.empty(a.shape, dtype=torch.float32, device=self.device)
        x.copy_(host, non_blocking=True)
        slot[1].record(torch.cuda.current_stream(self.device))
        return x

    def run_cached(self, start: int, end: int, caches: SpanCaches, blob, width: int, n_new: int,
                   quantized: bool) -> HiddenBlob:
        """`RealServerEngine.run_cached` (SP/server.py:93-100): all rows of
        [width*n_new, d] through blocks [start, end), appending n_new positions."""
        rows, d = width * n_new, self.config.hidden_dim
        with torch.cuda.device(self.device):
            xp, cp, sp_, keep = self._input_ptrs(blob, rows)
            y = torch.empty((rows, d), dtype=torch.float32, device=self.device)
            yc = ys = None
            if quantized:
                yc = torch.empty(rows * d, dtype=torch.int8, device=self.device)
                ys = torch.empty((rows * d + 63) // 64, dtype=torch.float32, device=self.device)
            _lib.check(self.lib.sp_span_forward(
                self.span.handle, caches.handle, start, end, xp, cp, sp_, y.data_ptr(),
                yc.data_ptr() if yc is not None else 0, ys.data_ptr() if ys is not None else 0,
                width, n_new, _stream(self.device)))
            del keep
        if quantized:
            return HiddenBlob.from_device(y, yc, ys)
        return HiddenBlob.from_device(y)

    def reorder(self, caches: SpanCaches, parents_zero_based: list[int]) -> None:
        idx = np.asarray(parents_zero_based, dtype=np.int32)
        if idx.size and (idx.min() < 0 or idx.max() >= caches.width):
            raise ProtocolError("reorder index out of range")
        with torch.cuda.device(self.device):
            _lib.check(self.lib.sp_kv_reorder(caches.handle, idx.ctypes.data, int(idx.size),
                                              _stream(self.device)))

    # -- stateless passes (prompt tuning) -----------------------------------------
    def forward(self, start: int, end: int, blob, batch: int, tokens: int,
                micro_batch_tokens: int, record: list | None) -> HiddenBlob:
        """`RealServerEngine.forward` (SP/server.py:106-125) with the same
        whole-sequence micro-batching (SP/server.py:189-194).

        ``record`` (prompt tuning) keeps every block input on the GPU for the
        backward pass; it is rejected up front for families without a backward
        (Llama / BLOOM shapes, quantised weights), whose records could never be
        used and would only hold (end - start) x rows x d floats of HBM."""
        if record is not None and not self.backward_defined:
            raise ProtocolError("forward(record=...) needs block_backward, defined for the "
                                "reference (toy, f32) family only")
        d = self.config.hidden_dim
        with torch.cuda.device(self.device):
            xp, cp, sp_, keep = self._input_ptrs(blob, batch * tokens)
            if cp:
                x = torch.empty(batch * tokens * d, dtype=torch.float32, device=self.device)
                _lib.check(self.lib.sp_dequantize_blockwise(cp, sp_, x.data_ptr(), x.numel(),
                                                            _stream(self.device)))
                keep = keep + (x,)
            else:
                x = keep[0]
            x = x.reshape(batch, tokens, d)
            y = torch.empty((batch, tokens, d), dtype=torch.float32, device=self.device)
            # chunk cap: the device chunk size, bounded by the KV pages free right
            # now (a stateless chunk holds ceil(tokens / 64) pages per sequence)
            fit = max(1, self.span.free_pages // max(1, -(-tokens // 64))) * tokens
            chunks = list(device_micro_batches(batch, tokens, min(micro_batch_tokens, fit),
                                               min(self.stateless_tokens, fit)))
            self.last_forward_chunks = len(chunks)
            for chunk in chunks:
                nb = chunk.stop - chunk.start
                xc = x[chunk].contiguous()
                rec = None
                if record is not None:
                    rec = torch.empty((end - start, nb * tokens, d), dtype=torch.float32,
                                      device=self.device)
                yc = y[chunk]
                _lib.check(self.lib.sp_span_forward_stateless(
                    self.span.handle, start, end, xc.data_ptr(), yc.data_ptr(),
                    rec.data_ptr() if rec is not None else 0, nb, tokens, _stream(self.device)))
                if record is not None:
                    record.append((chunk, [rec[i].reshape(nb, tokens, d)
                                           for i in range(end - start)]))
            del keep
        return HiddenBlob.from_device(y.reshape(batch * tokens, d))

    def backward(self, start: int, end: int, blob, batch: int, tokens: int,
                 record: list) -> HiddenBlob:
        """`RealServerEngine.backward` (SP/server.py:127-139): the gradient wrt the
        span input, block by block in reverse from the inputs `forward` recorded
        (per micro-batch chunk), each block recomputed in float64 on the GPU
        (`sp_span_block_backward`, block_backward of SP/model.py:320-381)."""
        d = self.config.hidden_dim
        with torch.cuda.device(self.device):
            here = self.device if isinstance(self.device, torch.device) else torch.device(
                "cuda", self.device)
            if getattr(blob, "dev", None) is not None:                # our device blob
                g = blob.dev.to(here)
            else:                                                      # host / coded / reference blob
                g = torch.from_numpy(np.ascontiguousarray(blob.array(), np.float32)).to(here)
            g = g.reshape(batch, tokens, d)
            grads = []
            for chunk, per_block in record:
                nb = chunk.stop - chunk.start
                gc = g[chunk].contiguous().reshape(nb * tokens, d)
                for offset, bi in enumerate(reversed(range(start, end))):
                    xin = per_block[len(per_block) - 1 - offset]
                    xin = torch.as_tensor(xin, device=here).reshape(nb * tokens, d).contiguous()
                    out = torch.empty_like(gc)
                    _lib.check(self.lib.sp_span_block_backward(
                        self.span.handle, bi, xin.data_ptr(), gc.data_ptr(), out.data_ptr(), nb,
                        tokens, _stream(self.device)))
                    gc = out
                grads.append(gc.reshape(nb, tokens, d))
            out = torch.cat(grads, dim=0).reshape(batch * tokens, d)
        return HiddenBlob.from_device(out)

    def blob_checksum(self, blob) -> int:
        """FNV-1a 64 over the f32 bytes (SP/server.py:141-142)."""
        a = np.ascontiguousarray(blob.array(), dtype=np.float32)
        return int(self.lib.sp_fnv1a64(a.ctypes.data, a.nbytes))


class _BlockList:
    """list-like `engine.blocks` (read-only, lazily materialised views)."""

    def __init__(self, span: DeviceSpan):
        self.span = span

    def __len__(self) -> int:
        return self.span.cfg.n_blocks

    def __getitem__(self, i: int) -> _BlockView:
        if i < 0:
            i += len(self)
        if not self.span.start <= i < self.span.end:
            raise IndexError(i)
        return _BlockView(self.span, i)

    def __iter__(self):
        return (self[i] for i in range(self.span.start, self.span.end))


def device_micro_batches(batch: int, tokens: int, micro_batch_tokens: int, device_tokens: int):
    """Whole-sequence chunks for the GPU: the reference's 1024-token micro-batches
    bound host memory (SP/server.py:189-194, 216) and its result is micro-batch
    invariant (T/test_server.py:247-255, array_equal), so the engine runs larger
    balanced chunks of up to max(micro_batch_tokens, device_tokens) tokens (the
    prefill GEMM's M); a single long sequence still runs unsplit."""
    cap = max(micro_batch_tokens, device_tokens)
    per = max(1, cap // max(tokens, 1))
    n = -(-batch // per)
    per = -(-batch // n)                               # balance: 32 x 132 -> 3 x 11/11/10
    for lo in range(0, batch, per):
        yield slice(lo, min(lo + per, batch))


def micro_batches(batch: int, tokens: int, micro_batch_tokens: int):
    """Whole-sequence chunks of at most micro_batch_tokens (SP/server.py:189-194)."""
    per_chunk = max(1, micro_batch_tokens // max(tokens, 1))
    for lo in range(0, batch, per_chunk):
        yield slice(lo, min(lo + per_chunk, batch))
