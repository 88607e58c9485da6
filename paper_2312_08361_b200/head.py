"""Client head on the GPU — the payload side of `RealClientEngine`
(SP/client.py:89-106): embedding rows for token ids, the tied logits
``row @ E^T`` (SP/model.py:393-395, no final norm) and the token choice, all
through libspanpipe.so (sp_head_*).

Interface = what the reference's SwarmClient calls on its client engine:
``embed_array(tokens) -> np.ndarray [n, d]``,
``pick(final_rows, mode, rng, top_k) -> int`` (greedy on the GPU; sampling
draws from GPU logits on the host with the reference's float64 recipe) and
``logits(rows) -> np.ndarray [n, vocab]`` (beam search).
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .config import from_reference


class ClientHead:
    def __init__(self, config, device: int = 0):
        self.config = from_reference(config)
        self.lib = _lib.load()
        self.device = torch.device("cuda", device)
        self._c = _lib.make_config(self.config)
        h = ctypes.c_void_p()
        _lib.check(self.lib.sp_head_create(ctypes.byref(self._c), device, ctypes.byref(h)))
        self.handle = h

    def __del__(self):
        h = getattr(self, "handle", None)
        if h and h.value:
            try:
                self.lib.sp_head_destroy(h)
            except Exception:
                pass

    def _stream(self) -> int:
        return torch.cuda.current_stream(self.device).cuda_stream

    def _rows_device(self, rows) -> torch.Tensor:
        d = self.config.hidden_dim
        if isinstance(rows, torch.Tensor):
            return rows.to(self.device, torch.float32).reshape(-1, d).contiguous()
        a = np.ascontiguousarray(np.asarray(rows, dtype=np.float32).reshape(-1, d))
        return torch.from_numpy(a).to(self.device)

    def embed_device(self, tokens) -> torch.Tensor:
        t = np.ascontiguousarray(tokens, dtype=np.int32)
        out = torch.empty((t.size, self.config.hidden_dim), dtype=torch.float32, device=self.device)
        _lib.check(self.lib.sp_head_embed(self.handle, t.ctypes.data, int(t.size), out.data_ptr(),
                                          self._stream()))
        return out

    def embed_array(self, tokens) -> np.ndarray:
        return self.embed_device(tokens).cpu().numpy()

    def pick_device(self, row: torch.Tensor) -> int:
        tok = np.zeros(1, np.int32)
        row = row.contiguous()
        _lib.check(self.lib.sp_head_greedy(self.handle, row.data_ptr(), tok.ctypes.data,
                                           self._stream()))
        return int(tok[0])

    def logits_device(self, rows) -> torch.Tensor:
        x = self._rows_device(rows)
        out = torch.empty((x.shape[0], self.config.vocab_size), dtype=torch.float32,
                          device=self.device)
        _lib.check(self.lib.sp_head_logits(self.handle, x.data_ptr(), int(x.shape[0]),
                                           out.data_ptr(), self._stream()))
        return out

    def logits(self, rows) -> np.ndarray:
        """[n, vocab] logits of n rows (`RealClientEngine.logits`, SP/client.py:104-105)."""
        return self.logits_device(rows).cpu().numpy()

    def pick(self, final_rows, mode: str = "greedy", rng=None, top_k=None) -> int:
        """Token from the last row (`RealClientEngine.pick`, SP/client.py:97-102)."""
        last = self._rows_device(final_rows)[-1:]
        if mode == "greedy":
            return self.pick_device(last[0])
        return sample_pick(self.logits_device(last)[0].cpu().numpy(), rng, top_k)

    def beam_select_device(self, scores, logits_dev: torch.Tensor, k: int):
        """`beam_select` (SP/model.py:470-491) on device logits [w, vocab]."""
        return beam_select_device(scores, logits_dev, k)

    def embedding(self) -> np.ndarray:
        out = np.empty((self.config.vocab_size, self.config.hidden_dim), np.float32)
        _lib.check(self.lib.sp_head_read_embedding(self.handle, out.ctypes.data))
        return out


def sample_pick(logits: np.ndarray, rng: np.random.Generator, top_k: int | None = None) -> int:
    """Seeded categorical draw over float64 softmax probabilities — the recipe
    of SP/model.py:403-416 (top-k mask to -inf, max-shifted exp, one uniform
    draw located in the cumulative sum), so a shared rng stream draws the same
    tokens as the reference client."""
    z = np.asarray(logits, dtype=np.float64)
    if top_k is not None and top_k < z.size:
        kept = np.argpartition(z, -top_k)[-top_k:]
        z = np.where(np.isin(np.arange(z.size), kept), z, -np.inf)
    p = np.exp(z - z.max())
    p = p / p.sum()
    return int(np.searchsorted(np.cumsum(p), rng.random(), side="right"))


def beam_select_device(scores, logits_dev: torch.Tensor, k: int):
    """One beam-search selection step on the GPU (sp_beam_select): float64
    log-softmax of each row, candidates scores[r] + logp, the k best ranked by
    (score desc, parent asc, token asc) — SP/model.py:470-491.  Returns
    (parents, tokens, new_scores) like the reference."""
    lib = _lib.load()
    lg = logits_dev.to(torch.float32).contiguous()
    w, vocab = int(lg.shape[0]), int(lg.shape[1])
    sc = np.ascontiguousarray(np.asarray(scores, dtype=np.float64).reshape(w))
    par = np.zeros(k, np.int32)
    tok = np.zeros(k, np.int32)
    out = np.zeros(k, np.float64)
    stream = torch.cuda.current_stream(lg.device).cuda_stream
    with torch.cuda.device(lg.device):
        _lib.check(lib.sp_beam_select(lg.data_ptr(), sc.ctypes.data, w, vocab, k, par.ctypes.data,
                                      tok.ctypes.data, out.ctypes.data, stream))
    return par.tolist(), tok.tolist(), out


def beam_select(scores, all_logits, k: int, device: int = 0):
    """Drop-in for the reference's `beam_select(scores, all_logits, k)` with host
    logits (uploaded to the GPU first)."""
    lg = torch.from_numpy(np.ascontiguousarray(all_logits, dtype=np.float32)).to(
        torch.device("cuda", device))
    return beam_select_device(scores, lg, k)
