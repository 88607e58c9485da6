"""Client head on the GPU (`RealClientEngine`, SP/client.py:89-106): embedding
rows for token ids and the greedy pick from the last output row, through
libspanpipe.so (sp_head_*).  Interface = what SwarmClient calls:
``embed_array(tokens) -> np.ndarray [n, d]`` and ``pick(rows) -> int``."""

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

    def pick(self, final_rows) -> int:
        last = np.ascontiguousarray(np.asarray(final_rows, dtype=np.float32).reshape(
            -1, self.config.hidden_dim)[-1])
        return self.pick_device(torch.from_numpy(last).to(self.device))

    def embedding(self) -> np.ndarray:
        out = np.empty((self.config.vocab_size, self.config.hidden_dim), np.float32)
        _lib.check(self.lib.sp_head_read_embedding(self.handle, out.ctypes.data))
        return out
