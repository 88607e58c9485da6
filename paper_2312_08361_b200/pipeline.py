"""Multi-GPU span pipeline: one process per GPU, each serving one contiguous
span; activations cross span boundaries as int8 codes + f32 scales
(`SP/quantize.py`, 8,704 B/token at d = 8192) by NCCL send/recv over NVLink.

Schedule (N ranks, N sessions in flight): at tick k rank r advances session
(k - r) mod N through its span.  Rank r's output of tick k is the input of
rank r+1 at tick k+1; the last rank returns the f32 rows of the final block
to rank 0 (the client side: only stage->stage boundaries are coded,
`SP/client.py:280-287`), which feeds them back as that session's next input.
Each tick ends with ONE grouped p2p (send this tick's output, receive next
tick's input), so the ring never deadlocks and the host never blocks.
With N == 1 this degenerates to plain autoregressive stepping of one session.

Relay checksum (SP/server.py:388-393, 413-426): every coded hop carries a
content hash of its codes + scales (`relay.py`), stamped by the sender and
verified by the receiver on the GPU before its span consumes the input; a
mismatch is raised by `verify()` (or at the next tick with `strict=True`).
"""

from __future__ import annotations

import torch

from . import _lib
from .relay import WireCheck, wire_layout


class SpanPipeline:
    def __init__(self, engine, start: int, end: int, caches: list, rank: int, world: int, d: int,
                 device: torch.device, seed: int = 7, width: int = 1, checksum=None,
                 strict: bool = False):
        self.eng, self.lib = engine, getattr(engine, "lib", None)
        self.start, self.end = start, end
        self.caches = caches
        self.rank, self.world, self.d = rank, world, d
        self.dev = device
        self.k = 0
        self.width = w = width                    # rows per session per tick (batch / beams)
        n = w * d
        n_sc = (n + 63) // 64
        g = torch.Generator(device=device).manual_seed(seed + rank)
        self.init_rows = torch.randn(max(1, world), w, d, device=device, generator=g)
        self.y = torch.empty(w, d, device=device)
        self.ring_in = torch.empty(w, d, device=device)            # rank 0: from the last rank
        # relay checksum: None = on for a CUDA device, False = off, or a checker
        # object with stamp / verify / raise_if_mismatch (CPU tests)
        if checksum is None:
            checksum = WireCheck(device) if device.type == "cuda" and world > 1 else False
        self.check = checksum or None
        self.strict = strict
        self.payload, self.hash_off, total = wire_layout(w, d, self.check is not None)
        self.out_wire = torch.zeros(total, dtype=torch.uint8, device=device)
        self.in_wire = torch.zeros(total, dtype=torch.uint8, device=device)
        self.out_codes = self.out_wire[:n].view(torch.int8)
        self.out_scales = self.out_wire[n:n + 4 * n_sc].view(torch.float32)
        self.in_codes = self.in_wire[:n].view(torch.int8)
        self.in_scales = self.in_wire[n:n + 4 * n_sc].view(torch.float32)
        if world == 1:
            self.y.copy_(self.init_rows[0])

    def _forward(self, session: int, x, coded_input: bool, quantize_out: bool) -> None:
        """One span pass of `session` (1 row): input `x` (f32 rows) or, when
        `coded_input`, the received int8 codes + scales; writes `self.y` and,
        when `quantize_out`, `self.out_codes` / `self.out_scales`."""
        st = torch.cuda.current_stream(self.dev).cuda_stream
        _lib.check(self.lib.sp_span_forward(
            self.eng.span.handle, self.caches[session].handle, self.start, self.end,
            0 if coded_input else x.data_ptr(),
            self.in_codes.data_ptr() if coded_input else 0,
            self.in_scales.data_ptr() if coded_input else 0, self.y.data_ptr(),
            self.out_codes.data_ptr() if quantize_out else 0,
            self.out_scales.data_ptr() if quantize_out else 0, self.width, 1, st))

    def step(self) -> None:
        k, r, N = self.k, self.rank, self.world
        if N == 1:
            # autoregressive feedback: the span output is the next input (in place)
            self._forward(0, self.y, False, False)
            self.k += 1
            return
        import torch.distributed as dist
        active = k >= r
        s = (k - r) % N
        last = r == N - 1
        if active:
            if r == 0:
                x = self.init_rows[s] if k < N else self.ring_in
                self._forward(s, x, False, True)
            else:
                if self.check is not None and self.strict:
                    self.check.raise_if_mismatch()
                self._forward(s, None, True, not last)
            if not last:
                self._stamp()
        ops = []
        if active:
            if last:
                ops.append(dist.P2POp(dist.isend, self.y, 0))
            else:
                ops.append(dist.P2POp(dist.isend, self.out_wire, r + 1))
        if r == 0:
            if k >= N - 1:
                ops.append(dist.P2POp(dist.irecv, self.ring_in, N - 1))
        elif k >= r - 1:
            ops.append(dist.P2POp(dist.irecv, self.in_wire, r - 1))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        if r > 0 and k >= r - 1:
            self._verify_in()
        self.k += 1

    def _stamp(self) -> None:
        if self.check is not None:
            self.check.stamp(self.out_wire, self.payload, self.hash_off)

    def _verify_in(self) -> None:
        if self.check is not None:
            self.check.verify(self.in_wire, self.payload, self.hash_off)

    def verify(self) -> None:
        """Raise ProtocolError if any received hop failed its relay checksum."""
        if self.check is not None:
            self.check.raise_if_mismatch()

    def step_api(self, host_rows) -> None:
        """One tick through the public engine API (`run_cached`): rank 0 takes its
        session's input row from host memory (H2D inside the call), the last rank
        reads its result to the host (D2H); the span-to-span wire is the same
        int8 codes + scales over NCCL.  (`bench.py` e2e at N > 1.)"""
        from .blob import HiddenBlob
        k, r, N = self.k, self.rank, self.world
        active = k >= r
        s = (k - r) % N
        last = r == N - 1
        if active:
            if r == 0:
                blob = HiddenBlob.from_array(host_rows[s])
            else:
                blob = HiddenBlob(self.width, self.d, dev_codes=self.in_codes,
                                  dev_scales=self.in_scales)
            out = self.eng.run_cached(self.start, self.end, self.caches[s], blob, self.width, 1,
                                      not last)
            if last:
                # the step's result to the host: the read is started now and
                # collected at the next tick, so this rank's host keeps the ring
                # fed instead of idling on its own stream (finish_api() collects
                # the last one)
                self.finish_api()
                if not hasattr(self, "_host_bufs"):      # two pinned result buffers, alternated
                    self._host_bufs = [torch.empty((self.width, self.d), dtype=torch.float32,
                                                   pin_memory=True) for _ in range(2)]
                    self._host_i = 0
                buf = self._host_bufs[self._host_i]
                self._host_i ^= 1
                self._pending = out.array_async(out=buf)
                self.y.copy_(out.dev)
            else:
                self.out_codes.copy_(out.dev_codes)
                self.out_scales.copy_(out.dev_scales)
                self._stamp()
        import torch.distributed as dist
        ops = []
        if active:
            ops.append(dist.P2POp(dist.isend, self.y if last else self.out_wire,
                                  0 if last else r + 1))
        if r == 0:
            if k >= N - 1:
                ops.append(dist.P2POp(dist.irecv, self.ring_in, N - 1))
        elif k >= r - 1:
            ops.append(dist.P2POp(dist.irecv, self.in_wire, r - 1))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        if r > 0 and k >= r - 1:
            self._verify_in()
        self.k += 1

    def finish_api(self):
        """Collect the outstanding device->host read of step_api (last rank)."""
        p = getattr(self, "_pending", None)
        if p is not None:
            self.host_out = p.result().copy()      # the buffer is reused two ticks later
            self._pending = None
        return getattr(self, "host_out", None)

    @property
    def wire_bytes_per_token(self) -> int:
        return int(self.out_wire.numel())
