"""Multi-process span ring with the dual-cache failover of the reference
(SP/client.py:340-415), one process per GPU.

Roles (world = N + 1 ranks):

* ring positions 0..N-1 serve the spans `stage_intervals(n_blocks, N)`; the
  rank at position 0 is also the client: it embeds tokens, picks the greedy
  token from the final row (the GPU client head) and keeps the client-side
  input cache of every stage;
* the last rank is a hot spare that holds the weights and joins the ring only
  when a span rank is dropped.

Data plane (NCCL send/recv, or gloo on CPU): each position sends its output to
the next as int8 codes + f32 scales (SP/quantize.py; stage->stage boundaries are
coded, SP/client.py:280-287) and — the relay mode of SP/client.py:668-777, where
every stage also answers the client — a copy to the client, which appends it to
that stage's input history.  The last position returns the final f32 row.

Control plane (the torch.distributed store, like the reference's RPCs): at every
tick boundary each live rank posts a heartbeat; the client waits for them with a
timeout (the reference's missing-ack budget, SP/netsim.py:53-54), declares a
missing rank dead (ban, SP/client.py:346-347) and publishes the route of the
tick.  p2p ops of a tick are posted only after its route is known, so no
collective is ever held open on a dropped rank.

Relay checksum (SP/server.py:388-393, 413-426): every coded wire (hop, relay
copy, replayed history) carries a content hash of its codes + scales, stamped
by the sender and verified by every receiver on the GPU (`relay.py`); a
mismatch raises ProtocolError("desync: relay checksum mismatch") at the tick
it is received.

Failover (`_replace_failed_stage` + `_restore`, SP/client.py:340-384,
SP/server.py:429-450): the client sends the spare, per session, the dropped
span's whole input history — the coded rows it cached — and the spare replays
it as one prefill per session (`run_cached` with n_new = t, the tensor-core
prefill path), rebuilding the KV caches; the input the dropped rank had received
but not processed is run as the resumed step, and the ring continues.
"""

from __future__ import annotations

import datetime
import json
import time

import torch

from .blob import HiddenBlob
from .placement import stage_intervals
from .relay import WireCheck, split_wire, wire_layout


class SwarmUnavailableError(RuntimeError):
    """No spare left to replace a dropped span (SP/errors.py:49)."""


class Membership:
    """Per-tick liveness agreement over the rendezvous store."""

    def __init__(self, store, rank: int, world: int, detect_timeout_s: float = 2.0,
                 prefix: str = "fo"):
        self.store, self.rank, self.world = store, rank, world
        self.timeout = datetime.timedelta(seconds=detect_timeout_s)
        self.prefix = prefix
        self.dead: set[int] = set()

    def tick(self, k: int) -> set[int]:
        """Heartbeat for tick k; returns the set of dead ranks (cumulative)."""
        p = self.prefix
        self.store.set(f"{p}/alive/{k}/{self.rank}", b"1")
        if self.rank == 0:
            for r in range(1, self.world):
                if r in self.dead:
                    continue
                try:
                    self.store.wait([f"{p}/alive/{k}/{r}"], self.timeout)
                except Exception:              # missing heartbeat: the rank is dropped
                    self.dead.add(r)
            self.store.set(f"{p}/route/{k}", json.dumps(sorted(self.dead)).encode())
        self.dead = set(json.loads(self.store.get(f"{p}/route/{k}").decode()))
        return self.dead


class FailoverRing:
    """Greedy generation of `n_sessions` sessions through an N-span ring with a
    spare rank.  `engine` = the span engine of this rank (`run_cached`,
    `make_caches`), `head` = the client head on rank 0 (`embed_device(tokens)`,
    `pick_device(row)`)."""

    def __init__(self, engine, head, cfg, rank: int, world: int, device: torch.device,
                 prefixes: list[list[int]], n_new: int, store=None, drop: tuple | None = None,
                 detect_timeout_s: float = 2.0, store_prefix: str = "fo", checksum=None):
        import torch.distributed as dist
        self.dist = dist
        if world < 3:
            raise ValueError("a failover ring needs >= 2 span ranks + 1 spare")
        self.eng, self.head, self.cfg = engine, head, cfg
        self.rank, self.world, self.dev = rank, world, device
        self.N = world - 1                       # span positions
        self.spare = world - 1
        self.spans = stage_intervals(cfg.n_blocks, self.N)
        self.pos2rank = list(range(self.N))
        self.S = len(prefixes)
        if self.S != self.N:
            raise ValueError("one session per ring position (the bench schedule)")
        self.prefixes = [list(p) for p in prefixes]
        self.P = len(prefixes[0])
        if any(len(p) != self.P for p in prefixes):
            raise ValueError("equal prompt lengths")
        self.T = n_new
        self.d = cfg.hidden_dim
        self.drop = drop                         # (rank, tick): emulated server loss
        self.members = Membership(store or dist.distributed_c10d._get_default_store(), rank,
                                  world, detect_timeout_s, store_prefix)
        self.tokens = [list(p) for p in prefixes]          # rank 0
        self.hist: dict = {}                     # rank 0: (position, session) -> [wire]
        self.caches = None
        self.pending = {}                        # position input wires received for next tick
        self.final_rows = {}                     # rank 0: session -> final f32 row
        self.replays: list[dict] = []
        self._span_of = None
        # relay checksum: None = on for a CUDA device, False = off, or a checker
        # object with stamp / verify / raise_if_mismatch (CPU tests)
        if checksum is None:
            checksum = WireCheck(device) if device.type == "cuda" else False
        self.check = checksum or None
        self._bind_position()

    # -- schedule ---------------------------------------------------------------
    def _work(self, pos: int, k: int):
        """(session, pass) processed at position pos in tick k, or None."""
        if k < pos:
            return None
        s = (k - pos) % self.N
        j = (k - pos - s) // self.N
        if s >= self.S or j >= self.T:
            return None
        return s, j

    def _rows(self, j: int) -> int:
        return self.P if j == 0 else 1

    def _layout(self, rows: int):
        return wire_layout(rows, self.d, self.check is not None)

    def _new_wire(self, rows: int) -> torch.Tensor:
        return torch.zeros(self._layout(rows)[2], dtype=torch.uint8, device=self.dev)

    def _stamp(self, w: torch.Tensor, rows: int) -> None:
        if self.check is not None:
            payload, off, _ = self._layout(rows)
            self.check.stamp(w, payload, off)

    def _verify(self, w: torch.Tensor, rows: int) -> None:
        if self.check is not None:
            payload, off, _ = self._layout(rows)
            self.check.verify(w, payload, off)

    @property
    def n_ticks(self) -> int:
        return self.N * (self.T - 1) + 2 * (self.N - 1) + 1

    def _bind_position(self):
        self.pos = self.pos2rank.index(self.rank) if self.rank in self.pos2rank else None
        if self.pos is not None and self._span_of != self.pos:
            a, b = self.spans[self.pos]
            self.caches = [self.eng.make_caches(a, b, 1) for _ in range(self.S)]
            self._span_of = self.pos

    # -- one tick ---------------------------------------------------------------
    def _forward(self, s: int, j: int, wire_in):
        a, b = self.spans[self.pos]
        last = self.pos == self.N - 1
        rows = self._rows(j)
        if self.pos == 0:
            toks = self.prefixes[s] if j == 0 else [self.tokens[s][-1]]
            blob = HiddenBlob.from_device(self.head.embed_device(toks))
        else:
            c, sc = split_wire(wire_in, rows, self.d)
            blob = HiddenBlob(rows, self.d, dev_codes=c, dev_scales=sc)
        out = self.eng.run_cached(a, b, self.caches[s], blob, 1, rows, not last)
        if last:
            return out.dev[-1].contiguous()
        w = self._new_wire(rows)
        c, sc = split_wire(w, rows, self.d)
        c.copy_(out.dev_codes)
        sc.copy_(out.dev_scales)
        self._stamp(w, rows)
        return w

    def step(self, k: int) -> None:
        dist = self.dist
        if self.drop is not None and self.drop == (self.rank, k):
            self.dropped = True
            return
        dead = self.members.tick(k)
        for r in dead:
            if r in self.pos2rank:
                self._replace(self.pos2rank.index(r), k)
        self._bind_position()
        ops, out = [], None
        if self.pos is not None:
            w = self._work(self.pos, k)
            if w is not None:
                s, j = w
                wire_in = self.pending.pop((s, j), None) if self.pos > 0 else None
                if self.pos > 0 and wire_in is None:
                    raise RuntimeError(f"rank {self.rank}: no input for session {s} pass {j}")
                out = self._forward(s, j, wire_in)
                if self.pos == 0:
                    self.hist.setdefault((1, s), []).append(out)
                nxt = self.pos2rank[(self.pos + 1) % self.N]
                ops.append(dist.P2POp(dist.isend, out, nxt))
                if 0 < self.pos < self.N - 1:        # relay copy to the client's cache
                    ops.append(dist.P2POp(dist.isend, out, self.pos2rank[0]))
        # receives for the next tick
        recvs = []
        if self.pos is not None and self.pos > 0:
            w = self._work(self.pos - 1, k)
            if w is not None:
                s, j = w
                buf = self._new_wire(self._rows(j))
                ops.append(dist.P2POp(dist.irecv, buf, self.pos2rank[self.pos - 1]))
                recvs.append(("in", s, j, buf))
        if self.pos == 0:
            w = self._work(self.N - 1, k)
            if w is not None:
                s, j = w
                buf = torch.empty(self.d, dtype=torch.float32, device=self.dev)
                ops.append(dist.P2POp(dist.irecv, buf, self.pos2rank[self.N - 1]))
                recvs.append(("final", s, j, buf))
            for p in range(1, self.N - 1):            # relay copies (client cache)
                w = self._work(p, k)
                if w is not None:
                    s, j = w
                    buf = self._new_wire(self._rows(j))
                    ops.append(dist.P2POp(dist.irecv, buf, self.pos2rank[p]))
                    recvs.append(("hist", s, j, buf, p + 1))
        if ops:
            for h in dist.batch_isend_irecv(ops):
                h.wait()
        for r in recvs:                               # relay checksums (in the stream)
            if r[0] != "final":
                self._verify(r[3], self._rows(r[2]))
        if self.check is not None and any(r[0] != "final" for r in recvs):
            self.check.raise_if_mismatch()
        for r in recvs:
            if r[0] == "in":
                self.pending[(r[1], r[2])] = r[3]
            elif r[0] == "final":
                s = r[1]
                self.tokens[s].append(self.head.pick_device(r[3]))
            else:
                self.hist.setdefault((r[4], r[1]), []).append(r[3])

    # -- failover ------------------------------------------------------------------
    def _replace(self, pos: int, k: int) -> None:
        """Ring position `pos` lost at the start of tick k: the spare takes it
        over after replaying the position's cached inputs (SP/client.py:340-384)."""
        dist = self.dist
        if pos == 0:
            raise SwarmUnavailableError("the client's own span cannot be replaced")
        if self.spare in self.pos2rank or self.spare in self.members.dead:
            raise SwarmUnavailableError("no spare left")
        t0 = time.perf_counter()
        self.pos2rank[pos] = self.spare
        # per session: all inputs the position ever received (rank 0's cache);
        # the last one is pending (sent at the end of tick k-1, not processed)
        pend = self._work(pos, k)
        counts = []
        for s in range(self.S):
            n_in = sum(1 for kk in range(k) if self._work(pos - 1, kk) is not None
                       and self._work(pos - 1, kk)[0] == s)
            counts.append(n_in)
        if self.rank == 0:
            for s in range(self.S):
                msgs = self.hist.get((pos, s), [])
                assert len(msgs) == counts[s], (pos, s, len(msgs), counts[s])
                if not msgs:
                    continue
                rows = [self._rows(j) for j in range(len(msgs))]
                # the history as ONE wire of sum(rows) rows (codes, scales, hash)
                n_rows = sum(rows)
                hw = self._new_wire(n_rows)
                hc, hs = split_wire(hw, n_rows, self.d)
                torch.cat([split_wire(m, r, self.d)[0] for m, r in zip(msgs, rows)], out=hc)
                torch.cat([split_wire(m, r, self.d)[1] for m, r in zip(msgs, rows)], out=hs)
                self._stamp(hw, n_rows)
                for h in dist.batch_isend_irecv([dist.P2POp(dist.isend, hw, self.spare)]):
                    h.wait()
            self.replays.append({"position": pos, "tick": k,
                                 "sessions": sum(1 for c in counts if c),
                                 "rows": [sum(self._rows(j) for j in range(c)) for c in counts],
                                 "client_send_s": time.perf_counter() - t0})
        elif self.rank == self.spare:
            self._bind_position()
            a, b = self.spans[pos]
            tr = time.perf_counter()
            for s in range(self.S):
                if not counts[s]:
                    continue
                rows = [self._rows(j) for j in range(counts[s])]
                n_rows = sum(rows)
                hw = self._new_wire(n_rows)
                for h in dist.batch_isend_irecv([dist.P2POp(dist.irecv, hw, 0)]):
                    h.wait()
                self._verify(hw, n_rows)
                if self.check is not None:
                    self.check.raise_if_mismatch()
                codes, scales = split_wire(hw, n_rows, self.d)
                done = n_rows
                if pend is not None and pend[0] == s:     # resumed step runs normally
                    r_last = rows[-1]
                    done = n_rows - r_last
                    w = self._new_wire(r_last)
                    wc, ws = split_wire(w, r_last, self.d)
                    wc.copy_(codes[done * self.d:])
                    ws.copy_(scales[done * self.d // 64:])
                    self.pending[(s, pend[1])] = w
                if done:
                    blob = HiddenBlob(done, self.d, dev_codes=codes[:done * self.d],
                                      dev_scales=scales[:done * self.d // 64])
                    self.eng.run_cached(a, b, self.caches[s], blob, 1, done,
                                        pos != self.N - 1)
            if self.dev.type == "cuda":
                torch.cuda.synchronize(self.dev)
            self.replays.append({"position": pos, "tick": k,
                                 "replay_s": time.perf_counter() - tr,
                                 "rows": [sum(self._rows(j) for j in range(c)) for c in counts]})

    def warm(self) -> None:
        """Open the p2p connections a failover would use (client <-> spare, spare <->
        every span rank) so that a measured replay does not include NCCL's lazy
        connection set-up.  Collective over all ranks."""
        dist = self.dist
        one = torch.zeros(1, device=self.dev)
        ops = []
        if self.rank == self.spare:
            for r in range(self.N):
                ops.append(dist.P2POp(dist.isend, one, r))
                ops.append(dist.P2POp(dist.irecv, torch.zeros(1, device=self.dev), r))
        else:
            ops.append(dist.P2POp(dist.irecv, torch.zeros(1, device=self.dev), self.spare))
            ops.append(dist.P2POp(dist.isend, one, self.spare))
        for h in dist.batch_isend_irecv(ops):
            h.wait()
        dist.barrier()

    def run(self) -> list[list[int]]:
        self.dropped = False
        for k in range(self.n_ticks):
            self.step(k)
            if self.dropped:
                break
        return self.tokens
