"""Span server: session semantics of the reference's BlockServer around a
payload engine (`SP/server.py:222-496`).

Behaviour kept from the reference, check by check: interval check on open
("not_serving", :371-382); TTL expiry ("expired", :348-355); desync on relay
checksum mismatch, position or width mismatch, and on diverged cache length
("desync", :385-415); capacity guard ("capacity", :399-400, :433-434);
restore rebuilds the caches from the replayed history and may return a 0-row
blob (:429-450); 1-based reorder indices ("bad_index", :452-462); stateless
forward with replay dedup by req_id (:464-485) and backward by record
(:487-496); crash injection after N messages (:323-325).
Announce / rebalance timers and the directory are control-plane features
(out of scope); block placement itself is in balancer.py.
"""

from __future__ import annotations

from dataclasses import dataclass

from .blob import HiddenBlob
from .messages import (Backward, Close, Error, Forward, OpenSession, Ping, Pong, Reorder,
                       Restore, Step, StepResult)
from .transport import SimulatedCrash

SESSION_TTL_S = 300.0          # SP/server.py:34
MICRO_BATCH_TOKENS = 1024      # SP/server.py:216


@dataclass
class ServerCfg:
    server_id: str
    capacity: int
    start: int = 0
    session_ttl_s: float = SESSION_TTL_S
    crash_after_messages: int | None = None

    def __post_init__(self) -> None:
        if self.capacity < 1:
            raise ValueError("capacity must be >= 1")


@dataclass
class SessionState:
    session_id: int
    start: int
    end: int
    width: int
    quantized: bool
    caches: object
    positions: int
    last_activity: float
    desynced: bool = False


class BlockServer:
    """Protocol handler for one span server (one GPU engine)."""

    def __init__(self, cfg: ServerCfg, engine, transport=None):
        self.cfg = cfg
        self.engine = engine
        self.transport = transport
        self.n_blocks = engine.config.n_blocks
        self.start = cfg.start
        self.end = min(cfg.start + cfg.capacity, self.n_blocks)
        self.sessions: dict[int, SessionState] = {}
        self.forward_records: dict = {}
        self.replay: dict = {}
        self.handled = 0

    @property
    def server_id(self) -> str:
        return self.cfg.server_id

    def _now(self) -> float:
        return self.transport.clock.now if self.transport is not None else 0.0

    # -- dispatch (SP/server.py:322-346) ---------------------------------------
    def handle(self, p, sid: int = 0):
        self.handled += 1
        if self.cfg.crash_after_messages is not None and self.handled > self.cfg.crash_after_messages:
            raise SimulatedCrash(self.server_id)
        if isinstance(p, Ping):
            return Pong()
        if isinstance(p, OpenSession):
            return self._open(sid, p)
        if isinstance(p, Step):
            return self._step(sid, p)
        if isinstance(p, Restore):
            return self._restore(sid, p)
        if isinstance(p, Reorder):
            return self._reorder(sid, p)
        if isinstance(p, Close):
            self.sessions.pop(sid, None)
            return Pong()
        if isinstance(p, Forward):
            return self._forward(sid, p)
        if isinstance(p, Backward):
            return self._backward(sid, p)
        return Error("protocol", f"unsupported payload {type(p).__name__}")

    def _session(self, sid: int) -> SessionState | None:
        s = self.sessions.get(sid)
        if s is None:
            return None
        if self._now() - s.last_activity > self.cfg.session_ttl_s:
            del self.sessions[sid]
            return None
        return s

    # -- sessions ------------------------------------------------------------------
    def _open(self, sid: int, p: OpenSession):
        if not (self.start <= p.start and p.end <= self.end and p.start < p.end):
            return Error("not_serving",
                         f"serves [{self.start}, {self.end}), asked [{p.start}, {p.end})")
        self.sessions[sid] = SessionState(sid, p.start, p.end, p.width, p.quantized,
                                          self.engine.make_caches(p.start, p.end, p.width), 0,
                                          self._now())
        return Pong()

    def _step(self, sid: int, p: Step):
        s = self._session(sid)
        if s is None:
            return Error("expired", "no such session")
        if s.desynced:
            return Error("desync", "relay checksum mismatch")
        if p.checksum and self.engine.blob_checksum(p.blob) != p.checksum:
            s.desynced = True
            return Error("desync", "relay checksum mismatch")
        if p.position_offset != s.positions:
            return Error("desync", f"at position {s.positions}, step claims {p.position_offset}")
        if p.width != s.width:
            return Error("desync", f"width {s.width} != {p.width}")
        if p.position_offset + p.n_new > self.engine.config.max_seq_len:
            return Error("capacity", "sequence exceeds max_seq_len")
        out = self.engine.run_cached(s.start, s.end, s.caches, p.blob, p.width, p.n_new,
                                     s.quantized)
        s.positions += p.n_new
        if self.engine.cache_length(s.caches) != s.positions:
            s.desynced = True
            return Error("desync", "cache length diverged")
        s.last_activity = self._now()
        return StepResult(p.position_offset, out, p.width, p.n_new)

    def _restore(self, sid: int, p: Restore):
        s = self._session(sid)
        if s is None:
            return Error("expired", "no such session")
        if p.t > self.engine.config.max_seq_len:
            return Error("capacity", "history exceeds max_seq_len")
        s.caches = self.engine.make_caches(s.start, s.end, p.width)
        s.width = p.width
        s.positions = 0
        s.desynced = False
        if p.t > 0:
            out = self.engine.run_cached(s.start, s.end, s.caches, p.blob, p.width, p.t,
                                         s.quantized)
            s.positions = p.t
        else:
            out = HiddenBlob.shape_only(0, self.engine.config.hidden_dim)
        s.last_activity = self._now()
        if not p.want_outputs:
            out = HiddenBlob.shape_only(0, self.engine.config.hidden_dim)
        return StepResult(0, out, p.width, p.t)

    def _reorder(self, sid: int, p: Reorder):
        s = self._session(sid)
        if s is None:
            return Error("expired", "no such session")
        if not p.indices or any(i < 1 or i > s.width for i in p.indices):
            return Error("bad_index", f"indices must be in [1, {s.width}]")
        self.engine.reorder(s.caches, [i - 1 for i in p.indices])
        s.width = len(p.indices)
        s.last_activity = self._now()
        return Pong()

    # -- stateless passes ---------------------------------------------------------
    def _forward(self, sid: int, p: Forward):
        hit = self.replay.get(sid)
        if hit is not None and hit[0] == p.req_id:
            return hit[1]
        record: list | None = [] if p.record else None
        out = self.engine.forward(self.start, self.end, p.blob, p.batch, p.tokens,
                                  MICRO_BATCH_TOKENS, record)
        if p.quantize_reply:
            out = HiddenBlob.from_array(out.array(), quantized=True)
        if p.record:
            self.forward_records[(sid, p.req_id)] = record
            for key in [k for k in self.forward_records if k[0] == sid and k[1] != p.req_id]:
                del self.forward_records[key]
        reply = StepResult(0, out, p.batch, p.tokens)
        self.replay[sid] = (p.req_id, reply)
        return reply

    def _backward(self, sid: int, p: Backward):
        record = self.forward_records.get((sid, p.req_id))
        if record is None:
            return Error("no_record", "no matching forward; repeat the pass")
        out = self.engine.backward(self.start, self.end, p.blob, p.batch, p.tokens, record)
        return StepResult(0, out, p.batch, p.tokens)
