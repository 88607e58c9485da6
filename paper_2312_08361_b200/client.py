"""Dual-cache inference client with failover replay — the reference's
`SwarmClient` DUAL_CACHE path (`SP/client.py:240-512`), unchanged in
semantics:

* per stage it keeps every activation it sent (the client-side input cache,
  `SP/client.py:310-323`), as rows, or as reorder ops for beams;
* a stage failure bans the server, routes a replacement chain for the failed
  stage's blocks, replays the cached history in ONE batched Restore per
  replacement hop (the prefill path of the GPU engine) and resumes the
  interrupted step at that stage (`SP/client.py:340-415`);
* "expired"/"desync" answers rebuild the session on the same server
  (`SP/client.py:417-427`, keeping the reference's quirk of opening it with
  the raw ``quantized`` flag);
* only stage->stage boundaries are int8-coded (`SP/client.py:280-287`).
The counters (messages, recoveries, reroutes, restore_events, step bytes)
are the reference's `RunCounters` (`SP/client.py:43-58`) and are reproduced
exactly for the same swarm and failure injection (tests/test_host_mirror.py).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .blob import HiddenBlob
from .errors import (CapacityError, ConfigurationError, ConnectionFailed, MessageDropped,
                     NoRouteError, SwarmUnavailableError)
from .messages import Close, Error, OpenSession, Reorder, Restore, Step
from .router import Hop, RoutingGraph, ServerRoute


@dataclass
class RunCounters:
    step_activation_bytes: int = 0
    per_step_bytes: list = field(default_factory=list)
    restore_events: list = field(default_factory=list)
    messages: int = 0
    recoveries: int = 0
    reroutes: int = 0
    restarts: int = 0
    retries: int = 0

    @property
    def restore_bytes(self) -> int:
        return sum(e[3] for e in self.restore_events)


@dataclass
class GenerateResult:
    tokens: list
    counters: RunCounters


class _StageFailure(Exception):
    def __init__(self, server_id: str, ban: bool, reason: str, recover_in_place: bool = False):
        super().__init__(f"{server_id}: {reason}")
        self.server_id = server_id
        self.ban = ban
        self.recover_in_place = recover_in_place


@dataclass
class _HistoryItem:
    kind: str                       # "rows" | "reorder"
    width: int = 1
    n_new: int = 0
    rows: np.ndarray | None = None  # [width, n_new, d]
    parents0: list | None = None


@dataclass
class _Stage:
    hop: Hop
    session_id: int
    history: list = field(default_factory=list)
    rows_sent: int = 0

    @property
    def server_id(self) -> str:
        return self.hop.server_id

    def history_matrix(self, d: int):
        chunks = [it.rows.reshape(-1, d) for it in self.history if it.kind == "rows"]
        return np.concatenate(chunks, axis=0) if chunks else None

    def lineage_matrix(self, d: int, final_width: int):
        """Per-slot input sequences after composing beam reorders (SP/client.py:154-172)."""
        anc = list(range(final_width))
        collected = [[] for _ in range(final_width)]
        for it in reversed(self.history):
            if it.kind == "reorder":
                anc = [it.parents0[a] for a in anc]
            else:
                for s in range(final_width):
                    collected[s].append(it.rows[anc[s]])
        return np.stack([np.concatenate(list(reversed(ch)), axis=0) for ch in collected])


class SwarmClient:
    def __init__(self, name: str, config, transport, routes: list[ServerRoute], engine,
                 max_reroutes: int = 10):
        self.name = name
        self.config = config
        self.net = transport
        self.routes = list(routes)
        self.engine = engine
        self.graph = RoutingGraph(config.n_blocks)
        self.banned: set[str] = set()
        self.max_reroutes = max_reroutes
        self._sid = 0

    # -- plumbing ------------------------------------------------------------------
    def _new_sid(self) -> int:
        self._sid += 1
        return self._sid

    def refresh_routes(self) -> None:
        self.graph.sync([r for r in self.routes if r.server_id not in self.banned])

    def _ban(self, server_id: str) -> None:
        self.banned.add(server_id)
        self.graph.ban(server_id)

    def _call_stage(self, stage: _Stage, payload):
        try:
            reply = self.net.rpc(self.name, stage.server_id, payload, stage.session_id)
        except (MessageDropped, ConnectionFailed) as e:
            raise _StageFailure(stage.server_id, ban=True, reason=str(e))
        if isinstance(reply, Error):
            if reply.code in ("expired", "desync"):
                raise _StageFailure(stage.server_id, ban=False, reason=reply.code,
                                    recover_in_place=True)
            if reply.code == "capacity":
                raise CapacityError(reply.detail)
            raise _StageFailure(stage.server_id, ban=True, reason=reply.code)
        return reply

    def _blob(self, rows, width: int, n_new: int, quantized: bool) -> HiddenBlob:
        return HiddenBlob.from_array(np.asarray(rows).reshape(width * n_new, -1), quantized)

    def _rows(self, res, width: int, n_new: int):
        if res.blob.synthetic:
            return None
        return res.blob.array().reshape(width, n_new, self.config.hidden_dim)

    def _route_chain(self, start: int, end: int):
        for _ in range(self.max_reroutes):
            self.refresh_routes()
            try:
                return self.graph.find_best_chain(start, end)
            except NoRouteError:
                continue
        raise SwarmUnavailableError(f"no chain for [{start}, {end}) after "
                                    f"{self.max_reroutes} reroutes")

    def _reply_quantized(self, hop: Hop, quantized: bool) -> bool:
        return quantized and hop.end < self.config.n_blocks

    def _request_quantized(self, hop: Hop, quantized: bool) -> bool:
        return quantized and hop.start > 0

    def _open_stage(self, hop: Hop, width: int, quantized: bool) -> _Stage:
        stage = _Stage(hop, self._new_sid())
        self._call_stage(stage, OpenSession(hop.start, hop.end, width,
                                            self._reply_quantized(hop, quantized)))
        return stage

    def _close_stages(self, stages) -> None:
        for s in stages:
            try:
                self.net.post(self.name, s.server_id, Close(), s.session_id)
            except Exception:
                pass

    # -- dual cache core (SP/client.py:310-427) --------------------------------------
    def _step_one_stage(self, stage: _Stage, rows, width: int, n_new: int, quantized: bool,
                        counters: RunCounters):
        blob = self._blob(rows, width, n_new, self._request_quantized(stage.hop, quantized))
        res = self._call_stage(stage, Step(stage.rows_sent, blob, width, n_new))
        counters.messages += 1
        counters.step_activation_bytes += width * n_new * self.config.hidden_dim * 4
        stage.history.append(_HistoryItem("rows", width, n_new,
                                          np.asarray(rows).reshape(width, n_new, -1).copy()))
        stage.rows_sent += n_new
        return self._rows(res, width, n_new)

    def _restore_stage(self, stage: _Stage, hist, t: int, width: int, quantized: bool,
                       counters: RunCounters, want_outputs: bool):
        wire_q = self._request_quantized(stage.hop, quantized)
        blob = (self._blob(hist, width, t, wire_q) if t > 0
                else HiddenBlob.shape_only(0, self.config.hidden_dim))
        res = self._call_stage(stage, Restore(t, blob, width, want_outputs))
        counters.messages += 1
        counters.restore_events.append(
            (stage.hop.start, stage.hop.end, t, width * t * self.config.hidden_dim * 4))
        stage.rows_sent = t
        if want_outputs and t > 0:
            return self._rows(res, width, t)
        return None

    def _replace_failed_stage(self, stages, idx: int, width: int, quantized: bool,
                              counters: RunCounters):
        failed = stages[idx]
        self._ban(failed.server_id)
        counters.recoveries += 1
        d = self.config.hidden_dim
        hist = failed.history_matrix(d) if width == 1 else failed.lineage_matrix(d, width)
        t = failed.rows_sent
        for _ in range(self.max_reroutes):
            counters.reroutes += 1
            seg = self._route_chain(failed.hop.start, failed.hop.end)
            try:
                new_stages = []
                inputs = hist
                for n, hop in enumerate(seg.hops):
                    is_last = n == len(seg.hops) - 1
                    stage = self._open_stage(hop, width, quantized)
                    out = self._restore_stage(stage, inputs, t, width, quantized, counters,
                                              want_outputs=not is_last and t > 0)
                    if t > 0:
                        stage.history = [_HistoryItem(
                            "rows", width, t, np.asarray(inputs).reshape(width, t, d).copy())]
                    new_stages.append(stage)
                    if not is_last:
                        inputs = out
                return new_stages
            except _StageFailure as f2:
                if f2.ban:
                    self._ban(f2.server_id)
        raise SwarmUnavailableError("replacements kept failing")

    def _reopen_in_place(self, stage: _Stage, width: int, quantized: bool,
                         counters: RunCounters) -> None:
        d = self.config.hidden_dim
        hist = stage.history_matrix(d) if width == 1 else stage.lineage_matrix(d, width)
        t = stage.rows_sent
        stage.session_id = self._new_sid()
        # raw `quantized` flag, as the reference does (SP/client.py:424-425)
        self._call_stage(stage, OpenSession(stage.hop.start, stage.hop.end, width, quantized))
        self._restore_stage(stage, hist, t, width, quantized, counters, want_outputs=False)

    def _run_chain_step(self, stages, rows, width: int, n_new: int, quantized: bool,
                        counters: RunCounters):
        idx, current = 0, rows
        while idx < len(stages):
            stage = stages[idx]
            try:
                current = self._step_one_stage(stage, current, width, n_new, quantized, counters)
                idx += 1
            except _StageFailure as f:
                if f.recover_in_place:
                    counters.recoveries += 1
                    try:
                        self._reopen_in_place(stage, width, quantized, counters)
                        continue
                    except _StageFailure:
                        pass
                stages[idx:idx + 1] = self._replace_failed_stage(stages, idx, width, quantized,
                                                                 counters)
        return current

    def _reorder_stages(self, stages, parents0: list, quantized: bool, counters: RunCounters,
                        width: int) -> None:
        """Beam cache reorder on every stage, recorded in the stage history
        (SP/client.py `_reorder_all`)."""
        for idx in range(len(stages)):
            stage = stages[idx]
            try:
                self._call_stage(stage, Reorder([p + 1 for p in parents0]))
            except _StageFailure:
                # the replacement replays the lineage, which already has this reorder
                stage.history.append(_HistoryItem("reorder", len(parents0), 0,
                                                  parents0=list(parents0)))
                stages[idx:idx + 1] = self._replace_failed_stage(stages, idx, len(parents0),
                                                                 quantized, counters)
                continue
            stage.history.append(_HistoryItem("reorder", len(parents0), 0,
                                              parents0=list(parents0)))

    # -- public API ---------------------------------------------------------------------
    def generate(self, prefix: list, n_new: int, quantized: bool = False,
                 teacher_tokens: list | None = None) -> GenerateResult:
        """Greedy generation through the swarm (SP/client.py:431-512, DUAL_CACHE)."""
        if not prefix:
            raise ConfigurationError("prefix must be non-empty")
        if len(prefix) + n_new > self.config.max_seq_len:
            raise CapacityError("prefix + n_new exceeds max_seq_len")
        counters = RunCounters()
        if n_new == 0:
            return GenerateResult(list(prefix), counters)
        chain = self._route_chain(0, self.config.n_blocks)
        while True:
            try:
                stages = [self._open_stage(h, 1, quantized) for h in chain.hops]
                break
            except _StageFailure as f:
                if f.ban:
                    self._ban(f.server_id)
                chain = self._route_chain(0, self.config.n_blocks)
        tokens = list(prefix)
        rows = self.engine.embed_array(prefix).reshape(1, -1, self.config.hidden_dim)
        n_in = len(prefix)
        for _ in range(n_new):
            out = self._run_chain_step(stages, rows, 1, n_in, quantized, counters)
            counters.per_step_bytes.append(n_in * self.config.hidden_dim * 4 * len(stages))
            tok = self.engine.pick(out[0])
            tokens.append(tok)
            feed = tok if teacher_tokens is None else teacher_tokens[len(tokens) - len(prefix) - 1]
            rows = self.engine.embed_array([feed]).reshape(1, 1, -1)
            n_in = 1
        self._close_stages(stages)
        return GenerateResult(tokens, counters)


def build_swarm(engine_factory, config, n_stages: int, replicas: int,
                crash: dict | None = None, transport=None, engine_for=None):
    """A one-process swarm like `build_sim_swarm` (SP/swarm.py:52-94):
    ``replicas`` servers per stage_intervals span, ids s{stage}{a,b,..}, with
    optional crash injection {server_id: crash_after_messages}.
    ``engine_for(server_id, stage, replica)`` gives a server its own engine
    (e.g. one GPU per server); otherwise all share ``engine_factory()``."""
    from .balancer import stage_intervals
    from .server import BlockServer, ServerCfg
    from .transport import LocalTransport
    net = transport or LocalTransport()
    servers, routes = {}, []
    eng = engine_factory() if engine_for is None else None
    for si, (a, b) in enumerate(stage_intervals(config.n_blocks, n_stages)):
        for r in range(replicas):
            sid = f"s{si}{chr(ord('a') + r)}"
            e = eng if engine_for is None else engine_for(sid, si, r)
            srv = BlockServer(ServerCfg(sid, b - a, a,
                                        crash_after_messages=(crash or {}).get(sid)), e, net)
            servers[sid] = srv
            net.register(sid, srv)
            routes.append(ServerRoute(sid, a, b))
    return net, servers, routes
