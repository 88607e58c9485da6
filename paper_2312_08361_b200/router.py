"""Chain routing over block boundaries — restatement of the query semantics of
`SP/router.py:52-162`: a server holding [a, b) contributes an edge i -> j for
every a <= i < j <= b with weight rtt + (j - i) * 1000 / throughput ms; the
chain is the minimum-cost path, ties resolved exactly like the reference
(servers visited in sorted id order, strict improvement only)."""

from __future__ import annotations

from dataclasses import dataclass

from .errors import NoRouteError, ProtocolError

_INF = float("inf")


@dataclass(frozen=True)
class ServerRoute:
    server_id: str
    start: int
    end: int
    throughput: float = 100.0
    rtt_ms: float = 5.0


@dataclass
class Hop:
    server_id: str
    start: int
    end: int
    cost_ms: float


@dataclass
class Chain:
    hops: list
    cost_ms: float

    def server_ids(self) -> list[str]:
        return [h.server_id for h in self.hops]


class RoutingGraph:
    def __init__(self, n_blocks: int):
        self.n_blocks = n_blocks
        self.servers: dict[str, ServerRoute] = {}

    def sync(self, routes: list[ServerRoute]) -> None:
        self.servers = {r.server_id: r for r in routes}

    def ban(self, server_id: str) -> None:
        self.servers.pop(server_id, None)

    def find_best_chain(self, start: int = 0, end: int | None = None) -> Chain:
        end = self.n_blocks if end is None else end
        if not (0 <= start < end <= self.n_blocks):
            raise ProtocolError(f"needed interval [{start}, {end}) out of range")
        n = end - start
        g = [_INF] * n + [0.0]
        choice: list = [None] * (n + 1)
        for i in range(end - 1, start - 1, -1):            # SP/router.py:131-140
            best, pick = _INF, None
            for sid in sorted(self.servers):
                r = self.servers[sid]
                if not (r.start <= i < r.end):
                    continue
                per_block = 1000.0 / r.throughput
                for j in range(i + 1, min(r.end, end) + 1):
                    c = r.rtt_ms + (j - i) * per_block + g[j - start]
                    if c < best:
                        best, pick = c, (sid, j)
            g[i - start] = best
            choice[i - start] = pick
        if g[0] == _INF:
            raise NoRouteError(f"no chain covers [{start}, {end})")
        hops, i = [], start
        while i < end:
            sid, j = choice[i - start]
            r = self.servers[sid]
            hops.append(Hop(sid, i, j, r.rtt_ms + (j - i) * 1000.0 / r.throughput))
            i = j
        return Chain(hops, g[0])
