"""Block assignment — restatement of the reference's placement policy
(`SP/balancer.py:39-149, 288-319`, `SP/swarm.py:40-49`).

These decide which GPU serves which span; the results are integer intervals
and must be bit-identical to the reference's, which
tests/test_balancer.py checks against the golden vectors.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ConfigurationError

STATE_ONLINE = "online"
STATE_JOINING = "joining"
STATE_OFFLINE = "offline"


@dataclass
class ServerInfo:
    """Directory record of one server (`SP/directory.py` ServerInfo)."""

    server_id: str
    address: str
    start: int
    end: int
    throughput: float
    state: str = STATE_ONLINE
    announced_at: float = 0.0


@dataclass
class RebalanceConfig:
    threshold_pct: float = 20.0
    check_period_s: float = 60.0

    def __post_init__(self) -> None:
        if self.threshold_pct <= 0:
            raise ConfigurationError("rebalance threshold must be > 0")


def stage_intervals(n_blocks: int, n_stages: int) -> list[tuple[int, int]]:
    """Near-even contiguous spans (SP/swarm.py:40-49): the first
    n_blocks % n_stages spans get one extra block."""
    base, extra = divmod(n_blocks, n_stages)
    out, at = [], 0
    for s in range(n_stages):
        size = base + (1 if s < extra else 0)
        out.append((at, at + size))
        at += size
    return out


def block_load(snapshot: list[ServerInfo], n_blocks: int) -> list[float]:
    """t_i per block (SP/directory.py:88-97), servers in id order."""
    t = [0.0] * n_blocks
    for r in sorted(snapshot, key=lambda r: r.server_id):
        if r.state == STATE_OFFLINE:
            continue
        for i in range(r.start, min(r.end, n_blocks)):
            t[i] += r.throughput
    return t


def choose_start(n_blocks: int, capacity: int, loads: list[float]) -> int:
    """Eq. 1 window (SP/balancer.py:39-67): lexicographically smallest sorted
    window load vector, leftmost on ties."""
    if not (1 <= capacity <= n_blocks):
        raise ConfigurationError(f"capacity {capacity} not in [1, {n_blocks}]")
    if len(loads) != n_blocks:
        raise ConfigurationError("load vector length != n_blocks")
    n_windows = n_blocks - capacity + 1
    if n_windows * capacity >= 256:
        arr = np.asarray(loads, dtype=np.float64)
        keys = np.sort(np.lib.stride_tricks.sliding_window_view(arr, capacity), axis=1)
        order = np.lexsort((np.arange(n_windows),)
                           + tuple(keys[:, c] for c in range(capacity - 1, -1, -1)))
        return int(order[0])
    best_start, best_key = 0, sorted(loads[0:capacity])
    for start in range(1, n_windows):
        key = sorted(loads[start:start + capacity])
        if key < best_key:
            best_key, best_start = key, start
    return best_start


def swarm_throughput(snapshot: list[ServerInfo], n_blocks: int) -> float:
    """Bottleneck rate over blocks (SP/balancer.py:70-79)."""
    cover = [0.0] * n_blocks
    for r in snapshot:
        if r.state != STATE_ONLINE:
            continue
        for i in range(r.start, min(r.end, n_blocks)):
            cover[i] += r.throughput
    return min(cover) if cover else 0.0


def greedy_fixpoint(snapshot: list[ServerInfo], n_blocks: int,
                    max_sweeps: int | None = None) -> list[ServerInfo]:
    """Cascade simulation (SP/balancer.py:90-118)."""
    state = {r.server_id: ServerInfo(r.server_id, r.address, r.start, r.end, r.throughput,
                                     r.state, r.announced_at)
             for r in snapshot if r.state != STATE_OFFLINE}
    order = sorted(state)
    limit = max_sweeps if max_sweeps is not None else 2 * max(1, len(order))
    for _ in range(limit):
        moved = False
        loads = block_load(list(state.values()), n_blocks)
        for sid in order:
            rec = state[sid]
            cap = rec.end - rec.start
            for b in range(rec.start, rec.end):
                loads[b] -= rec.throughput
            start = choose_start(n_blocks, cap, loads)
            if start != rec.start:
                rec.start, rec.end = start, start + cap
                rec.state = STATE_ONLINE
                moved = True
            for b in range(rec.start, rec.end):
                loads[b] += rec.throughput
        if not moved:
            break
    return list(state.values())


def propose_rebalance(self_id: str, snapshot: list[ServerInfo], n_blocks: int,
                      config: RebalanceConfig) -> tuple[int, int] | None:
    """Move only if the simulated eventual throughput beats the current one by
    the threshold (SP/balancer.py:121-149)."""
    me = next((r for r in snapshot if r.server_id == self_id), None)
    if me is None or me.state == STATE_OFFLINE:
        return None
    cap = me.end - me.start
    loads = block_load([r for r in snapshot if r.server_id != self_id], n_blocks)
    start = choose_start(n_blocks, cap, loads)
    if start == me.start:
        return None
    current = swarm_throughput(snapshot, n_blocks)
    hyp = [ServerInfo(r.server_id, r.address, r.start, r.end, r.throughput, r.state,
                      r.announced_at) for r in snapshot]
    for r in hyp:
        if r.server_id == self_id:
            r.start, r.end, r.state = start, start + cap, STATE_ONLINE
    eventual = swarm_throughput(greedy_fixpoint(hyp, n_blocks), n_blocks)
    if eventual >= (1.0 + config.threshold_pct / 100.0) * current and eventual > 0:
        return (start, start + cap)
    return None


def greedy_join_assignment(servers: list[tuple[int, float]], n_blocks: int,
                           order: list[int] | None = None):
    """Servers join one at a time under the placement rule (SP/balancer.py:288-303)."""
    loads = [0.0] * n_blocks
    assign: dict[int, tuple[int, int]] = {}
    for i in (order if order is not None else range(len(servers))):
        cap, thr = min(servers[i][0], n_blocks), servers[i][1]
        s = choose_start(n_blocks, cap, loads)
        assign[i] = (s, s + cap)
        for b in range(s, s + cap):
            loads[b] += thr
    value = min((sum(servers[i][1] for i, (s, e) in assign.items() if s <= b < e)
                 for b in range(n_blocks)), default=0.0)
    return assign, value


def greedy_swarm_assignment(servers: list[tuple[int, float]], n_blocks: int,
                            order: list[int] | None = None):
    """Join, then iterate the rule to its fixpoint (SP/balancer.py:306-319)."""
    assign, _ = greedy_join_assignment(servers, n_blocks, order)
    snap = [ServerInfo(f"s{i:03d}", f"s{i:03d}", assign[i][0], assign[i][1], servers[i][1])
            for i in assign]
    fixed = greedy_fixpoint(snap, n_blocks)
    out = {int(r.server_id[1:]): (r.start, r.end) for r in fixed}
    value = min((sum(servers[i][1] for i, (s, e) in out.items() if s <= b < e)
                 for b in range(n_blocks)), default=0.0)
    return out, value


def gpu_span_plan(n_blocks: int, n_gpus: int, method: str = "even") -> list[tuple[int, int]]:
    """Span per GPU for a one-box swarm.  "even" = stage_intervals (the
    reference's build_sim_swarm split); "greedy" = equal-capacity servers
    joining under the Eq. 1 rule then settling at the fixpoint."""
    if method == "even":
        return stage_intervals(n_blocks, n_gpus)
    cap = -(-n_blocks // n_gpus)
    assign, _ = greedy_swarm_assignment([(cap, 1.0)] * n_gpus, n_blocks)
    return [assign[i] for i in range(n_gpus)]
