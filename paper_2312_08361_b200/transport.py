"""In-process request/response transport between clients and span servers.

A deterministic stand-in for the reference's transports (`SP/netsim.py:154-297`,
`SP/realnet.py`) with exactly the failure semantics the dual-cache path
depends on: a server configured with ``crash_after_messages`` raises
``SimulatedCrash`` on the next message (`SP/server.py:323-325`), the transport
marks it crashed and the caller sees ``ConnectionFailed``
(`SP/netsim.py:262-266`); later calls to it fail the same way.  Link latency,
bandwidth, random drops and churn are simulation features of the reference
harness and are out of scope here.
"""

from __future__ import annotations

from .errors import ConnectionFailed


class SimulatedCrash(Exception):
    """Raised by a server handler to simulate a process crash (SP/netsim.py:109)."""


class VirtualClock:
    """Monotonic simulated time; advanced only explicitly (SP/netsim.py:77-106)."""

    def __init__(self) -> None:
        self.now = 0.0

    def advance(self, dt: float) -> None:
        self.now += max(0.0, dt)


class LocalTransport:
    def __init__(self) -> None:
        self.clock = VirtualClock()
        self._handlers: dict = {}
        self._crashed: set[str] = set()
        self.messages = 0

    def register(self, addr: str, handler) -> None:
        self._handlers[addr] = handler

    def set_crashed(self, addr: str, crashed: bool = True) -> None:
        (self._crashed.add if crashed else self._crashed.discard)(addr)

    def online(self, addr: str) -> bool:
        return addr in self._handlers and addr not in self._crashed

    def rpc(self, src: str, dst: str, payload, session_id: int = 0):
        if not self.online(dst):
            raise ConnectionFailed(f"{dst} is offline")
        self.messages += 1
        try:
            return self._handlers[dst].handle(payload, session_id)
        except SimulatedCrash:
            self._crashed.add(dst)
            raise ConnectionFailed(f"{dst} crashed mid-request")

    def post(self, src: str, dst: str, payload, session_id: int = 0) -> bool:
        """Fire-and-forget (used for Close); failures are ignored by callers."""
        self.rpc(src, dst, payload, session_id)
        return True
