"""Protocol payloads of the session RPCs — the message kinds of `SP/wire.py:47-59`
and their fields (`SP/wire.py:150-230`).  In this build they travel in
process (transport.py) or stay on the device (pipeline.py); the byte framing
and FNV trailer of the TCP transport are out of scope."""

from __future__ import annotations

from dataclasses import dataclass, field

from .blob import HiddenBlob


@dataclass
class OpenSession:
    start: int
    end: int
    width: int = 1
    quantized: bool = False
    client_id: int = 0
    relay_next: str = ""
    client_addr: str = ""


@dataclass
class Step:
    position_offset: int
    blob: HiddenBlob
    width: int = 1
    n_new: int = 1
    checksum: int = 0


@dataclass
class StepResult:
    position_offset: int
    blob: HiddenBlob
    width: int = 1
    n_new: int = 1
    checksum: int = 0


@dataclass
class Restore:
    t: int
    blob: HiddenBlob
    width: int = 1
    want_outputs: bool = True


@dataclass
class Reorder:
    indices: list = field(default_factory=list)    # 1-based slots, length = new width


@dataclass
class Forward:
    req_id: int
    blob: HiddenBlob
    batch: int
    tokens: int
    record: bool = False
    quantize_reply: bool = False


@dataclass
class Backward:
    req_id: int
    blob: HiddenBlob
    batch: int
    tokens: int


@dataclass
class Close:
    pass


@dataclass
class Ping:
    pass


@dataclass
class Pong:
    pass


@dataclass
class Error:
    code: str        # "expired" | "desync" | "capacity" | "not_serving" | "bad_index" | "no_record" | "protocol"
    detail: str = ""
