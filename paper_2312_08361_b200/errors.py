"""Exception hierarchy of the host mirror — same names and meaning as
`SP/errors.py:8-55` so callers written against the reference read the same."""


class SwarmError(Exception):
    """Base of all swarm errors (SP/errors.py:8)."""


class ConfigurationError(SwarmError):
    pass


class CapacityError(SwarmError):
    pass


class StateDesyncError(SwarmError):
    pass


class ProtocolError(SwarmError):
    pass


class TransportError(SwarmError):
    pass


class MessageDropped(TransportError):
    pass


class ConnectionFailed(TransportError):
    pass


class NoRouteError(SwarmError):
    pass


class SwarmUnavailableError(SwarmError):
    pass


class BudgetExhausted(SwarmError):
    pass
