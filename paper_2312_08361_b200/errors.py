"""The one error class the engine raises itself: a request the span cannot
serve.  The reference engine protocol raises `ProtocolError` (SP/errors.py:24;
SURVEY.md §8b) and its BlockServer lets engine exceptions propagate, so only
the name and meaning matter to callers."""


class ProtocolError(Exception):
    """Invalid request for the span engine (SP/errors.py:24)."""
