"""Exception types, mirroring the reference's (names and base classes are part of the drop-in contract)."""


class DegenerateResidualError(ValueError):
    """No residual mass: the target distribution never rejects the draft (accept_model.py:28-29)."""


class CapacityExceededError(ValueError):
    """A fixed-window request does not fit into the verification budget (selector.py:24-25)."""


class OracleSizeExceededError(ValueError):
    """Instance too large for exhaustive enumeration (selector.py:28-29)."""
