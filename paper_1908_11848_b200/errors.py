"""The reference's exception classes, re-declared so callers catch the same
names (policy.py:29-30, server.py:20-21, simnet.py:28-31)."""


class ProtocolError(RuntimeError):
    """A worker broke the push/grant/pull protocol."""


class DivergenceError(RuntimeError):
    """Weights went non-finite; the run cannot continue."""


class DeadlockError(RuntimeError):
    def __init__(self, stuck):
        self.stuck = tuple(sorted(stuck))
        super().__init__(f"simulation deadlocked with workers {self.stuck} unfinished")
