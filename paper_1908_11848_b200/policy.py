"""SyncPolicy drop-in whose decision machine lives on the GPU.

Same surface as stalesync/policy.py (the names a caller or test touches):
``GRANT``/``DEFER``, ``SyncDecision`` (:33-40), ``ProtocolError`` (:29-30),
``SyncPolicy(config).on_push(p, now)`` (:152-170), the tables ``.clocks``
(IterationClockTable, :43-73), ``.history`` (PushHistoryTable, :76-90),
``.credits`` (CreditTable, :93-105) and ``.deferred``, plus
``synchronization_controller`` (:108-132) and ``max_staleness_bound``
(:209-219). The state of record is the device control block; the Python
objects here are views over its host mirror, and writes (tests set credits
or clocks directly, tests/test_policy.py:156-166, :209-220) go back to the
device through ps_set_state.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .engine import Engine
from .errors import ProtocolError

GRANT = "grant"
DEFER = "defer"
INTERVAL_FLOOR = 1e-9


@dataclass(frozen=True)
class SyncDecision:
    outcome: str
    released: tuple = ()

    @property
    def granted(self) -> bool:
        return self.outcome == GRANT


def _mask_to_ids(mask, P):
    return tuple(q for q in range(P) if (mask >> q) & 1)


class _WriteThroughDict(dict):
    """A dict snapshot of one device table; item writes go to the device."""

    def __init__(self, owner, table, data):
        super().__init__(data)
        self._owner, self._table = owner, table

    def __setitem__(self, key, value):
        super().__setitem__(key, value)
        self._owner._write_entry(self._table, key, value)

    def update(self, *args, **kw):
        for k, v in dict(*args, **kw).items():
            self[k] = v


class IterationClockView:
    """IterationClockTable surface (policy.py:43-73) over the device clocks."""

    def __init__(self, policy):
        self._p = policy

    @property
    def counts(self):
        st, P = self._p._engine.state, self._p.worker_count
        return _WriteThroughDict(self._p, "clocks", {w: int(st.clocks[w]) for w in range(P)})

    def __getitem__(self, worker):
        if not 0 <= worker < self._p.worker_count:
            raise KeyError(worker)
        return int(self._p._engine.state.clocks[worker])

    def minimum(self):
        return min(self.counts.values())

    def maximum(self):
        return max(self.counts.values())

    def slowest(self):
        counts = self.counts
        low = min(counts.values())
        return min(w for w, n in counts.items() if n == low)

    def is_fastest(self, worker):
        return self[worker] >= self.maximum()


class PushHistoryView:
    """PushHistoryTable surface (policy.py:76-90), read-only."""

    def __init__(self, policy):
        self._p = policy

    def _table(self, name):
        st = self._p._engine.state
        return {w: getattr(st, name)[w] for w in range(self._p.worker_count)}

    @property
    def latest(self):
        return {w: float(v) for w, v in self._table("latest").items()}

    @property
    def previous(self):
        return {w: float(v) for w, v in self._table("previous").items()}

    @property
    def populated(self):
        return {w: int(v) for w, v in self._table("populated").items()}

    def interval(self, worker):
        return max(self.latest[worker] - self.previous[worker], INTERVAL_FLOOR)


class CreditView:
    """CreditTable surface (policy.py:93-105): non-negative, device-backed."""

    def __init__(self, policy):
        self._p = policy

    @property
    def credits(self):
        st = self._p._engine.state
        return {w: int(st.credits[w]) for w in range(self._p.worker_count)}

    def __getitem__(self, worker):
        return int(self._p._engine.state.credits[worker])

    def __setitem__(self, worker, value):
        if value < 0:
            raise ValueError("credits cannot go negative")
        self._p._write_entry("credits", worker, int(value))


class SyncPolicy:
    """Decision machine for one run on the GPU; callers serialize on_push
    calls (policy.py:136). Constructed standalone it owns a small engine of
    its own; a ParameterServer built without a policy binds one to its own
    engine so handle_push runs apply + decision in one launch."""

    def __init__(self, config, device: int = 0, _engine: Engine | None = None):
        self.paradigm = config.paradigm
        self.worker_count = config.worker_count
        self.s_lower = config.staleness.s_lower
        self.r_max = config.staleness.r_max
        self.threshold = 0 if self.paradigm == "bsp" else self.s_lower
        self._engine = _engine if _engine is not None else Engine(
            self.paradigm, self.worker_count, self.s_lower, self.r_max, 1.0, 4, device=device)
        self.clocks = IterationClockView(self)
        self.history = PushHistoryView(self)
        self.credits = CreditView(self)

    @property
    def deferred(self):
        st = self._engine.state
        return {q for q in range(self.worker_count) if (st.deferred >> q) & 1}

    def _write_entry(self, table, key, value):
        st = self._engine.refresh()
        if not 0 <= key < self.worker_count:
            raise KeyError(key)
        getattr(st, table)[key] = value
        self._engine.write_state(st)

    def on_push(self, p, now) -> SyncDecision:
        granted, released = self._engine.decide(p, now)
        if not granted:
            return SyncDecision(DEFER)
        return SyncDecision(GRANT, _mask_to_ids(released, self.worker_count))

    def decision_from(self, granted, released) -> SyncDecision:
        if not granted:
            return SyncDecision(DEFER)
        return SyncDecision(GRANT, _mask_to_ids(released, self.worker_count))


def controller_batch(tables, r_max, device: int = 0):
    """Run the controller grid on the GPU for many (latest_p, prev_p,
    latest_s, prev_s) rows at once (oracle hook, policy.py:127-132)."""
    lib = _lib.load()
    t = np.ascontiguousarray(tables, dtype=np.float64).reshape(-1, 4)
    r = np.ascontiguousarray(r_max, dtype=np.int32)
    out = np.zeros(len(r), dtype=np.int32)
    rc = lib.ps_controller_batch(int(device), t.ctypes.data, r.ctypes.data, len(r), out.ctypes.data)
    if rc:
        raise RuntimeError(lib.ps_last_error(None).decode())
    return out


def synchronization_controller(history, p, push_time, clocks, r_max, device: int = 0) -> int:
    """policy.py:108-132 on the GPU: records push_time for p, then predicts.
    `history`/`clocks` are PushHistoryTable/IterationClockTable-shaped objects
    (the reference's own tables work)."""
    history.record(p, push_time)
    if r_max <= 0:
        return 0
    slowest = clocks.slowest()
    if history.populated[p] < 2 or history.populated[slowest] < 2:
        return 0
    row = [[history.latest[p], history.previous[p], history.latest[slowest],
            history.previous[slowest]]]
    return int(controller_batch(row, [r_max], device)[0])


def max_staleness_bound(config) -> int:
    """policy.py:209-219."""
    if config.paradigm == "ssp":
        return config.staleness.s_lower
    if config.paradigm == "dssp":
        return config.staleness.s_lower + config.staleness.r_max
    if config.paradigm == "bsp":
        raise ValueError("bsp: staleness bound is 0 by construction")
    if config.paradigm == "asp":
        raise ValueError("asp: staleness is unbounded")
    raise ValueError(f"unknown paradigm {config.paradigm!r}")
