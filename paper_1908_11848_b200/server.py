"""ParameterServer drop-in backed by the B200 engine.

Surface of stalesync/server.py kept name for name: ``DivergenceError``
(:20-21), ``initial_weights`` (:24-26), ``apply_update`` (:29-42),
``ParameterServer(config, dimension, policy=None)`` with ``.weights``,
``.policy``, ``.clocks``, ``.pending``, ``.rejected_updates``,
``apply_gradient`` (:58-69), ``decide_push`` (:71-78), ``handle_push``
(:80-82) and ``handle_pull`` (:84-91).

Differences a caller can observe, both deliberate:
the weights are fp32 on the GPU (``.weights.values`` is a read-only fp32
host copy, fetched lazily and cached per version), and a pull MATERIALIZES
the snapshot at call time -- into a host array, or into a caller-owned CUDA
tensor via ``handle_pull(p, out=tensor)`` -- instead of sharing an immutable
object, which keeps the reference's snapshot isolation
(tests/test_server.py:107-120).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .config import initial_weights_f64
from .engine import Engine, raise_for
from .errors import DivergenceError, ProtocolError
from .policy import SyncDecision, SyncPolicy


def _frozen(values, dtype):
    arr = np.array(values, dtype=dtype)
    arr.flags.writeable = False
    return arr


@dataclass(frozen=True)
class WeightVector:
    """Dense parameters plus the server's update counter (config.py:54-68)."""

    values: np.ndarray
    version: int = 0

    def __post_init__(self):
        if not (isinstance(self.values, np.ndarray) and not self.values.flags.writeable):
            object.__setattr__(self, "values", _frozen(self.values, np.float64))
        if self.version < 0:
            raise ValueError("version must be non-negative")

    @property
    def dimension(self) -> int:
        return self.values.shape[0]


@dataclass(frozen=True)
class GradientVector:
    """A mini-batch update tagged with its worker (config.py:71-85). `values`
    may be a host array or a CUDA tensor (pushed without a host copy)."""

    values: object
    source: int
    source_iter: int = 0

    @property
    def dimension(self) -> int:
        return int(self.values.shape[0])


def initial_weights(config, dimension: int) -> WeightVector:
    return WeightVector(initial_weights_f64(config, dimension), version=0)


def apply_update(weights, g, learning_rate: float, device: int = 0) -> WeightVector:
    """server.py:29-42 as one device pass; returns a new fp32 WeightVector."""
    if learning_rate <= 0:
        raise ValueError("learning_rate must be > 0")
    gd = int(np.asarray(g.values).shape[0])
    if gd != weights.dimension:
        raise ValueError(f"gradient dimension {gd} != weights dimension {weights.dimension}")
    lib = _lib.load()
    w = np.ascontiguousarray(weights.values, dtype=np.float64)
    gv = np.ascontiguousarray(np.asarray(g.values), dtype=np.float64)
    out = np.empty_like(w)
    import ctypes
    status = ctypes.c_int32(0)
    rc = lib.ps_apply_vectors(int(device), w.ctypes.data, gv.ctypes.data, _lib.F64, w.size,
                              float(learning_rate), out.ctypes.data, ctypes.byref(status))
    raise_for(rc, lib.ps_last_error(None).decode())
    if status.value == _lib.E_DIVERGED:
        raise DivergenceError(f"non-finite weights after update {weights.version + 1} "
                              f"from worker {g.source}")
    return WeightVector(_frozen(out.astype(np.float32), np.float32), weights.version + 1)


class ParameterServer:
    """``resident=N`` (N > 0) serves every call from a persistent N-CTA kernel
    through a host-mapped mailbox instead of a launch + stream sync per call
    (include/dssp_ps.h, ps_set_resident)."""

    def __init__(self, config, dimension: int, policy=None, device: int = 0, resident=None):
        self.config = config
        self.dimension = int(dimension)
        self._engine = Engine(config.paradigm, config.worker_count, config.staleness.s_lower,
                              config.staleness.r_max, config.learning_rate, dimension,
                              w0=initial_weights_f64(config, dimension), device=device)
        if policy is None:
            policy = SyncPolicy(config, _engine=self._engine)
        self.policy = policy
        self._fused = isinstance(policy, SyncPolicy) and policy._engine is self._engine
        self.pending: dict = {}
        self._cache = None
        if resident is None:  # PS_RESIDENT: a process-wide default (the tests run both modes)
            import os
            resident = int(os.environ.get("PS_RESIDENT", "0") or 0)
        if resident:
            self._engine.set_resident(resident)

    @property
    def clocks(self):
        return self.policy.clocks

    @property
    def rejected_updates(self) -> int:
        return int(self._engine.state.rejected)

    @property
    def engine(self) -> Engine:
        return self._engine

    @property
    def weights(self) -> WeightVector:
        version = int(self._engine.state.version)
        if self._cache is None or self._cache.version != version:
            values, version = self._engine.read()
            values.flags.writeable = False
            self._cache = WeightVector(values, version)
        return self._cache

    def _dimension_of(self, g):
        return int(g.values.shape[0])

    def apply_gradient(self, g) -> bool:
        """Apply one update; a non-finite update is rejected and counted."""
        if self._dimension_of(g) != self.dimension:
            raise ValueError(f"gradient dimension {self._dimension_of(g)} != weights dimension "
                             f"{self.dimension}")
        return self._engine.apply(g.source, g.values)

    def _bookkeep(self, p, now, decision):
        if decision.granted:
            for released in decision.released:
                self.pending.pop(released, None)
        else:
            self.pending[p] = now
        return decision

    def decide_push(self, p, now) -> SyncDecision:
        return self._bookkeep(p, now, self.policy.on_push(p, now))

    def handle_push(self, g, now) -> SyncDecision:
        if not self._fused:
            self.apply_gradient(g)
            return self.decide_push(g.source, now)
        if self._dimension_of(g) != self.dimension:
            raise ValueError(f"gradient dimension {self._dimension_of(g)} != weights dimension "
                             f"{self.dimension}")
        _, granted, released = self._engine.push(g.source, g.values, now)
        return self._bookkeep(g.source, now, self.policy.decision_from(granted, released))

    def handle_pull(self, p, out=None):
        """Materialized snapshot of the current weights. With `out` (host
        array or CUDA tensor) the copy lands there and (out, version) is
        returned; without it a frozen fp32 WeightVector is."""
        if p not in self.policy.clocks.counts:
            raise ProtocolError(f"unknown worker {p}")
        if p in self.pending:
            raise ProtocolError(f"worker {p} pulled while deferred")
        if out is not None:
            return self._engine.read(out=out)
        values, version = self._engine.read()
        values.flags.writeable = False
        return WeightVector(values, version)
