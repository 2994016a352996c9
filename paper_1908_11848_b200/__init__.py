"""paper_1908_11848_b200 -- a B200-native parameter-server engine for the
data-parallel hot path of arXiv 1908.11848 (DSSP): push-apply, pull and the
dynamic-staleness synchronization gate, behind the reference `stalesync`
package's server/policy API.

The numerics run only in the sm_100a CUDA library ``libdssp_ps.so``
(include/dssp_ps.h); Python here is the host-side mirror of the reference
interface. Importing the package does not touch the GPU; the first engine
call does, and raises :class:`EngineUnavailable` if the library or a GPU is
missing (there is no CPU fallback).
"""

from ._lib import EngineUnavailable
from .config import (ConfigError, ExperimentConfig, StalenessRange, TimingSpec, make_config,
                     push_budget, rng_stream, validate_config)
from .errors import DeadlockError, DivergenceError, ProtocolError
from .policy import (DEFER, GRANT, SyncDecision, SyncPolicy, controller_batch,
                     max_staleness_bound, synchronization_controller)
from .server import GradientVector, ParameterServer, WeightVector, apply_update, initial_weights
from .sim import DeviceSimulation, run_device_simulation
from .trace import TraceEntry, decision_token, format_trace

__all__ = [
    "EngineUnavailable", "ConfigError", "ExperimentConfig", "StalenessRange", "TimingSpec",
    "make_config", "validate_config", "push_budget", "rng_stream",
    "DeadlockError", "DivergenceError", "ProtocolError",
    "GRANT", "DEFER", "SyncDecision", "SyncPolicy", "controller_batch",
    "synchronization_controller", "max_staleness_bound",
    "GradientVector", "WeightVector", "ParameterServer", "apply_update", "initial_weights",
    "DeviceSimulation", "run_device_simulation",
    "TraceEntry", "decision_token", "format_trace",
]
