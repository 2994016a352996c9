"""Host-side value types and experiment configuration.

The engine keeps the reference package's vocabulary so a caller can hand it
either a reference ``stalesync.config.ExperimentConfig`` (duck-typed: only
attributes are read) or one built here. Mirrors config.py:15-123 (fields and
defaults), :151-181 (``make_config`` flat keys), :242-315 (normalizations used
by the hot path) and :318-328 (seeded per-purpose RNG streams).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field, replace

import numpy as np

PARADIGMS = ("bsp", "asp", "ssp", "dssp")
TIMING_PRESETS = ("homogeneous", "jitter", "gtx-mix", "straggler", "lognormal")
MODEL_KINDS = ("quadratic_bowl", "linear_regression", "logistic_regression", "tiny_mlp")
GTX_MIX_RATIO = 2.2        # simnet.py:23
JITTER_SPREAD = 0.2        # simnet.py:24
LOGNORMAL_SIGMA = 0.25     # simnet.py:25
DEFAULT_LOSS_TARGET = {"quadratic_bowl": 1e-8, "linear_regression": 1e-6,
                       "logistic_regression": 0.5, "tiny_mlp": 0.05}
_RNG_PURPOSES = ("init_weights", "dataset", "shuffle", "timing", "model")


class ConfigError(ValueError):
    """A configuration violates an invariant; the message names the field."""


@dataclass(frozen=True)
class StalenessRange:
    s_lower: int = 0
    r_max: int = 0


@dataclass(frozen=True)
class TimingSpec:
    preset: str = "homogeneous"
    compute_base: float = 1.0
    comm_delay: float = 0.0
    straggler_ratio: float = 3.0
    # Engine extension (not a reference key): per-worker compute multipliers,
    # e.g. (1, 2, 4) for BASELINE configs[3]'s throttled cluster.
    throttle: tuple = ()


@dataclass(frozen=True)
class ExperimentConfig:
    paradigm: str = "bsp"
    mode: str = "simulated"
    worker_count: int = 1
    staleness: StalenessRange = field(default_factory=StalenessRange)
    timing_model: TimingSpec = field(default_factory=TimingSpec)
    model_kind: str = "quadratic_bowl"
    dimension: int = 8
    dataset_size: int = 0
    noise: float = 0.0
    batch_size: int = 8
    learning_rate: float = 0.05
    epochs: int = 1
    seed: int = 0
    loss_target: float = 0.0
    loss_every: int = 1


_STALENESS_KEYS = ("s_lower", "r_max")
_TIMING_KEYS = {"timing_preset": "preset", "compute_base": "compute_base",
                "comm_delay": "comm_delay", "straggler_ratio": "straggler_ratio",
                "throttle": "throttle"}


def make_config(**flat) -> ExperimentConfig:
    """Build a config from the reference's flat key vocabulary."""
    top = {f for f in ExperimentConfig.__dataclass_fields__} - {"staleness", "timing_model"}
    staleness, timing, kwargs = {}, {}, {}
    for key, value in flat.items():
        if key in _STALENESS_KEYS:
            staleness[key] = int(value)
        elif key in _TIMING_KEYS:
            timing[_TIMING_KEYS[key]] = tuple(value) if key == "throttle" else (
                str(value) if key == "timing_preset" else float(value))
        elif key in top:
            kwargs[key] = value
        else:
            raise ConfigError(f"{key}: unknown configuration key")
    if staleness:
        kwargs["staleness"] = StalenessRange(**staleness)
    if timing:
        kwargs["timing_model"] = TimingSpec(**timing)
    return ExperimentConfig(**kwargs)


def validate_config(config) -> ExperimentConfig:
    """The normalizations the hot path depends on (config.py:290-315):
    SSP zeroes r_max, BSP/ASP zero the whole range, dataset_size defaults to
    eight batches per worker and rounds up to a multiple of worker_count, an
    unset loss_target takes the per-model default."""
    if config.paradigm not in PARADIGMS:
        raise ConfigError(f"paradigm: must be one of {', '.join(PARADIGMS)}, got {config.paradigm!r}")
    if not (isinstance(config.worker_count, int) and config.worker_count >= 1):
        raise ConfigError(f"worker_count: must be an integer >= 1, got {config.worker_count!r}")
    if config.staleness.s_lower < 0 or config.staleness.r_max < 0:
        raise ConfigError("staleness: s_lower and r_max must be >= 0")
    if config.learning_rate <= 0:
        raise ConfigError(f"learning_rate: must be > 0, got {config.learning_rate}")
    if config.timing_model.preset not in TIMING_PRESETS:
        raise ConfigError(f"timing_model.preset: unknown {config.timing_model.preset!r}")
    minimum = config.worker_count * config.batch_size
    size = config.dataset_size or max(minimum, 8 * minimum)
    if size < minimum:
        raise ConfigError(f"dataset_size: must be >= worker_count * batch_size = {minimum}")
    if size % config.worker_count:
        size += config.worker_count - size % config.worker_count
    staleness = config.staleness
    if config.paradigm == "ssp":
        staleness = StalenessRange(staleness.s_lower, 0)
    elif config.paradigm in ("bsp", "asp"):
        staleness = StalenessRange(0, 0)
    target = config.loss_target or DEFAULT_LOSS_TARGET.get(config.model_kind, 0.0)
    return replace(config, staleness=staleness, dataset_size=size, loss_target=target,
                   seed=int(config.seed))


def rng_stream(seed: int, purpose: str, worker: int = 0) -> np.random.Generator:
    """Independent stream keyed by (seed, purpose, worker), config.py:318-328."""
    if purpose not in _RNG_PURPOSES:
        raise ValueError(f"unknown rng purpose {purpose!r}")
    seq = np.random.SeedSequence(entropy=int(seed) & (2 ** 64 - 1),
                                 spawn_key=(_RNG_PURPOSES.index(purpose), int(worker)))
    return np.random.default_rng(seq)


def push_budget(config) -> int:
    """engine.py:243-248: pushes per worker."""
    shard = config.dataset_size // config.worker_count
    return math.ceil(config.epochs * shard / config.batch_size)


def compute_time_table(config, budget: int) -> np.ndarray:
    """Every compute-time draw the run will consume, [P, budget] fp64.

    The reference draws worker w's k-th compute time when w adopts its k-th
    pull (simnet.py:156-163) from its own stream rng_stream(seed, "timing", w)
    (simnet.py:34-69), so the per-worker sequences are fixed in advance and
    the device loop can index them by (worker, iteration)."""
    spec = config.timing_model
    P = config.worker_count
    base = spec.compute_base
    if spec.preset == "gtx-mix":
        fast = (P + 1) // 2
        bases = [base if w < fast else GTX_MIX_RATIO * base for w in range(P)]
    elif spec.preset == "straggler":
        bases = [base] * P
        if P > 1:
            bases[P - 1] = spec.straggler_ratio * base
    else:
        bases = [base] * P
    throttle = tuple(getattr(spec, "throttle", ()) or ())
    if throttle:
        bases = [b * float(throttle[w % len(throttle)]) for w, b in enumerate(bases)]
    out = np.empty((P, budget), dtype=np.float64)
    for w in range(P):
        if spec.preset == "jitter":
            rng = rng_stream(config.seed, "timing", w)
            lo, hi = (1.0 - JITTER_SPREAD) * bases[w], (1.0 + JITTER_SPREAD) * bases[w]
            out[w] = [float(rng.uniform(lo, hi)) for _ in range(budget)]
        elif spec.preset == "lognormal":
            rng = rng_stream(config.seed, "timing", w)
            mu = math.log(bases[w])
            out[w] = [float(rng.lognormal(mu, LOGNORMAL_SIGMA)) for _ in range(budget)]
        else:
            out[w] = bases[w]
    return out


def initial_weights_f64(config, dimension: int) -> np.ndarray:
    """server.py:24-26: uniform[-0.5, 0.5) from the "init_weights" stream."""
    return rng_stream(config.seed, "init_weights").uniform(-0.5, 0.5, size=dimension)


def bowl_center(config, dimension: int) -> np.ndarray:
    """engine.py:159-162: QuadraticBowl center from the "model" stream."""
    return rng_stream(config.seed, "model").normal(size=dimension)
