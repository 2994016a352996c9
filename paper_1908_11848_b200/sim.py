"""Device-resident simulated runs: the reference simulator's schedule with the
server hot path (pull, update, apply, gate) executed by one persistent kernel.

``run_device_simulation(config)`` is the drop-in counterpart of
``stalesync.simnet.run_simulation`` (simnet.py:211-218) for the server side
of a run: same (time, seq) event order, same push aggregation, same trace
(byte-identical once rendered with :func:`trace.format_trace`). Worker
compute is replaced by an on-device update generator -- the quadratic bowl
model (engine.py:46-60, g = w_local - c, closed loop) or resident synthetic
N(0,1) buffers -- because the reference's numpy models are outside the hot
path.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .config import bowl_center, compute_time_table, initial_weights_f64, push_budget
from .engine import Engine, raise_for
from .errors import DeadlockError
from .trace import rows_to_entries


@dataclass
class DeviceRunReport:
    entries: list
    events: int
    pushes: int
    applied: int
    rejected: int
    device_ms: float
    version: int
    loss_curve: list = field(default_factory=list)
    final_weights: np.ndarray | None = None
    control_ms: float = 0.0
    data_ms: float = 0.0
    completed: bool = True
    stuck: list = field(default_factory=list)

    @property
    def updates_per_s(self) -> float:
        return self.applied / (self.device_ms * 1e-3) if self.device_ms > 0 else 0.0


def check_synthetic(tensor, workers, count, dimension, device):
    """The C-ABI takes the resident updates as a bare pointer with no length:
    enforce the layout its float4 loads assume ([P, count, round_up(d,4)]
    contiguous fp32 on the engine's device, 16-byte aligned)."""
    import torch
    if not isinstance(tensor, torch.Tensor) or not tensor.is_cuda:
        raise ValueError("resident updates must be a CUDA tensor")
    if tensor.dtype != torch.float32:
        raise ValueError(f"resident updates must be float32, got {tensor.dtype}")
    if tensor.device.index != int(device):
        raise ValueError(f"resident updates live on cuda:{tensor.device.index}, the engine on cuda:{device}")
    want = (int(workers), int(count), (int(dimension) + 3) // 4 * 4)
    if tuple(tensor.shape) != want:
        raise ValueError(f"resident updates must have shape {want}, got {tuple(tensor.shape)}")
    if not tensor.is_contiguous() or tensor.data_ptr() % 16:
        raise ValueError("resident updates must be contiguous and 16-byte aligned")
    if int(count) < 1:
        raise ValueError("at least one resident update per worker")


class DeviceSimulation:
    """Owns one engine and runs simulated schedules on it."""

    def __init__(self, config, dimension=None, grad="bowl", device: int = 0, engine=None):
        self.config = config
        self.dimension = int(dimension if dimension is not None else config.dimension)
        self.grad = grad
        self.device = device
        self.engine = engine or Engine(
            config.paradigm, config.worker_count, config.staleness.s_lower,
            config.staleness.r_max, config.learning_rate, self.dimension,
            w0=initial_weights_f64(config, self.dimension), device=device)
        self.budget = push_budget(config)
        self.ctime = np.ascontiguousarray(compute_time_table(config, self.budget))
        self._center = None
        self._synthetic = None
        self._synth_count = 0
        if grad == "bowl":
            self._center = np.ascontiguousarray(bowl_center(config, self.dimension))
        elif grad != "synthetic":
            raise ValueError("grad must be 'bowl' or 'synthetic'")

    def set_synthetic(self, tensor, count):
        """Resident updates: a CUDA fp32 tensor [P, count, round_up(d, 4)]."""
        check_synthetic(tensor, self.config.worker_count, count, self.dimension, self.engine.device)
        self._synthetic = tensor
        self._synth_count = int(count)

    def run(self, record_trace=True, loss_every=None, max_events=0, data_ctas=0,
            read_weights=True, reset_gate=False, realtime_scale=None, deadline_s=None):
        """One run of the device loop.

        ``realtime_scale`` switches to the free-running mode: every event
        waits for its own wall-clock instant (simulated seconds x scale on
        the GPU's global timer) and pushes are decided at the time they
        actually reach the control warp, so decisions follow real arrival
        order rather than the simulator's aggregated instants
        (server.py:93-128 driven by real workers). ``deadline_s`` bounds the
        run; on expiry (or :meth:`abort`) the report comes back with
        ``completed=False`` and the workers still outstanding in ``stuck``.
        """
        sc = _lib.PSSimConfig()
        sc.budget = self.budget
        sc.grad_kind = _lib.GRAD_BOWL if self.grad == "bowl" else _lib.GRAD_SYNTHETIC
        le = self.config.loss_every if loss_every is None else loss_every
        sc.loss_every = int(le) if self.grad == "bowl" else 0
        sc.n_synthetic = self._synth_count
        sc.comm_delay = float(self.config.timing_model.comm_delay)
        sc.compute_time = self.ctime.ctypes.data
        if self._center is not None:
            sc.center = self._center.ctypes.data
            sc.center_dtype = _lib.F64
        sc.record_trace = 1 if record_trace else 0
        if self._synthetic is not None:
            sc.synthetic = self._synthetic.data_ptr()
        sc.max_events = int(max_events or 0)
        sc.data_ctas = int(data_ctas)
        sc.reset_gate = 1 if reset_gate else 0
        if realtime_scale is not None:
            sc.mode = 2
            sc.time_scale = float(realtime_scale)
            sc.deadline_s = float(deadline_s or 0.0)
        res = _lib.PSSimResult()
        lib = self.engine.lib
        self.engine._order_after(self._synthetic)
        rc = lib.ps_sim_run(self.engine.handle, ctypes.byref(sc), ctypes.byref(res))
        stuck = [q for q in range(self.config.worker_count) if (res.unfinished >> q) & 1]
        if rc == _lib.E_DEADLOCK:
            raise DeadlockError(stuck)
        completed = True
        if rc == _lib.E_TIMEOUT and sc.mode == 2:
            completed = False
        else:
            raise_for(rc, self.engine.error())
        entries = []
        if record_trace:
            n = res.trace_rows
            rows = (_lib.PSTraceRow * max(n, 1))()
            got = ctypes.c_int64(0)
            self.engine.check(lib.ps_sim_trace(self.engine.handle, rows, n, ctypes.byref(got)))
            entries = rows_to_entries(rows, n)
        curve = []
        if sc.loss_every > 0 and res.loss_samples > 0:
            m = res.loss_samples
            vs = (ctypes.c_int64 * m)()
            ls = (ctypes.c_double * m)()
            got = ctypes.c_int64(0)
            self.engine.check(lib.ps_sim_losses(self.engine.handle, vs, ls, m, ctypes.byref(got)))
            curve = [(int(vs[i]), float(ls[i])) for i in range(m)]
        self.engine.refresh(sync=False)  # the run already mirrored the control block
        weights = self.engine.read()[0] if read_weights else None
        return DeviceRunReport(entries=entries, events=res.events, pushes=res.pushes,
                               applied=res.applied, rejected=res.rejected,
                               device_ms=res.device_ms, version=int(self.engine.state.version),
                               loss_curve=curve, final_weights=weights,
                               control_ms=res.control_ms, data_ms=res.data_ms,
                               completed=completed, stuck=stuck if not completed else [])

    def abort(self):
        """Stop a free-running run in flight (callable from another thread)."""
        self.engine.check(self.engine.lib.ps_abort(self.engine.handle))


def run_device_simulation(config, grad="bowl", device: int = 0, **kw):
    return DeviceSimulation(config, grad=grad, device=device).run(**kw)


CALL_PULL, CALL_APPLY, CALL_DECIDE = 0, 1, 2
_CALL_DTYPE = np.dtype([("now", np.float64), ("kind", np.int32), ("worker", np.int32)])


def decode_decisions(raw):
    """Decision words ((released << 8) | outcome) -> [(outcome, released ids)]."""
    out = []
    for v in np.asarray(raw, dtype=np.int64).tolist():
        rel = v >> 8
        ids = []
        q = 0
        while rel:
            if rel & 1:
                ids.append(q)
            rel >>= 1
            q += 1
        out.append(("grant" if (v & 0xff) == 0 else "defer", tuple(ids)))
    return out


@dataclass
class ReplayReport:
    raw: np.ndarray      # one decision word per decide: (released << 8) | outcome
    applied: int
    rejected: int
    pushes: int
    device_ms: float
    control_ms: float = 0.0   # gate warp: start -> last decision (%globaltimer)
    data_ms: float = 0.0      # start -> last data warp done

    @property
    def decisions(self) -> list:
        """[(outcome, released tuple)] per decide (decoded on demand)."""
        return decode_decisions(self.raw)

    @property
    def updates_per_s(self) -> float:
        return self.applied / (self.device_ms * 1e-3) if self.device_ms > 0 else 0.0


class DeviceReplay:
    """The server serving a recorded request stream on the device: the
    reference's boundary calls (see calls_from_trace) replayed in one
    persistent kernel, decisions by the device gate (ps_replay_run)."""

    def __init__(self, engine, calls, synthetic, count):
        self.engine = engine
        arr = np.zeros(len(calls), dtype=_CALL_DTYPE)
        for i, c in enumerate(calls):
            if c[0] == "pull":
                arr[i] = (0.0, CALL_PULL, c[1])
            elif c[0] == "apply":
                arr[i] = (0.0, CALL_APPLY, c[1])
            else:
                arr[i] = (float(c[2]), CALL_DECIDE, c[1])
        self.calls = arr
        check_synthetic(synthetic, engine.worker_count, count, engine.dimension, engine.device)
        self.synthetic = synthetic
        self.count = int(count)

    def run(self, reset_gate=True, data_ctas=0, decisions=True):
        res = _lib.PSSimResult()
        lib = self.engine.lib
        self.engine._order_after(self.synthetic)
        rc = lib.ps_replay_run(self.engine.handle, self.calls.ctypes.data, len(self.calls),
                               self.synthetic.data_ptr(), self.count, 1 if reset_gate else 0,
                               int(data_ctas), ctypes.byref(res))
        raise_for(rc, self.engine.error())
        raw = np.zeros(0, dtype=np.int64)
        if decisions:
            n = res.trace_rows
            raw = np.empty(max(n, 1), dtype=np.int64)
            got = ctypes.c_int64(0)
            self.engine.check(lib.ps_replay_decisions(
                self.engine.handle, raw.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), n,
                ctypes.byref(got)))
            raw = raw[:n]
        self.engine.refresh(sync=False)  # the run already mirrored the control block
        return ReplayReport(raw=raw, applied=res.applied, rejected=res.rejected,
                            pushes=res.pushes, device_ms=res.device_ms, control_ms=res.control_ms,
                            data_ms=res.data_ms)

    def replica(self, worker, buf):
        """The weights pull k of `worker` materialized, for (k + 1) % 2 == buf."""
        return read_replica(self.engine, worker, buf)


def read_replica(engine, worker, buf):
    """Worker `worker`'s replica buffer `buf` after a run (d fp32 values): in a
    replay, pull k (k = 0, 1, ...) of that worker landed in buffer (k + 1) % 2."""
    out = np.empty(engine.dimension, dtype=np.float32)
    engine.check(engine.lib.ps_replay_read_replica(engine.handle, int(worker), int(buf),
                                                   out.ctypes.data))
    return out


def calls_from_trace(entries):
    """The server-call sequence a host driver makes for this trace, in the
    reference's order (simnet.py:127-201): ("pull", w) at PULL_ARRIVE, and for
    every same-instant push group all ("apply", w) first, then each
    ("decide", w, t). Consecutive push_arrive rows at one instant are one
    group (the loop records a group's decisions back to back)."""
    calls = []
    i, n = 0, len(entries)
    while i < n:
        e = entries[i]
        if e.kind == "pull_arrive":
            calls.append(("pull", e.worker))
            i += 1
        elif e.kind == "push_arrive":
            j = i
            while j < n and entries[j].kind == "push_arrive" and entries[j].time == e.time:
                j += 1
            group = entries[i:j]
            calls.extend(("apply", g.worker) for g in group)
            calls.extend(("decide", g.worker, g.time) for g in group)
            i = j
        else:
            i += 1
    return calls
