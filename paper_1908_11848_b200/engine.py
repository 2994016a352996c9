"""Thin owner of one ps_server handle: status translation, host mirrors.

Everything numeric happens on the GPU behind include/dssp_ps.h; this class
only moves pointers across the C-ABI and turns status codes back into the
reference's exception classes (policy.py:29-30, server.py:20-21, :31-35).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .errors import DeadlockError, DivergenceError, ProtocolError


def raise_for(rc, message, stuck=()):
    if rc in (_lib.OK, _lib.REJECTED):
        return
    if rc == _lib.E_PROTOCOL:
        raise ProtocolError(message)
    if rc == _lib.E_VALUE:
        raise ValueError(message)
    if rc == _lib.E_DIVERGED:
        raise DivergenceError(message)
    if rc == _lib.E_DEADLOCK:
        raise DeadlockError(stuck)
    if rc == _lib.E_BUDGET:
        raise RuntimeError(message)
    raise RuntimeError(f"engine error {rc}: {message}")


def as_f32_host(values):
    arr = np.asarray(values)
    if arr.dtype == np.float64:
        return np.ascontiguousarray(arr), _lib.F64
    return np.ascontiguousarray(arr, dtype=np.float32), _lib.F32


def device_pointer(values):
    """(pointer, dtype) of a CUDA torch tensor, or None for host arrays."""
    if hasattr(values, "data_ptr") and getattr(values, "is_cuda", False):
        if not values.is_contiguous():
            raise ValueError("device updates must be contiguous")
        import torch
        if values.dtype == torch.float32:
            return values.data_ptr(), _lib.F32
        if values.dtype == torch.float64:
            return values.data_ptr(), _lib.F64
        raise ValueError(f"unsupported device dtype {values.dtype}")
    return None


class Engine:
    """One single-GPU server: weights, control block, gate."""

    def __init__(self, paradigm, worker_count, s_lower, r_max, learning_rate, dimension,
                 w0=None, device=0):
        self.lib = _lib.load()
        cfg = _lib.PSConfig()
        cfg.paradigm = _lib.PARADIGMS[paradigm]
        cfg.worker_count = int(worker_count)
        cfg.s_lower = int(s_lower)
        cfg.r_max = int(r_max)
        cfg.learning_rate = float(learning_rate)
        cfg.dimension = int(dimension)
        cfg.device = int(device)
        self.dimension = int(dimension)
        self.worker_count = int(worker_count)
        self.device = int(device)
        self._h = ctypes.c_void_p()
        if w0 is not None:
            w0, dt = as_f32_host(w0)
            if w0.shape != (self.dimension,):
                raise ValueError("initial weights have the wrong dimension")
            rc = self.lib.ps_create(ctypes.byref(cfg), w0.ctypes.data, dt, ctypes.byref(self._h))
        else:
            rc = self.lib.ps_create(ctypes.byref(cfg), None, _lib.F32, ctypes.byref(self._h))
        if rc:
            raise_for(rc, self.lib.ps_last_error(None).decode())
        self._state = _lib.PSGateState()
        self._stale = False
        self.refresh(sync=False)

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            self.lib.ps_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def error(self):
        return self.lib.ps_last_error(self._h).decode()

    def check(self, rc):
        raise_for(rc, self.error())
        return rc

    # -- state ---------------------------------------------------------------
    def refresh(self, sync=True):
        fn = self.lib.ps_get_state if sync else self.lib.ps_peek_state
        self.check(fn(self._h, ctypes.byref(self._state)))
        self._stale = False
        return self._state

    @property
    def state(self):
        """The gate tables as of the last op (the host-mapped mirror the op
        kernels publish into; copied on demand, not after every call)."""
        if self._stale:
            self.lib.ps_peek_state(self._h, ctypes.byref(self._state))
            self._stale = False
        return self._state

    def write_state(self, state):
        self.check(self.lib.ps_set_state(self._h, ctypes.byref(state)))
        self.refresh(sync=False)

    # -- hot path -----------------------------------------------------------
    def _order_after(self, tensor):
        """Device tensors come from (or go to) the caller's current CUDA
        stream: order the server's stream after it (no host sync)."""
        if tensor is None:
            ptr = None
        else:
            import torch
            # handle 0 is the legacy default stream: name it cudaStreamLegacy
            # (0x1), because NULL means "no producer" at the C-ABI
            raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
            ptr = (raw(tensor.device.index) if raw is not None
                   else torch.cuda.current_stream(tensor.device).cuda_stream) or 1
        if ptr != getattr(self, "_producer", None):
            self.lib.ps_set_producer_stream(self._h, ptr)
            self._producer = ptr

    def _gradient_args(self, values):
        dev = device_pointer(values)
        if dev is not None:
            self._order_after(values)
            return dev[0], dev[1], 1, values
        self._order_after(None)
        arr, dt = as_f32_host(values)
        return arr.ctypes.data, dt, 0, arr

    def apply(self, worker, values):
        ptr, dt, on_dev, keep = self._gradient_args(values)
        applied = ctypes.c_int32(0)
        rc = self.lib.ps_apply(self._h, int(worker), ptr, dt, on_dev, ctypes.byref(applied))
        self._stale = True
        self.check(rc)
        return bool(applied.value)

    def decide(self, worker, now):
        granted = ctypes.c_int32(0)
        released = ctypes.c_uint64(0)
        rc = self.lib.ps_decide(self._h, int(worker), float(now), ctypes.byref(granted),
                                ctypes.byref(released))
        self._stale = True
        self.check(rc)
        return bool(granted.value), released.value

    def push(self, worker, values, now):
        ptr, dt, on_dev, keep = self._gradient_args(values)
        applied = ctypes.c_int32(0)
        granted = ctypes.c_int32(0)
        released = ctypes.c_uint64(0)
        rc = self.lib.ps_push(self._h, int(worker), ptr, dt, on_dev, float(now),
                              ctypes.byref(applied), ctypes.byref(granted), ctypes.byref(released))
        self._stale = True
        self.check(rc)
        return bool(applied.value), bool(granted.value), released.value

    def read(self, out=None, worker=None, dtype=np.float32):
        """Materialize the current weights into `out` (host ndarray or CUDA
        tensor) -- a pull when `worker` is given (server.py:84-91)."""
        if out is None:
            out = np.empty(self.dimension, dtype=dtype)
        dev = device_pointer(out)
        if dev is not None:
            ptr, dt, on_dev = dev[0], dev[1], 1
            self._order_after(out)
        else:
            self._order_after(None)
            if not (out.flags.c_contiguous and out.dtype in (np.float32, np.float64)):
                raise ValueError("pull destination must be a contiguous fp32/fp64 array")
            ptr, dt, on_dev = out.ctypes.data, (_lib.F64 if out.dtype == np.float64 else _lib.F32), 0
        version = ctypes.c_int64(0)
        if worker is None:
            rc = self.lib.ps_read_weights(self._h, ptr, dt, on_dev, ctypes.byref(version))
        else:
            rc = self.lib.ps_pull(self._h, int(worker), ptr, dt, on_dev, ctypes.byref(version))
        self.check(rc)
        return out, int(version.value)

    def last_kernel_ms(self):
        ms = ctypes.c_double(0)
        self.lib.ps_last_kernel_ms(self._h, ctypes.byref(ms))
        return ms.value

    def set_resident(self, ctas=16):
        """Serve the per-op calls from a persistent kernel through a host-mapped
        mailbox (no launch / stream sync per call); 0 turns it off."""
        self.check(self.lib.ps_set_resident(self._h, int(ctas)))

    def profile_floor_ms(self):
        """The profiling bracket around an empty kernel (ps_profile_floor)."""
        ms = ctypes.c_double(0)
        self.check(self.lib.ps_profile_floor(self._h, ctypes.byref(ms)))
        return ms.value

    def replay_ceiling_ms(self, pulls, applies, reps=5):
        """The replay's data side with no control (ps_replay_ceiling): best
        device ms of `pulls` stores and `applies` loads+applies per warp."""
        ms = ctypes.c_double(0)
        self.check(self.lib.ps_replay_ceiling(self._h, int(pulls), int(applies), int(reps), ctypes.byref(ms)))
        return ms.value

    def set_profiling(self, on=True):
        """Bracket every per-op launch with CUDA events (last_kernel_ms)."""
        self.lib.ps_set_profiling(self._h, 1 if on else 0)
