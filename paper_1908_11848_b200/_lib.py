"""ctypes binding of libdssp_ps.so (include/dssp_ps.h).

The product path has exactly one implementation: the CUDA engine behind this
C-ABI. If the shared library is missing or no GPU is visible, every entry
point raises -- there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DSSP_PS_LIB") or os.path.join(HERE, "libdssp_ps.so")  # env: profiling builds
HEADER = os.path.join(os.path.dirname(HERE), "include", "dssp_ps.h")

MAX_WORKERS = 64
BSP, ASP, SSP, DSSP = 0, 1, 2, 3
PARADIGMS = {"bsp": BSP, "asp": ASP, "ssp": SSP, "dssp": DSSP}
F32, F64 = 0, 1

OK, REJECTED = 0, 1
E_PROTOCOL, E_VALUE, E_DIVERGED, E_CUDA, E_DEADLOCK, E_BUDGET, E_TIMEOUT = -1, -2, -3, -4, -5, -6, -7

GRAD_BOWL, GRAD_SYNTHETIC = 0, 1
EVENT_KINDS = ("compute_done", "push_arrive", "grant_deliver", "pull_arrive", "pull_return")


class PSConfig(ctypes.Structure):
    _fields_ = [("paradigm", ctypes.c_int32), ("worker_count", ctypes.c_int32),
                ("s_lower", ctypes.c_int32), ("r_max", ctypes.c_int32),
                ("learning_rate", ctypes.c_double), ("dimension", ctypes.c_int64),
                ("device", ctypes.c_int32), ("reserved", ctypes.c_int32 * 7)]


class PSGateState(ctypes.Structure):
    _fields_ = [("paradigm", ctypes.c_int32), ("worker_count", ctypes.c_int32),
                ("s_lower", ctypes.c_int32), ("r_max", ctypes.c_int32),
                ("threshold", ctypes.c_int32), ("_pad", ctypes.c_int32),
                ("clocks", ctypes.c_int64 * MAX_WORKERS),
                ("latest", ctypes.c_double * MAX_WORKERS),
                ("previous", ctypes.c_double * MAX_WORKERS),
                ("populated", ctypes.c_int64 * MAX_WORKERS),
                ("credits", ctypes.c_int64 * MAX_WORKERS),
                ("deferred", ctypes.c_uint64), ("version", ctypes.c_int64),
                ("rejected", ctypes.c_int64), ("decisions", ctypes.c_int64)]


class PSSimConfig(ctypes.Structure):
    _fields_ = [("budget", ctypes.c_int32), ("grad_kind", ctypes.c_int32),
                ("loss_every", ctypes.c_int32), ("n_synthetic", ctypes.c_int32),
                ("comm_delay", ctypes.c_double), ("compute_time", ctypes.c_void_p),
                ("center", ctypes.c_void_p), ("center_dtype", ctypes.c_int32),
                ("record_trace", ctypes.c_int32), ("synthetic", ctypes.c_void_p),
                ("max_events", ctypes.c_int64), ("data_ctas", ctypes.c_int32),
                ("reset_gate", ctypes.c_int32), ("mode", ctypes.c_int32), ("_pad", ctypes.c_int32),
                ("time_scale", ctypes.c_double), ("deadline_s", ctypes.c_double)]


class PSSimResult(ctypes.Structure):
    _fields_ = [("events", ctypes.c_int64), ("pushes", ctypes.c_int64),
                ("applied", ctypes.c_int64), ("rejected", ctypes.c_int64),
                ("trace_rows", ctypes.c_int64), ("loss_samples", ctypes.c_int64),
                ("unfinished", ctypes.c_uint64), ("status", ctypes.c_int32),
                ("diverged_worker", ctypes.c_int32), ("device_ms", ctypes.c_double),
                ("control_ms", ctypes.c_double), ("data_ms", ctypes.c_double)]


class PSTraceRow(ctypes.Structure):
    _fields_ = [("time", ctypes.c_double), ("worker", ctypes.c_int32),
                ("kind", ctypes.c_int32), ("count", ctypes.c_int64),
                ("decision", ctypes.c_int32), ("_pad", ctypes.c_int32),
                ("released", ctypes.c_uint64)]


_P = ctypes.c_void_p
_I32, _I64, _D = ctypes.c_int32, ctypes.c_int64, ctypes.c_double
_PI32, _PI64, _PU64, _PD = (ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int64),
                            ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_double))

# name -> (restype, argtypes); the complete export list of include/dssp_ps.h
SIGNATURES = {
    "ps_create": (ctypes.c_int, [ctypes.POINTER(PSConfig), _P, _I32, ctypes.POINTER(_P)]),
    "ps_destroy": (None, [_P]),
    "ps_last_error": (ctypes.c_char_p, [_P]),
    "ps_device_count": (ctypes.c_int, [_PI32]),
    "ps_apply": (ctypes.c_int, [_P, _I32, _P, _I32, _I32, _PI32]),
    "ps_decide": (ctypes.c_int, [_P, _I32, _D, _PI32, _PU64]),
    "ps_push": (ctypes.c_int, [_P, _I32, _P, _I32, _I32, _D, _PI32, _PI32, _PU64]),
    "ps_pull": (ctypes.c_int, [_P, _I32, _P, _I32, _I32, _PI64]),
    "ps_read_weights": (ctypes.c_int, [_P, _P, _I32, _I32, _PI64]),
    "ps_get_state": (ctypes.c_int, [_P, ctypes.POINTER(PSGateState)]),
    "ps_set_state": (ctypes.c_int, [_P, ctypes.POINTER(PSGateState)]),
    "ps_peek_state": (ctypes.c_int, [_P, ctypes.POINTER(PSGateState)]),
    "ps_controller_batch": (ctypes.c_int, [_I32, _P, _P, _I32, _P]),
    "ps_apply_vectors": (ctypes.c_int, [_I32, _P, _P, _I32, _I64, _D, _P, _PI32]),
    "ps_sim_run": (ctypes.c_int, [_P, ctypes.POINTER(PSSimConfig), ctypes.POINTER(PSSimResult)]),
    "ps_sim_trace": (ctypes.c_int, [_P, ctypes.POINTER(PSTraceRow), _I64, _PI64]),
    "ps_abort": (ctypes.c_int, [_P]),
    "ps_replay_run": (ctypes.c_int, [_P, _P, _I64, _P, _I32, _I32, _I32, ctypes.POINTER(PSSimResult)]),
    "ps_replay_decisions": (ctypes.c_int, [_P, _PI64, _I64, _PI64]),
    "ps_replay_read_replica": (ctypes.c_int, [_P, _I32, _I32, _P]),
    "ps_replay_ceiling": (ctypes.c_int, [_P, _I32, _I32, _I32, _PD]),
    "ps_sim_losses": (ctypes.c_int, [_P, _PI64, _PD, _I64, _PI64]),
    "ps_last_kernel_ms": (ctypes.c_int, [_P, _PD]),
    "ps_set_profiling": (ctypes.c_int, [_P, _I32]),
    "ps_profile_floor": (ctypes.c_int, [_P, _PD]),
    "ps_set_producer_stream": (ctypes.c_int, [_P, _P]),
    "ps_set_resident": (ctypes.c_int, [_P, _I32]),
    "ps_workers_start": (ctypes.c_int, [_P, _I64, _D]),
    "ps_bind_worker_stream": (ctypes.c_int, [_P, _I32, _P, _P, _P]),
    "ps_enqueue_iteration": (ctypes.c_int, [_P, _I32, _P, ctypes.c_uint64]),
    "ps_worker_record": (ctypes.c_int, [_P, _I32, _P, _I64]),
    "ps_workers_status": (ctypes.c_int, [_P, _P]),
    "ps_workers_log": (ctypes.c_int, [_P, _P, _I64, _P, _I64, _PI64, _PI64]),
    "ps_workers_abort": (ctypes.c_int, [_P]),
    "ps_shard_create": (ctypes.c_int, [ctypes.POINTER(PSConfig), _I32, _I32, _P, _I64,
                                       ctypes.POINTER(_P)]),
    "ps_shard_ipc_handles": (ctypes.c_int, [_P, _P, _I64]),
    "ps_shard_connect": (ctypes.c_int, [_P, _P, _I64]),
    "ps_shard_destroy": (None, [_P]),
    "ps_shard_disconnect": (ctypes.c_int, [_P]),
    "ps_shard_last_error": (ctypes.c_char_p, [_P]),
    "ps_shard_update_buffer": (ctypes.c_int, [_P, ctypes.POINTER(_P), _PI64]),
    "ps_shard_replica_buffer": (ctypes.c_int, [_P, ctypes.POINTER(_P), _PI64]),
    "ps_shard_run": (ctypes.c_int, [_P, _I64, _I32, _P, _P, _PD]),
    "ps_shard_run_groups": (ctypes.c_int, [_P, _I64, _I32, _P, _P, _P, _PD]),
    "ps_shard_read_shard": (ctypes.c_int, [_P, _P, _PI64]),
    "ps_shard_read_replica": (ctypes.c_int, [_P, _P]),
    "ps_shard_get_state": (ctypes.c_int, [_P, ctypes.POINTER(PSGateState)]),
    "ps_shard_trace": (ctypes.c_int, [_P, ctypes.POINTER(PSTraceRow), _I64, _PI64]),
    "ps_shard_range": (ctypes.c_int, [_I64, _I32, _I32, _PI64, _PI64]),
    "ps_shard_set_profiling": (ctypes.c_int, [_P, _I32]),
    "ps_shard_stream_probe": (ctypes.c_int, [_P, _I32, _PD]),
    "ps_shard_phase_ms": (ctypes.c_int, [_P, _PD]),
}

_lib = None
_lock = threading.Lock()


class EngineUnavailable(RuntimeError):
    """The CUDA engine (libdssp_ps.so or a GPU) is missing: no fallback exists."""


def load(require_gpu: bool = True):
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise EngineUnavailable(
                    f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
            L = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(L, name, None)
                if fn is None:
                    continue
                fn.restype = res
                fn.argtypes = args
            _lib = L
    if require_gpu:
        n = ctypes.c_int32(0)
        _lib.ps_device_count(ctypes.byref(n))
        if n.value < 1:
            raise EngineUnavailable("no CUDA device visible: the engine has no CPU fallback")
    return _lib


def declared_symbols():
    """Function names declared in include/dssp_ps.h."""
    import re
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|const char\*)\s+(ps_\w+)\s*\(", text, re.M)))
