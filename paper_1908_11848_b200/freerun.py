"""Free-running workers on device flags (north star (4)).

The reference's threaded runner (runner.py:168-291) gives every worker an OS
thread and serializes apply -> decide -> (park on a release Event) -> pull
through one lock. Here every worker is a CUDA stream and one training
iteration is captured ONCE as a CUDA graph:

    forward + backward            (PyTorch, gradients into the flat buffer)
    [device busy-wait]            (optional 1x/2x/4x throttle, runner.py:185-189)
    push kernel                   (ticket, apply in ticket order, gate decision
                                   at the device clock, go flags of the granted
                                   and released workers)
    wait go[p] == 1               (cuStreamWaitValue32: a deferred worker's
                                   stream blocks here, no SM and no host thread)
    pull kernel                   (ticket, weights into the parameters)

The host then enqueues every iteration's graph launch up front and never
synchronizes until the run is over: grants and releases happen entirely on
the device (include/dssp_ps.h, ps_enqueue_iteration).
"""

from __future__ import annotations

import ctypes
import os
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .engine import raise_for

# Streams that block on device flags must not share a hardware queue with the
# streams that release them. Effective only if set before CUDA initializes.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")


class PSWorkersReport(ctypes.Structure):
    _fields_ = [("tickets", ctypes.c_int64), ("decisions", ctypes.c_int64),
                ("pulls", ctypes.c_int64), ("go_mask", ctypes.c_uint64),
                ("status", ctypes.c_int32), ("diverged_worker", ctypes.c_int32),
                ("aborted", ctypes.c_int32), ("_pad", ctypes.c_int32)]


DECISION_DTYPE = np.dtype([("ticket", np.uint64), ("now", np.float64), ("worker", np.int32),
                           ("outcome", np.int32), ("released", np.uint64), ("version", np.int64),
                           ("applied", np.int32), ("_pad", np.int32)])
PULL_DTYPE = np.dtype([("ticket", np.uint64), ("now", np.float64), ("worker", np.int32),
                       ("_pad", np.int32), ("version", np.int64)])


@dataclass
class FreeRunReport:
    decisions: np.ndarray          # DECISION_DTYPE rows in ticket order
    pulls: np.ndarray              # PULL_DTYPE rows in ticket order
    wall_s: float
    status: int
    aborted: bool = False
    iterations: dict = field(default_factory=dict)
    stuck: list = field(default_factory=list)   # workers still blocked at the deadline

    @property
    def pushes(self) -> int:
        return int(self.decisions.size)

    @property
    def iters_per_s(self) -> float:
        return self.pushes / self.wall_s if self.wall_s > 0 else 0.0

    def decision_sequence(self):
        """[(worker, now, outcome, released ids)] in the order the gate saw them."""
        out = []
        for r in self.decisions:
            rel = int(r["released"])
            out.append((int(r["worker"]), float(r["now"]), "grant" if r["outcome"] == 0 else "defer",
                        tuple(q for q in range(64) if (rel >> q) & 1)))
        return out

    def wait_s(self, worker):
        """Gate time worker `worker` spent deferred: from each of its defers to
        the grant that released it (runner.py:243-263's park interval)."""
        total, since = 0.0, None
        for w, now, outcome, released in self.decision_sequence():
            if w == worker and outcome == "defer":
                since = now
            elif since is not None and worker in released:
                total += now - since
                since = None
        return total

    def defers(self, worker=None):
        return sum(1 for w, _, o, _ in self.decision_sequence()
                   if o == "defer" and (worker is None or w == worker))

    def max_staleness(self):
        """max over grants of (max clock - pusher clock) after the push, the
        runner's staleness figure (runner.py:235-239)."""
        clocks, worst = {}, 0
        for w, _, _, _ in self.decision_sequence():
            clocks[w] = clocks.get(w, 0) + 1
            worst = max(worst, max(clocks.values()) - clocks[w])
        return worst


class FreeRunningCluster:
    """P workers behind one engine, gated by device flags.

    ``workers`` are objects with ``.params`` / ``.grads`` (flat fp32 CUDA
    buffers, 16-byte aligned) and ``.step()`` (forward + backward writing the
    gradient buffer on the current stream), e.g. workers.TorchWorker. A worker
    runs on the GPU its buffers live on: the engine's GPU, or a peer GPU of the
    same box (its push / pull kernels then reach the server over NVLink).
    """

    def __init__(self, engine, workers, throttle_ns=None, graphs=True, time_scale=1.0,
                 log_cap=1 << 16):
        import torch
        self.engine = engine
        self.lib = engine.lib
        self.workers = list(workers)
        self.P = len(self.workers)
        if self.P != engine.worker_count:
            raise ValueError("one worker per engine worker slot")
        self.throttle_ns = [int(x) for x in (throttle_ns or [0] * self.P)]
        self.graphs = graphs
        self.time_scale = float(time_scale)
        self.log_cap = int(log_cap)
        self.devices = [wk.params.device for wk in self.workers]
        self.streams = [torch.cuda.Stream(device=dev) for dev in self.devices]
        self._graphs = [None] * self.P
        self._check(self.lib.ps_workers_start(engine.handle, self.log_cap, self.time_scale))
        for p, wk in enumerate(self.workers):
            self._check(self.lib.ps_bind_worker_stream(engine.handle, p, self.streams[p].cuda_stream,
                                                       wk.grads.data_ptr(), wk.params.data_ptr()))

    def _check(self, rc):
        raise_for(rc, self.engine.error())

    def record(self, worker, ring):
        """Keep a copy of every update `worker` pushes (diagnostics/parity)."""
        self._check(self.lib.ps_worker_record(self.engine.handle, worker,
                                              ring.data_ptr() if ring is not None else None,
                                              ring.shape[0] if ring is not None else 0))

    def _iteration(self, p, stream_ptr):
        self.workers[p].step()
        self._check(self.lib.ps_enqueue_iteration(self.engine.handle, p, stream_ptr,
                                                  self.throttle_ns[p]))

    def capture(self, warmup=3):
        """Warm the workers' kernels (cuDNN autotuning) without touching the
        server, then capture one iteration per worker as a CUDA graph."""
        import torch
        for p, wk in enumerate(self.workers):
            with torch.cuda.device(self.devices[p]), torch.cuda.stream(self.streams[p]):
                for _ in range(warmup):
                    wk.step()
        self._sync_all()
        if not self.graphs:
            return
        for p in range(self.P):
            with torch.cuda.device(self.devices[p]):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=self.streams[p]):
                    self._iteration(p, torch.cuda.current_stream().cuda_stream)
            self._graphs[p] = g
        self._sync_all()

    def _sync_all(self):
        import torch
        for dev in sorted({d.index for d in self.devices} | {self.engine.device}):
            torch.cuda.synchronize(dev)

    def run(self, iterations, restart=True, deadline_s=120.0):
        """`iterations` per worker, every launch enqueued up front, one host
        wait at the end. The wait polls the worker streams; past `deadline_s`
        the run is aborted like the runner's deadline_guard (runner.py:294-298:
        every go flag raised, later kernels only advance the ticket) and the
        report comes back with ``aborted`` set and ``stuck`` naming the workers
        whose streams had not finished -- a blocked stream never hangs the
        host. Returns a FreeRunReport."""
        import torch
        if restart:
            self._check(self.lib.ps_workers_start(self.engine.handle, self.log_cap, self.time_scale))
        self._sync_all()
        t0 = time.perf_counter()
        for _ in range(int(iterations)):
            for p in range(self.P):
                with torch.cuda.device(self.devices[p]), torch.cuda.stream(self.streams[p]):
                    if self._graphs[p] is not None:
                        self._graphs[p].replay()
                    else:
                        self._iteration(p, self.streams[p].cuda_stream)
        stuck = self._wait(t0, deadline_s)
        wall = time.perf_counter() - t0
        rep = self.report(wall)
        rep.stuck = stuck
        return rep

    def _wait(self, t0, deadline_s):
        pending = set(range(self.P))
        while pending:
            pending = {p for p in pending if not self.streams[p].query()}
            if not pending:
                break
            if deadline_s is not None and time.perf_counter() - t0 > deadline_s:
                stuck = sorted(pending)
                self.abort()
                self._sync_all()
                return stuck
            time.sleep(50e-6)
        self._sync_all()
        return []

    def report(self, wall=0.0):
        st = PSWorkersReport()
        self._check(self.lib.ps_workers_status(self.engine.handle, ctypes.byref(st)))
        n = min(int(st.decisions), self.log_cap)
        m = min(int(st.pulls), self.log_cap)
        dec = np.zeros(max(n, 1), dtype=DECISION_DTYPE)
        pul = np.zeros(max(m, 1), dtype=PULL_DTYPE)
        nd, npl = ctypes.c_int64(0), ctypes.c_int64(0)
        self._check(self.lib.ps_workers_log(self.engine.handle, dec.ctypes.data, n, pul.ctypes.data, m,
                                            ctypes.byref(nd), ctypes.byref(npl)))
        self.engine.refresh(sync=False)
        rep = FreeRunReport(decisions=dec[:n], pulls=pul[:m], wall_s=wall, status=int(st.status),
                            aborted=bool(st.aborted))
        for p in range(self.P):
            rep.iterations[p] = int(np.sum(rep.decisions["worker"] == p))
        if st.status == _lib.E_TIMEOUT:
            raise RuntimeError("free-running run: a ticket wait hit the device watchdog")
        if st.status != _lib.OK:
            raise_for(int(st.status), f"free-running run stopped (status {st.status}); "
                                      f"diverged worker {st.diverged_worker}")
        return rep

    def abort(self):
        self._check(self.lib.ps_workers_abort(self.engine.handle))
