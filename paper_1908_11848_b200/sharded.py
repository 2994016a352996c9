"""The sharded parameter server: one process per GPU (torchrun), contiguous-range
shards, push/pull over NVLink P2P, replicated device gate.

torch.distributed is plumbing only: it exchanges the CUDA-IPC blobs once at
start-up (all_gather_object), broadcasts the initial weights once over NCCL
(the north star's only collective) and takes the max of the per-rank device
times for the benchmark. A run of steps after that is ONE persistent kernel
per rank that talks to its peers through mapped device memory
(csrc/ps_shard.cu).
"""

from __future__ import annotations

import ctypes
import json
import os
import time

import numpy as np

from . import _lib
from .config import initial_weights_f64, make_config, validate_config
from .engine import raise_for
from .trace import rows_to_entries

BLOB_BYTES = 512


def shard_range(d, world, rank):
    lib = _lib.load(require_gpu=False)
    lo, hi = ctypes.c_int64(0), ctypes.c_int64(0)
    lib.ps_shard_range(int(d), int(world), int(rank), ctypes.byref(lo), ctypes.byref(hi))
    return lo.value, hi.value


def homogeneous_push_times(compute_base, comm_delay, steps):
    """Push instants of the homogeneous schedule, accumulated with the same
    sequence of additions simnet.py performs (PULL_ARRIVE at comm, PULL_RETURN
    +comm, COMPUTE_DONE +compute, PUSH_ARRIVE +comm, then GRANT_DELIVER +comm,
    PULL_ARRIVE +comm, ...), so the gate sees bit-identical timestamps."""
    at = comm_delay
    at = at + comm_delay
    at = at + compute_base
    at = at + comm_delay
    out = [at]
    for _ in range(steps - 1):
        at = at + comm_delay
        at = at + comm_delay
        at = at + comm_delay
        at = at + compute_base
        at = at + comm_delay
        out.append(at)
    return out


GROUP_STRIDE = 18  # PS_SHARD_GROUP_STRIDE (include/dssp_ps.h)


def groups_from_trace(entries):
    """The push groups of a trace (simnet.py:167-201): consecutive
    push_arrive rows at one instant form a group, served in row order; every
    pull_arrive row belongs to the group before it (the weights it snapshots
    are the ones after that group). Pulls before the first group see w0.
    Returns [(time, [workers], [pulling workers])]."""
    groups = []
    open_time = None
    for e in entries:
        if e.kind == "push_arrive":
            if open_time is not None and e.time == open_time and groups:
                groups[-1][1].append(e.worker)
            else:
                groups.append((e.time, [e.worker], []))
                open_time = e.time
        else:
            if e.kind == "pull_arrive" and groups:
                groups[-1][2].append(e.worker)
            open_time = None if e.kind != "push_arrive" else open_time
    return groups


def exchange_blobs(mine: bytes):
    """All-gather every rank's IPC blob, ordered by rank (host plumbing)."""
    import torch.distributed as dist
    everyone = [None] * dist.get_world_size()
    dist.all_gather_object(everyone, mine)
    return everyone


def max_over_ranks(value: float) -> float:
    """Max of a per-rank scalar (device times are reported as max over ranks)."""
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


class _CudaArray:
    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (ptr, False),
                                         "version": 3}


class ShardedServer:
    """Rank-local handle of the G-GPU server. All ranks construct it
    collectively (it all-gathers the IPC blobs)."""

    def __init__(self, config, dimension, rank, world, device, w0_device=None, w0_host=None):
        import torch
        import torch.distributed as dist
        self.lib = _lib.load()
        self.config = config
        self.dimension = int(dimension)
        self.rank, self.world, self.device = int(rank), int(world), int(device)
        cfg = _lib.PSConfig()
        cfg.paradigm = _lib.PARADIGMS[config.paradigm]
        cfg.worker_count = int(config.worker_count)
        cfg.s_lower = int(config.staleness.s_lower)
        cfg.r_max = int(config.staleness.r_max)
        cfg.learning_rate = float(config.learning_rate)
        cfg.dimension = self.dimension
        cfg.device = self.device
        self._h = ctypes.c_void_p()
        if w0_device is not None:
            ptr, flags = w0_device.data_ptr(), 1 | (2 if w0_device.dtype == torch.float64 else 0)
        elif w0_host is not None:
            w0_host = np.ascontiguousarray(w0_host)
            ptr, flags = w0_host.ctypes.data, (2 if w0_host.dtype == np.float64 else 0)
        else:
            ptr, flags = None, 0
        rc = self.lib.ps_shard_create(ctypes.byref(cfg), self.world, self.rank, ptr, flags,
                                      ctypes.byref(self._h))
        if rc:
            raise_for(rc, self.lib.ps_shard_last_error(None).decode())
        blob = (ctypes.c_char * BLOB_BYTES)()
        n = self.lib.ps_shard_ipc_handles(self._h, blob, BLOB_BYTES)
        if n <= 0:
            self._check(n)
        joined = b"".join(exchange_blobs(bytes(blob)[:n]))
        self._check(self.lib.ps_shard_connect(self._h, joined, len(joined)))
        p = ctypes.c_void_p()
        padded = ctypes.c_int64(0)
        self.lib.ps_shard_update_buffer(self._h, ctypes.byref(p), ctypes.byref(padded))
        self.update = torch.as_tensor(_CudaArray(p.value, padded.value), device=f"cuda:{self.device}")
        # the worker's replica: w0 at start, rewritten by every owner at each pull
        self.lib.ps_shard_replica_buffer(self._h, ctypes.byref(p), ctypes.byref(padded))
        self.replica = torch.as_tensor(_CudaArray(p.value, padded.value), device=f"cuda:{self.device}")
        self.lo, self.hi = shard_range(self.dimension, self.world, self.rank)
        self.ticket = 1

    def _check(self, rc):
        raise_for(rc, self.lib.ps_shard_last_error(self._h).decode())

    def close(self):
        """Collective: unmap the peers' buffers, wait for every rank to have
        done the same, then free this rank's own (ps_shard_disconnect)."""
        if self._h and self._h.value:
            import torch.distributed as dist
            self.lib.ps_shard_disconnect(self._h)
            if dist.is_initialized():
                dist.barrier()
            self.lib.ps_shard_destroy(self._h)
            self._h = ctypes.c_void_p()

    def run(self, now_times, dst=None):
        """Enqueue len(now_times) push groups (+ this rank's pulls); returns
        the device time in ms. dst: CUDA fp32 tensor with >= round_up(d,4)
        elements, or None for the internal replica."""
        import torch
        # the update buffer is written on the caller's stream (copy_, normal_,
        # a backward); the run's own stream must not start before that work
        torch.cuda.current_stream(self.device).synchronize()
        now = np.ascontiguousarray(now_times, dtype=np.float64)
        ms = ctypes.c_double(0)
        rc = self.lib.ps_shard_run(self._h, self.ticket, len(now), now.ctypes.data,
                                   dst.data_ptr() if dst is not None else None, ctypes.byref(ms))
        self._check(rc)
        self.ticket += len(now)
        return ms.value

    def run_groups(self, groups, dst=None):
        """Heterogeneous schedules: ``groups`` is a list of (time, ticket order,
        pulling workers) -- the workers that push at that instant in the order
        the reference serves them, and the workers whose pull arrives before
        the next group (see groups_from_trace). Returns the device time in ms."""
        import torch
        torch.cuda.current_stream(self.device).synchronize()
        n = len(groups)
        now = np.ascontiguousarray([float(g[0]) for g in groups], dtype=np.float64)
        rows = np.zeros((max(n, 1), GROUP_STRIDE), dtype=np.int32)
        for i, (_, order, pulls) in enumerate(groups):
            rows[i, 0] = len(order)
            rows[i, 1] = int(sum(1 << int(q) for q in set(pulls)))
            rows[i, 2:2 + len(order)] = order
        ms = ctypes.c_double(0)
        rc = self.lib.ps_shard_run_groups(self._h, self.ticket, n, now.ctypes.data, rows.ctypes.data,
                                          dst.data_ptr() if dst is not None else None, ctypes.byref(ms))
        self._check(rc)
        self.ticket += n
        return ms.value

    def read_shard(self):
        out = np.empty(max(self.hi - self.lo, 1), dtype=np.float32)
        n = ctypes.c_int64(0)
        self._check(self.lib.ps_shard_read_shard(self._h, out.ctypes.data, ctypes.byref(n)))
        return out[:n.value]

    def read_replica(self):
        out = np.empty(self.dimension, dtype=np.float32)
        self._check(self.lib.ps_shard_read_replica(self._h, out.ctypes.data))
        return out

    def state(self):
        st = _lib.PSGateState()
        self._check(self.lib.ps_shard_get_state(self._h, ctypes.byref(st)))
        return st

    def trace(self):
        n = ctypes.c_int64(0)
        self._check(self.lib.ps_shard_trace(self._h, None, 0, ctypes.byref(n)))
        rows = (_lib.PSTraceRow * max(n.value, 1))()
        got = ctypes.c_int64(0)
        self._check(self.lib.ps_shard_trace(self._h, rows, n.value, ctypes.byref(got)))
        return rows_to_entries(rows, n.value)


# ---------------------------------------------------------------------------
# benchmark at N > 1 (bench.py delegates here under torchrun)
# ---------------------------------------------------------------------------

C3_DIM = 23_528_522
PARADIGMS = (("dssp", 3, 12), ("ssp", 3, 0), ("bsp", 0, 0), ("asp", 0, 0))


def c3_config(paradigm, s_lower, r_max, world):
    return validate_config(make_config(
        paradigm=paradigm, worker_count=world, s_lower=s_lower, r_max=r_max,
        timing_preset="homogeneous", compute_base=1.0, comm_delay=0.05,
        learning_rate=0.05, seed=0, dimension=C3_DIM, batch_size=1, dataset_size=world))


SWEEP_MB = (1, 4, 16, 64, 256, 1024)


def bandwidth_sweep(world, rank, local, warm, steps):
    """BASELINE configs[4] at N GPUs: the sharded push+pull step on 1 MB - 1 GB
    parameter vectors (ASP, every worker pushes every step), NVLink GB/s
    received per GPU against the 770 GB/s peer-copy peak. Returns rank 0's
    rows (max-over-ranks device times)."""
    import torch
    import torch.distributed as dist

    rows = []
    for mb in SWEEP_MB:
        d = mb * (1 << 18)
        cfg = validate_config(make_config(
            paradigm="asp", worker_count=world, timing_preset="homogeneous", compute_base=1.0,
            comm_delay=0.05, learning_rate=0.05, seed=0, dimension=d, batch_size=1,
            dataset_size=world))
        w0 = torch.zeros(d, dtype=torch.float32, device=f"cuda:{local}")
        srv = ShardedServer(cfg, d, rank, world, local, w0_device=w0)
        gen = torch.Generator(device=f"cuda:{local}")
        gen.manual_seed(7 + rank)
        srv.update[:d].normal_(generator=gen)
        times = homogeneous_push_times(1.0, 0.05, warm + steps)
        srv.run(times[:warm])
        dist.barrier()
        torch.cuda.synchronize()
        ms = max_over_ranks(srv.run(times[warm:warm + steps])) / steps
        lo, hi = shard_range(d, world, rank)
        nv_bytes = 2 * (world - 1) * (hi - lo) * 4
        gbs = nv_bytes / (ms * 1e-3) / 1e9
        rows.append({"mbytes": mb, "d": d, "step_ms": round(ms, 4),
                     "updates_per_s": round(world / (ms * 1e-3), 1),
                     "nvlink_gbs": round(gbs, 1), "nvlink_frac": round(gbs / 770.0, 3)})
        torch.cuda.synchronize()
        dist.barrier()
        srv.close()
        del w0
        torch.cuda.empty_cache()
    return rows


C4_DIM = 1_730_714  # ResNet-110 (CIFAR)


def throttled_bench(world, rank, local):
    """configs[3] across GPUs: one worker per GPU, throttled 1x / 2x / 4x
    (cycling), ResNet-110-sized server. The push groups come from the
    simulator's schedule for that cluster (the device run loop on a small
    vector -- every rank derives the same groups); the sharded server then
    serves them with its replicated gate: DSSP vs SSP vs BSP vs ASP, updates/s
    and the fast worker's waiting (virtual time)."""
    import torch
    import torch.distributed as dist
    from .metrics import per_worker, staleness_histogram
    from .sim import DeviceSimulation

    throttle = tuple((1, 2, 4)[q % 3] for q in range(world))
    out = {}
    for name, s, r in PARADIGMS:
        cfg = validate_config(make_config(
            paradigm=name, worker_count=world, s_lower=s, r_max=r, timing_preset="homogeneous",
            compute_base=1.0, comm_delay=0.05, throttle=throttle, model_kind="quadratic_bowl",
            dimension=C4_DIM, dataset_size=world * 400, batch_size=16, learning_rate=0.05,
            epochs=1, seed=0))
        sched = DeviceSimulation(cfg, dimension=64, device=local).run(loss_every=0, read_weights=False)
        groups = groups_from_trace(sched.entries)
        srv = ShardedServer(cfg, C4_DIM, rank, world, local)
        srv.update[:C4_DIM].normal_()
        srv.run_groups(groups[:8])  # warm-up
        dist.barrier()
        torch.cuda.synchronize()
        ms = max_over_ranks(srv.run_groups(groups[8:]))
        pushes = sum(len(g[1]) for g in groups[8:])
        trace = srv.trace()
        ok = [e.decision for e in trace] == [e.decision for e in sched.entries if e.kind == "push_arrive"]
        # and against the reference simulator's trace of the same cluster
        # (tests/golden/c4_sharded_schedule.json.gz), every rendered row
        want = _golden_push_rows("c4_sharded_schedule.json.gz", f"c4sh_{name}_p{world}")
        got_rows = [e.render().split("\t") for e in trace]
        ref_ok = (got_rows == want) if want else None
        pw = per_worker(sched.entries)
        hist = staleness_histogram(sched.entries)
        out[name] = {"updates_per_s": pushes / (ms * 1e-3), "groups": len(groups) - 8,
                     "updates": pushes, "decisions_match_single_gpu_engine": ok,
                     "trace_identical_to_reference": ref_ok,
                     "fast_worker_wait_s": pw[0].wait_s, "max_staleness": max(hist) if hist else 0,
                     "throttle": list(throttle)}
        torch.cuda.synchronize()
        dist.barrier()
        srv.close()
    return out


def torch_workers_bench(world, rank, local, warm, steps, batch=128):
    """configs[2] with real workers: a torchvision ResNet-50 (10 classes,
    23,528,522 parameters) per GPU on synthetic 32x32x3 batches, parameters
    living in the server's replica and gradients in its update buffer; one
    step = every worker's forward/backward + one sharded push/apply/pull.
    Returns rank 0's iterations/s per paradigm (max-over-ranks time)."""
    import torch
    import torch.distributed as dist
    import torch.nn.functional as F
    from .workers import flatten_, resnet50_cifar, synthetic_cifar

    out = {}
    for name, s, r in PARADIGMS:
        torch.manual_seed(0)
        model = resnet50_cifar().cuda()
        w0 = torch.cat([p.detach().reshape(-1) for p in model.parameters()])
        d = w0.numel()
        cfg = validate_config(make_config(
            paradigm=name, worker_count=world, s_lower=s, r_max=r, timing_preset="homogeneous",
            compute_base=1.0, comm_delay=0.05, learning_rate=0.01, seed=0, dimension=d,
            batch_size=batch, dataset_size=world * batch))
        srv = ShardedServer(cfg, d, rank, world, local, w0_device=w0)
        flatten_(model, into=(srv.replica, srv.update), copy_params=False)
        del w0
        batches = synthetic_cifar(2, batch, seed=100 + rank)
        times = homogeneous_push_times(1.0, 0.05, warm + steps)
        ps_ms = 0.0

        def step(i):
            x, y = batches[i % 2]
            srv.update.zero_()
            F.cross_entropy(model(x), y).backward()
            return srv.run(times[i:i + 1])

        for i in range(warm):
            step(i)
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i in range(warm, warm + steps):
            ps_ms += step(i)
        torch.cuda.synchronize()
        wall = max_over_ranks(time.perf_counter() - t0)
        out[name] = {"iters_per_s": steps * world / wall, "server_device_share_of_wall": ps_ms * 1e-3 / wall,
                     "model": "ResNet-50 (torchvision, 10 classes, 23,528,522 params)",
                     "batch_per_worker": batch, "workers": world}
        torch.cuda.synchronize()
        dist.barrier()
        srv.close()
        del model
        torch.cuda.empty_cache()
    return out


class NvlinkCounters:
    """NVLink data counters of one GPU (NVML field values, KiB per link,
    summed over links), read before and after a timed region: the bytes the
    GPU actually sent and received over NVLink there. Diagnostics only; any
    NVML failure leaves the figures None."""

    FIELDS = {"data_tx_kib": 138, "data_rx_kib": 139}  # NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX/RX

    def __init__(self, index):
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(int(index))
            self.links = 18
            self.ok = self.read() is not None
        except Exception:
            self.ok = False

    def read(self):
        try:
            req = [(fid, link) for fid in self.FIELDS.values() for link in range(self.links)]
            vals = self.nv.nvmlDeviceGetFieldValues(self.h, req)
            out = dict.fromkeys(self.FIELDS, 0)
            seen = False
            for (fid, _link), v in zip(req, vals):
                if v.nvmlReturn != 0:
                    continue
                seen = True
                name = next(k for k, f in self.FIELDS.items() if f == fid)
                out[name] += int(v.value.ullVal)
            return out if seen else None
        except Exception:
            return None


def _fp32_checksums(arr):
    """Order-independent bit-exact fingerprint of an fp32 vector: (xor, sum)
    of its bit patterns -- the shard/replica parity figure of the bench."""
    u = np.ascontiguousarray(arr, dtype=np.float32).view(np.uint32)
    return [int(np.bitwise_xor.reduce(u)) if u.size else 0, int(u.astype(np.uint64).sum())]


def host_update(d, rank, seed=0):
    """The bench's synthetic update of worker `rank`: N(0,1) fp32 from
    PCG64(seed * 1000 + rank), drawn on the host."""
    rng = np.random.Generator(np.random.PCG64(seed * 1000 + rank))
    return rng.standard_normal(d, dtype=np.float32)


def bench_main(args, metric, extras=None):
    """The headline at every N (BASELINE configs[2], "C3"): d = 23,528,522
    fp32 sharded over the N GPUs, one homogeneous worker per GPU, all four
    paradigms (N = 1 is the same server at G = 1). One step = one push group:
    every worker pushes, each owner applies the N updates in ticket order,
    the replicated gate decides, every worker pulls. Weak scaling: every GPU
    owns d/N parameters and applies N updates to them per step (d element
    updates per GPU per step at every N). `extras(torch, ps, line)` adds the
    single-GPU blocks at N = 1 (rank 0)."""
    import torch
    import torch.distributed as dist

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", str(29650 + os.getpid() % 500))
    os.environ.setdefault("RANK", str(rank))
    os.environ.setdefault("WORLD_SIZE", str(world))
    torch.cuda.set_device(local)
    if not dist.is_initialized():
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    d = C3_DIM
    # initial weights: rank 0 draws them (server.py:24-26) and NCCL-broadcasts
    w0 = torch.empty(d, dtype=torch.float32, device="cuda")
    if rank == 0:
        w0.copy_(torch.from_numpy(initial_weights_f64(c3_config("dssp", 3, 12, world), d)
                                  .astype(np.float32)))
    dist.broadcast(w0, 0)
    steps, warm = args.steps, args.warmup
    e2e_steps = max(3, min(steps, 10))
    times = homogeneous_push_times(1.0, 0.05, warm + steps + e2e_steps + 1)
    S_lo, S_hi = shard_range(d, world, rank)
    upd_host = torch.from_numpy(host_update(d, rank)).pin_memory()
    results, parity = {}, {}
    sampler = None
    if rank == 0:
        from bench import ClockSampler
        sampler = ClockSampler(local)
        sampler.__enter__()
    nvl = NvlinkCounters(local) if world > 1 else None
    nvl_delta = None
    for name, s, r in PARADIGMS:
        cfg = c3_config(name, s, r, world)
        srv = ShardedServer(cfg, d, rank, world, local, w0_device=w0)
        srv.update[:d].copy_(upd_host)
        srv.run(times[:warm])
        dist.barrier()
        torch.cuda.synchronize()
        c0 = nvl.read() if (nvl is not None and nvl.ok and name == "dssp") else None
        ms = srv.run(times[warm:warm + steps])
        if c0 is not None:
            c1 = nvl.read()
            if c1 is not None:
                nvl_delta = {k: (c1[k] - c0[k]) * 1024 / steps for k in c0}
        ms_max = max_over_ranks(ms)
        entries = srv.trace()
        decisions = [e.decision for e in entries]
        results[name] = {"updates_per_s": steps * world / (ms_max * 1e-3),
                         "iters_per_s": steps * world / (ms_max * 1e-3),
                         "ms_per_step": ms_max / steps,
                         "defers": sum(1 for x in decisions if x == "defer")}
        # parity: decisions of every step against the reference simulator's
        # trace of this schedule (tests/golden/c3_schedule.json.gz) ...
        want = _c3_reference_decisions(name, world)
        got = [e.render().split("\t") for e in entries][:len(want)]
        parity.setdefault("decisions_identical_to_reference", {})[name] = (
            len(got) == min(len(want), (warm + steps) * world) and got == want[:len(got)])
        if name == "dssp":
            # ... and the weights: every rank's shard and replica fingerprint
            # against the fp32 replay of the same (warm + steps) x N applies
            sums = {"shard": _fp32_checksums(srv.read_shard()),
                    "replica": _fp32_checksums(srv.read_replica()), "lo": S_lo, "hi": S_hi}
            everyone = [None] * world
            dist.all_gather_object(everyone, sums)
            parity["_weights_applies"] = (warm + steps) * world
            parity["_rank_sums"] = everyone
            # e2e: the same step through the public API with the worker's
            # update arriving from pinned host memory (H2D, 94 MB) and the
            # step's result -- the gate's decisions and version -- leaving
            # to the host (D2H); the pulled weights stay in this GPU's replica
            dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            base = warm + steps
            for i in range(e2e_steps):
                srv.update[:d].copy_(upd_host, non_blocking=True)
                srv.run(times[base + i:base + i + 1])
                srv.state()
            torch.cuda.synchronize()
            e2e_s = time.perf_counter() - t0
            results["_e2e"] = {"value": e2e_steps * world / max_over_ranks(e2e_s), "unit": "updates/s",
                               "h2d_bytes_per_step": 4 * d,
                               "d2h_bytes_per_step": ctypes.sizeof(_lib.PSGateState),
                               "api": "ShardedServer.run (C-ABI ps_shard_run) with the update from "
                                      "pinned host memory; gate state read back per step",
                               "steps": e2e_steps}
        torch.cuda.synchronize()
        dist.barrier()  # no peer may still be reading this rank's memory
        srv.close()
    del w0
    torch.cuda.empty_cache()
    full = not getattr(args, "no_sweep", False)
    sweep = bandwidth_sweep(world, rank, local, warm, steps) if (full and world > 1) else None
    tw = torch_workers_bench(world, rank, local, max(warm, 5), min(steps, 10)) if full else None
    c4 = throttled_bench(world, rank, local) if (full and world > 1) else None
    line = None
    if rank == 0:
        head = results["dssp"]
        S = S_hi - S_lo
        line = {
            "metric": metric, "value": head["updates_per_s"], "unit": "updates/s",
            "n_gpus": world, "steps": steps, "warmup": warm, "ms_per_step": head["ms_per_step"],
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": "C3 (BASELINE configs[2]): ResNet-50-sized server d=23528522 fp32 "
                                   f"sharded {world} way(s), {world} homogeneous worker(s), one per GPU, "
                                   "DSSP(3,12); step = one push group (every worker pushes, owners "
                                   "apply in ticket order, gate decides) + every worker's pull",
                       "d": d, "workers": world, "paradigm": "dssp", "s_lower": 3, "r_max": 12,
                       "parallelism": f"sharded server x{world}" + (", P2P NVLink" if world > 1 else ""),
                       "l2": "inputs larger than L2: per GPU the 94 MB update, the 94 MB replica "
                             "and the double-buffered shard are touched every step"},
            "per_paradigm": {k: v for k, v in results.items() if not k.startswith("_")},
            "parity": parity,
            "e2e": results["_e2e"],
            "gpu_launches": 1,  # one persistent k_shard_run covers all K timed steps
        }
        if world == 1:
            alg = 16 * d  # read w, read update, write w, write the replica (the pull)
            achieved = alg / (head["ms_per_step"] * 1e-3) / 1e9
            from bench import peaks, shard_traffic
            hbm_peak, peak_kind = peaks()
            line["roofline"] = {
                "bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                "frac": achieved / hbm_peak, "frac_vs_8000": achieved / 8000.0,
                "traffic": shard_traffic(), "peak_kind": peak_kind,
                "kernel": "k_shard_run (persistent; whole step: apply, pull, verdict, gate)",
                "bytes_model": "16 B/param per step: read shard 4 + read update 4 + write shard 4 "
                               "+ write replica 4 (the pull, fused into the apply pass)"}
        else:
            nv_bytes = 2 * (world - 1) * S * 4          # push slices in + pull shards in, per GPU
            achieved = nv_bytes / (head["ms_per_step"] * 1e-3) / 1e9
            line["roofline"] = {
                "bound": "nvlink", "achieved": achieved, "peak": 770.0, "unit": "GB/s",
                "frac": achieved / 770.0, "frac_vs_900": achieved / 900.0,
                "traffic": _probe_traffic(world, "received_user_bytes_per_gpu_per_step")
                           or (nvl_delta or {}).get("data_rx_kib"),
                "traffic_link_bytes_with_protocol": _probe_traffic(world, "received_link_bytes_per_gpu_per_step"),
                "traffic_source": "ncu nvlrx/nvltx byte counters of the same streaming pass, one-sided "
                                  "(profiles/k_shard_run_nvlink_bytes.json, tools/shard_nvlink_probe.py): "
                                  "received NVLink user bytes per GPU per step",
                "traffic_counters": nvl_delta,
                "traffic_note": "NVML NVLink data counters of rank 0's GPU around the timed DSSP run, "
                                "bytes per step, when the box supports them (these report "
                                "NOT_SUPPORTED: profiles/r2_nvml_probe.txt); ncu cannot attach to a "
                                "multi-rank run, so the link-byte evidence is the single-process ncu "
                                "capture of the P2P push/pull kernels, profiles/r2_ncu_nvlink_probe.csv",
                "peak_kind": "measured peer copy per direction (B200_PROFILING.md); frac_vs_900 "
                             "against the NVLink 5 spec",
                "kernel": "k_shard_run (persistent; whole step: push, apply, pull, verdict, gate)",
                "bytes_model": "2*(G-1)*S*4 B received over NVLink per GPU per step"}
        line["sweep"] = sweep
        line["torch_workers"] = tw
        if c4 is not None:
            line["c4_throttled_sharded"] = c4
    dist.barrier()
    if rank == 0:
        # the reference's CPU implementation on a bounded sample of this same
        # workload, pinned to one host core, plus the fp32 replay fingerprints
        # of the weights (a separate process: the checker, not the product)
        from bench import cpu_baseline_c3
        try:
            base = cpu_baseline_c3(world, parity["_weights_applies"])
            line["cpu_baseline"] = base["cpu_baseline"]
            want = base["fingerprints"]
            ok_shard = all(rs["shard"] == [want["shards"][i][0], want["shards"][i][1]]
                           for i, rs in enumerate(parity["_rank_sums"]))
            ok_rep = all(rs["replica"] == want["replica"] for rs in parity["_rank_sums"])
            parity["weights_bit_exact_vs_fp32_replay"] = {"shards": ok_shard, "replicas": ok_rep,
                                                         "applies": parity["_weights_applies"]}
        except Exception as exc:  # noqa: BLE001 -- the checker failed, not the engine
            line["cpu_baseline"] = {"error": f"{type(exc).__name__}: {exc}"[:500]}
            parity["weights_bit_exact_vs_fp32_replay"] = "unchecked (the CPU checker failed)"
        parity.pop("_rank_sums")
        parity.pop("_weights_applies")
        from bench import _safe
        if extras is not None:
            import paper_1908_11848_b200 as ps
            _safe(line, "_extras", lambda: extras(torch, ps, line))
            if line.get("_extras") is None:
                line.pop("_extras", None)
        if world > 1 and full:
            # configs[3] across GPUs with real workers: 3 x ResNet-110 at
            # 1x/2x/4x, one per GPU, blocked and released by device flags
            # (the server on this rank's GPU, the others over NVLink)
            import paper_1908_11848_b200 as ps
            from bench import free_running
            _safe(line, "free_running_c4_multi_gpu", lambda: free_running(
                torch, ps, 110, 3, (1.0, 2.0, 4.0), 24, devices=[q % world for q in range(3)]))
        if sampler is not None:
            sampler.__exit__(None, None, None)
            line["clocks"] = sampler.summary()
        print(json.dumps(line))
    # the other ranks wait on the host store, not in an NCCL kernel that would
    # hold SMs of the GPUs rank 0's multi-GPU blocks run on
    from datetime import timedelta
    store = dist.distributed_c10d._get_default_store()
    if rank == 0:
        store.set("bench_done", "1")
    else:
        store.wait(["bench_done"], timedelta(seconds=3600))
    dist.destroy_process_group()
    return 0


def _probe_traffic(world, key):
    """NVLink bytes per GPU per step of the sharded streaming pass at this
    world size, from the committed ncu capture, or None."""
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                        "k_shard_run_nvlink_bytes.json")
    try:
        return json.load(open(path))["per_world"][str(world)][key]
    except Exception:
        return None


def _golden_push_rows(fixture, name):
    """Push rows of a reference simulator trace committed under tests/golden
    (recorded by make_golden.py), or [] if absent."""
    import gzip
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                        fixture)
    try:
        with gzip.open(path, "rt") as fh:
            runs = json.load(fh)["runs"]
    except OSError:
        return []
    for r in runs:
        if r["name"] == name:
            return [ln.split("\t") for ln in r["trace"].splitlines() if ln.split("\t")[2] == "push_arrive"]
    return []


def _c3_reference_decisions(paradigm, world):
    """Push rows of the reference simulator's trace of the C3 schedule
    (tests/golden/c3_schedule.json.gz), or [] for an unrecorded world size."""
    return _golden_push_rows("c3_schedule.json.gz", f"c3_{paradigm}_p{world}")
