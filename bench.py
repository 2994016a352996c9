#!/usr/bin/env python
"""Benchmark of the parameter-server hot path (push-apply, pull, DSSP gate).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl engine|reference]

N=1 (default) measures BASELINE.json configs[1] ("C2"): a ResNet-20-sized
server (d = 272,474 fp32) with P = 4 workers on the heterogeneous gtx-mix
schedule (simnet.py:34-69; 2 fast + 2 workers 2.2x slower). One "step" is the
server serving the request stream of one complete run (250 iterations per
worker: 1,000 push-applies, 1,004 pulls, 1,000 gate decisions) in the order
the reference simulator issues them (tests/golden/c2_schedule.json.gz,
recorded from stalesync itself), in one device-resident kernel; every
decision is checked against the recorded one. The closed-loop variant (the
simulator's whole event loop on the device, trace byte-identical) is reported
as device_simulation. Updates are synthetic N(0,1) fp32 vectors resident in
HBM (2 per worker), lr = 0.05. The headline paradigm is DSSP(3, 12); BSP,
SSP(3) and ASP are reported beside it.

N>1 (torchrun, one process per GPU) measures configs[2] ("C3"): a
ResNet-50-sized server (d = 23,528,522 fp32) sharded by contiguous range
across the N GPUs, one worker per GPU, homogeneous workers; each step every
worker pushes its update to every shard owner over NVLink P2P, the owners
apply all N updates in ticket order, the replicated device gate decides, and
every worker pulls the full weights back over NVLink.

The line also carries:
  e2e          the same metric through the reference-facing API
               (ParameterServer drop-in, host buffers, H2D/D2H per call);
  roofline     the dominant kernel's achieved bytes/s vs the measured peak;
  cpu_baseline the reference algorithm (oracle/ port, fp64 numpy, 1 core) on
               a bounded sample of the same call sequence;
  sweep        push-apply / pull kernels at 1 MB .. 1 GB (configs[4]).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM_GBS = 6650.0   # B200_PROFILING.md fallback
NVLINK_GBS = 770.0          # B200_PROFILING.md measured peer copy per direction
C2_DIM = 272_474            # ResNet-20 (CIFAR-10) parameter count
C3_DIM = 23_528_522         # ResNet-50 (torchvision layout, 10 classes)
METRIC = "PS push+pull updates/sec (HBM/NVLink GB/s); iters/sec per paradigm at 1/2/4/8 B200"
PARADIGMS = (("dssp", 3, 12), ("ssp", 3, 0), ("bsp", 0, 0), ("asp", 0, 0))


def peaks():
    try:
        with open(PEAKS_PATH) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled DURING the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS,
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                return
            self._stop.wait(0.1)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        mx = [float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit()]
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 5 + i and s[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def c2_config(paradigm, s_lower, r_max):
    import paper_1908_11848_b200 as ps
    return ps.validate_config(ps.make_config(
        paradigm=paradigm, worker_count=4, s_lower=s_lower, r_max=r_max,
        timing_preset="gtx-mix", compute_base=1.0, comm_delay=0.05, model_kind="tiny_mlp",
        dimension=3072, dataset_size=4000, batch_size=16, learning_rate=0.05, epochs=4, seed=0))


def synthetic_host(P, K, d):
    """N(0,1) fp32 updates from PCG64(seed*1000 + worker) per SURVEY.md 8(d)."""
    out = np.zeros((P, K, (d + 3) // 4 * 4), dtype=np.float32)
    for p in range(P):
        rng = np.random.Generator(np.random.PCG64(0 * 1000 + p))
        for k in range(K):
            out[p, k, :d] = rng.standard_normal(d, dtype=np.float32)
    return out


def flush_l2(torch, buf):
    buf.add_(1.0)  # 256 MiB write: larger than the 126 MB L2


# ---------------------------------------------------------------------------
# reference arm / cpu baseline: the oracle port of the reference algorithm
# ---------------------------------------------------------------------------

def reference_sample(calls, synth, d, paradigm, s_lower, r_max, lr, max_updates):
    """Time the reference algorithm (oracle.RefPortServer: fp64 numpy apply
    with the reference's temporaries and frozen copies, Python gate) on the
    first `max_updates` applies of the call sequence. Returns (updates, s)."""
    import oracle
    w0 = oracle.initial_weights_f64(0, d)
    srv = oracle.RefPortServer(paradigm, synth.shape[0], s_lower, r_max, lr, w0)
    g64 = [[np.array(synth[p, k, :d], dtype=np.float64) for k in range(synth.shape[1])]
           for p in range(synth.shape[0])]
    for row in g64:
        for g in row:
            g.flags.writeable = False
    pushes = {}
    updates = 0
    t0 = time.perf_counter()
    for call in calls:
        if call[0] == "apply":
            k = pushes.get(call[1], 0)
            pushes[call[1]] = k + 1
            srv.apply_gradient(g64[call[1]][k % len(g64[call[1]])])
            updates += 1
        elif call[0] == "decide":
            srv.decide_push(call[1], call[2])
        elif call[0] == "pull":
            srv.handle_pull(call[1])
        if updates >= max_updates and call[0] == "decide":
            break
    return updates, time.perf_counter() - t0


def reference_c3_step(srv, grads, times_i, world):
    """One C3 push group through the reference algorithm (simnet.py:167-201):
    every worker's apply in seq order, then each decision, then every pull."""
    for p in range(world):
        srv.apply_gradient(grads[p % len(grads)])
    for p in range(world):
        srv.decide_push(p, times_i)
    for p in range(world):
        srv.handle_pull(p)


def run_reference_arm_sharded(args, world):
    """N > 1: the reference CPU server on OUR arm's N>1 workload (C3: d =
    23,528,522, `world` homogeneous workers, DSSP(3,12)); one step = one push
    group, exactly what one step of the sharded engine does."""
    import oracle
    from paper_1908_11848_b200.sharded import C3_DIM, homogeneous_push_times
    d = C3_DIM
    rng = np.random.default_rng(1000)
    grads = []
    for _ in range(2):  # two distinct N(0,1) updates, alternated by worker (memory bound on the host)
        g = rng.standard_normal(d)
        g.flags.writeable = False
        grads.append(g)
    srv = oracle.RefPortServer("dssp", world, 3, 12, 0.05, oracle.initial_weights_f64(0, d))
    times = homogeneous_push_times(1.0, 0.05, args.warmup + args.steps)
    for i in range(args.warmup):
        reference_c3_step(srv, grads, times[i], world)
    t0 = time.perf_counter()
    for i in range(args.steps):
        reference_c3_step(srv, grads, times[args.warmup + i], world)
    total = time.perf_counter() - t0
    value = args.steps * world / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "updates/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"C3 (BASELINE configs[2]): d={d}, {world} homogeneous workers, "
                               "DSSP(3,12); step = one push group (every worker's apply, decide, pull)",
                   "d": d, "workers": world},
        "cpu_baseline": {"value": value, "unit": "updates/s", "cores": 1, "kind": "port",
                         "sample": f"{args.steps} push groups of {world} updates (oracle.RefPortServer, "
                                   "fp64 numpy, single-threaded like the reference)"},
        "e2e": {"value": value, "unit": "updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    if world > 1:
        return run_reference_arm_sharded(args, world)
    import paper_1908_11848_b200 as ps
    # the call sequence of the C2 schedule is fixed by the reference
    # simulator semantics; replay it with the same synthetic updates
    cfg = c2_config("dssp", 3, 12)
    calls, _ = reference_calls("dssp")
    synth = synthetic_host(4, 2, C2_DIM)
    n_updates = sum(1 for c in calls if c[0] == "apply")
    per_step = min(n_updates, 250)
    for _ in range(args.warmup):
        reference_sample(calls, synth, C2_DIM, "dssp", 3, 12, cfg.learning_rate, per_step)
    times, ups = [], 0
    for _ in range(args.steps):
        u, s = reference_sample(calls, synth, C2_DIM, "dssp", 3, 12, cfg.learning_rate, per_step)
        times.append(s)
        ups += u
    total = sum(times)
    value = ups / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "updates/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "C2 call sequence (DSSP(3,12), P=4, gtx-mix), d=272474; "
                               f"each step = the first {per_step} updates"},
        "cpu_baseline": {"value": value, "unit": "updates/s", "cores": 1, "kind": "port",
                         "sample": f"{per_step} updates x {args.steps} steps of the C2 call sequence"},
        "e2e": {"value": value, "unit": "updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def reference_calls(paradigm="dssp"):
    """The C2 server-call sequence and trace recorded from the reference
    simulator itself (tests/golden/c2_schedule.json.gz, made by
    tests/golden/make_golden.py)."""
    import oracle
    for run in oracle.load_golden("c2_schedule.json.gz")["runs"]:
        if run["name"] == f"c2_{paradigm}":
            calls = [tuple(c[:2]) if c[0] != "decide" else ("decide", c[1], c[2])
                     for c in run["calls"] if c[0] in ("pull", "apply", "decide")]
            return calls, run["trace"]
    raise KeyError(paradigm)


# ---------------------------------------------------------------------------
# engine arm, N = 1
# ---------------------------------------------------------------------------

def apply_sweep(torch, ps, hbm_peak):
    """configs[4]: push-apply (12 B/param) and pull (8 B/param) kernels from
    1 MB to 1 GB of fp32 parameters; L2 flushed before every timed launch.
    The library's profiling events bracket the op behind a 50 us device spin,
    so each time is the op's device time (its launches, the apply's
    flag reduction and host-mirror publish included), not the host's submit
    gap on an idle stream."""
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    out = []
    for mb in (1, 4, 16, 64, 256, 1024):
        d = mb * (1 << 20) // 4
        eng = ps.engine.Engine("asp", 1, 0, 0, 0.05, d, device=0)
        eng.set_profiling(True)
        g = torch.randn(d, device="cuda", dtype=torch.float32)
        dst = torch.empty(d, device="cuda", dtype=torch.float32)
        ap, pl = [], []
        for it in range(8):
            flush_l2(torch, flush)
            torch.cuda.synchronize()
            eng.apply(0, g)
            if it >= 3:
                ap.append(eng.last_kernel_ms())
            flush_l2(torch, flush)
            torch.cuda.synchronize()
            eng.read(out=dst)
            if it >= 3:
                pl.append(eng.last_kernel_ms())
        eng.close()
        a_ms, p_ms = statistics.median(ap), statistics.median(pl)
        out.append({"mbytes": mb, "d": d,
                    "apply_ms": round(a_ms, 4), "apply_gbs": round(12 * d / a_ms / 1e6, 1),
                    "apply_frac": round(12 * d / a_ms / 1e6 / hbm_peak, 3),
                    "pull_ms": round(p_ms, 4), "pull_gbs": round(8 * d / p_ms / 1e6, 1),
                    "pull_frac": round(8 * d / p_ms / 1e6 / hbm_peak, 3)})
        del g, dst
    del flush
    torch.cuda.empty_cache()
    return out


C4_DIM = 1_730_714  # ResNet-110 (CIFAR)


def c4_config(paradigm, s_lower, r_max):
    """BASELINE configs[3]: three workers throttled 1x / 2x / 4x."""
    import paper_1908_11848_b200 as ps
    return ps.validate_config(ps.make_config(
        paradigm=paradigm, worker_count=3, s_lower=s_lower, r_max=r_max,
        timing_preset="homogeneous", compute_base=1.0, comm_delay=0.05, throttle=(1, 2, 4),
        model_kind="tiny_mlp", dimension=3072, dataset_size=3 * 1600, batch_size=16,
        learning_rate=0.05, epochs=1, seed=0))


def c4_throttled(torch, ps, reps=3):
    """configs[3]: DSSP threshold adaptation vs fixed SSP on a 1x/2x/4x
    cluster, ResNet-110-sized server, device run loop; reports device
    throughput and the schedule's virtual-time outcome per paradigm."""
    from paper_1908_11848_b200.metrics import per_worker, staleness_histogram
    d = C4_DIM
    synth = torch.from_numpy(synthetic_host(3, 2, d)).cuda()
    out = {}
    for name, s, r in PARADIGMS:
        cfg = c4_config(name, s, r)
        sim = ps.DeviceSimulation(cfg, dimension=d, grad="synthetic")
        sim.set_synthetic(synth, 2)
        sim.run(read_weights=False, reset_gate=True)
        times = []
        for _ in range(reps):
            rep = sim.run(read_weights=False, reset_gate=True)
            times.append(rep.device_ms)
        pw = per_worker(rep.entries)
        hist = staleness_histogram(rep.entries)
        out[name] = {"updates_per_s": rep.applied / (statistics.median(times) * 1e-3),
                     "updates": rep.applied,
                     "virtual_duration_s": max(e.time for e in rep.entries),
                     "fast_worker_wait_s": pw[0].wait_s,
                     "total_wait_s": sum(w.wait_s for w in pw.values()),
                     "max_staleness": max(hist) if hist else 0}
        sim.engine.close()
    del synth
    return out


def c4_realtime(torch, ps, scale=1e-3):
    """configs[3] free-running: the same 1x/2x/4x cluster on the wall clock
    (1 virtual second = `scale` s of GPU global time), every push decided at
    the instant it reaches the device gate. Reports the wall-clock makespan,
    the fast worker's wait and the staleness the gate allowed."""
    from paper_1908_11848_b200.metrics import per_worker, staleness_histogram
    d = C4_DIM
    synth = torch.from_numpy(synthetic_host(3, 2, d)).cuda()
    out = {}
    for name, s, r in PARADIGMS:
        cfg = c4_config(name, s, r)
        sim = ps.DeviceSimulation(cfg, dimension=d, grad="synthetic")
        sim.set_synthetic(synth, 2)
        rep = sim.run(read_weights=False, reset_gate=True, realtime_scale=scale, deadline_s=30.0)
        pw = per_worker(rep.entries)
        hist = staleness_histogram(rep.entries)
        out[name] = {"completed": rep.completed, "updates": rep.applied,
                     "wall_ms": rep.device_ms,
                     "virtual_duration_s": max(e.time for e in rep.entries),
                     "fast_worker_wait_s": pw[0].wait_s,
                     "max_staleness": max(hist) if hist else 0,
                     "time_scale": scale}
        sim.engine.close()
    del synth
    return out


def torch_workers(torch, ps, iters=48, batch=128):
    """Real ResNet-20 workers (PyTorch fwd/bwd) on one GPU,
    round-robin, pushing .grad views and pulling into parameter views through
    the drop-in. Reports iterations/s per paradigm and the share of wall time
    spent in the server calls."""
    from paper_1908_11848_b200.workers import CifarResNet, TorchWorker, synthetic_cifar
    out = {}
    for name, s, r in PARADIGMS:
        cfg = ps.validate_config(ps.make_config(paradigm=name, worker_count=4, s_lower=s,
                                                r_max=r, learning_rate=0.01, seed=0))
        torch.manual_seed(0)
        workers = [TorchWorker(p, CifarResNet(20), synthetic_cifar(2, batch, seed=p))
                   for p in range(4)]
        server = ps.ParameterServer(cfg, workers[0].dimension)
        for wk in workers:
            wk.adopt_from(server)
        pending, done, ps_s = set(), 0, 0.0
        # warm-up (cuDNN autotuning), then the timed iterations
        for phase, n in (("warm", 8), ("timed", iters)):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            ps_s, done, it, now = 0.0, 0, 0, 0.0
            while done < n:
                p = it % 4
                it += 1
                if p in pending:
                    continue
                g = workers[p].begin_iteration()
                now += 1.0 + 0.5 * p
                t1 = time.perf_counter()
                dec = server.handle_push(g, now)
                if dec.granted:
                    for q in dec.released:
                        pending.discard(q)
                        workers[q].adopt_from(server)
                    workers[p].adopt_from(server)
                else:
                    pending.add(p)
                ps_s += time.perf_counter() - t1
                done += 1
            torch.cuda.synchronize()
            wall = time.perf_counter() - t0
        out[name] = {"iters_per_s": done / wall, "ps_share_of_wall": ps_s / wall,
                     "model": "CIFAR ResNet-20 (272,474 params)", "batch": batch, "workers": 4}
    return out


def e2e_drop_in(torch, ps, cfg, calls, synth_host, d):
    """The same workload through the reference-facing API: ParameterServer
    drop-in, gradients from pinned host memory (H2D per push), pulls into
    pinned host memory (D2H per pull). Returns (updates/s, h2d, d2h bytes)."""
    server = ps.ParameterServer(cfg, d)
    P, K = synth_host.shape[0], synth_host.shape[1]
    pinned = torch.from_numpy(np.ascontiguousarray(synth_host[:, :, :d])).pin_memory()
    host_g = [[pinned[p, k].numpy() for k in range(K)] for p in range(P)]
    pull_buf = torch.empty(d, dtype=torch.float32).pin_memory().numpy()
    grads = {}
    pushes = {}

    def replay():
        h2d = d2h = updates = 0
        for call in calls:
            if call[0] == "pull":
                server.handle_pull(call[1], out=pull_buf)
                d2h += 4 * d
            elif call[0] == "apply":
                p = call[1]
                k = pushes.get(p, 0)
                pushes[p] = k + 1
                server.apply_gradient(ps.GradientVector(host_g[p][k % K], p, k))
                h2d += 4 * d
                updates += 1
            else:
                server.decide_push(call[1], call[2])
        return updates, h2d, d2h

    # warm-up pass on a fresh gate, then the timed pass on another fresh one
    replay()
    server = ps.ParameterServer(cfg, d)
    pushes.clear()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    updates, h2d, d2h = replay()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    return updates / dt, h2d, d2h, updates


def e2e_batched(torch, ps, calls, synth_host, d, w0, steps=30):
    """The same request stream through the engine's batch C-ABI call
    (ps_replay_run via DeviceReplay) with HOST buffers: every step copies its
    inputs -- the call stream and the resident updates -- from host memory and
    reads its results -- every decision and the final weights -- back.
    Returns (updates/s, h2d bytes, d2h bytes per step)."""
    from paper_1908_11848_b200.engine import Engine
    from paper_1908_11848_b200.sim import DeviceReplay
    eng = Engine("dssp", synth_host.shape[0], 3, 12, 0.05, d, w0=w0)
    pinned = torch.from_numpy(np.ascontiguousarray(synth_host)).pin_memory()
    dev = torch.empty(pinned.shape, dtype=torch.float32, device="cuda")
    out_w = torch.empty(d, dtype=torch.float32).pin_memory().numpy()
    rp = DeviceReplay(eng, calls, dev, synth_host.shape[1])

    def step():
        dev.copy_(pinned, non_blocking=True)   # H2D: the step's updates
        r = rp.run(decisions=True)             # H2D of the calls inside; decisions D2H
        eng.read(out=out_w)                    # D2H: the weights after the step
        return r

    step()
    step()
    torch.cuda.synchronize()
    # wall clock per step (every step ends in a host read of its results);
    # the median step, so a host hiccup does not stand in for the engine
    per_step, applied = [], 0
    for _ in range(steps):
        t0 = time.perf_counter()
        r = step()
        torch.cuda.synchronize()
        per_step.append(time.perf_counter() - t0)
        applied = r.applied
    dt = statistics.median(per_step)
    n_dec = sum(1 for c in calls if c[0] == "decide")
    h2d = pinned.numel() * 4 + 16 * len(calls)
    d2h = 8 * n_dec + 4 * d
    eng.close()
    return applied / dt, h2d, d2h


def bench_single(args):
    import torch
    import paper_1908_11848_b200 as ps
    from paper_1908_11848_b200.engine import Engine
    from paper_1908_11848_b200.sim import DeviceReplay

    hbm_peak, peak_kind = peaks()
    d = C2_DIM
    P, K = 4, 2
    synth_host = synthetic_host(P, K, d)
    synth = torch.from_numpy(synth_host).cuda()
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    import oracle
    w0 = oracle.initial_weights_f64(0, d)
    # (1) headline: the device serving the recorded C2 request stream
    #     (pull / apply / decide, reference order), decisions by the device gate
    replays, sims, recorded = {}, {}, {}
    for name, s, r in PARADIGMS:
        calls, trace = reference_calls(name)
        recorded[name] = trace
        eng = Engine(name, P, s, r, 0.05, d, w0=w0)
        replays[name] = DeviceReplay(eng, calls, synth, K)
        cfg = c2_config(name, s, r)
        sim = ps.DeviceSimulation(cfg, dimension=d, grad="synthetic")
        sim.set_synthetic(synth, K)
        sims[name] = (cfg, sim)
        for _ in range(args.warmup):
            replays[name].run(decisions=False)
            sim.run(read_weights=False, reset_gate=True)
    sampler = ClockSampler(0)
    per_paradigm, device_sim, parity, reports = {}, {}, {}, {}
    with sampler:
        for name, s, r in PARADIGMS:
            times, applied = [], 0
            for _ in range(args.steps):
                flush_l2(torch, flush)
                torch.cuda.synchronize()
                rr = replays[name].run(decisions=False)
                times.append(rr.device_ms)
                applied += rr.applied
            total_ms = sum(times)
            check = replays[name].run()
            want = [(ln.split("\t")[4]) for ln in recorded[name].splitlines()
                    if ln.split("\t")[2] == "push_arrive"]
            got = [ps.decision_token(o == "grant", rel) for o, rel in check.decisions]
            per_paradigm[name] = {"updates_per_s": applied / (total_ms * 1e-3),
                                  "iters_per_s": applied / (total_ms * 1e-3),
                                  "ms_per_step": total_ms / args.steps,
                                  "defers_per_step": sum(1 for o, _ in check.decisions if o == "defer")}
            parity.setdefault("replay_decisions_identical_to_reference", {})[name] = got == want
        # (2) the closed loop: the simulator's whole event loop on the device
        for name, s, r in PARADIGMS:
            cfg, sim = sims[name]
            times, applied = [], 0
            rep = None
            for _ in range(args.steps):
                flush_l2(torch, flush)
                torch.cuda.synchronize()
                rep = sim.run(read_weights=False, reset_gate=True)
                times.append(rep.device_ms)
                applied += rep.applied
            reports[name] = rep
            total_ms = sum(times)
            device_sim[name] = {"updates_per_s": applied / (total_ms * 1e-3),
                                "ms_per_step": total_ms / args.steps,
                                "virtual_duration_s": max(e.time for e in rep.entries)}
            parity.setdefault("simulation_trace_identical_to_reference", {})[name] = \
                ps.format_trace(rep.entries) == recorded[name]
    head = per_paradigm["dssp"]
    calls, _ = reference_calls("dssp")
    n_apply = sum(1 for c in calls if c[0] == "apply")
    n_pull = sum(1 for c in calls if c[0] == "pull")
    # roofline of the dominant kernel (k_sim, replay mode): algorithmic bytes
    # per launch = updates x 12 B/param (push-apply) + pulls x 8 B/param
    alg_bytes = n_apply * 12 * d + n_pull * 8 * d
    achieved = alg_bytes / (head["ms_per_step"] * 1e-3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "k_sim_dram_bytes.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    cfg = c2_config("dssp", 3, 12)
    e2e_value, h2d, d2h, e2e_updates = e2e_drop_in(torch, ps, cfg, calls, synth_host, d)
    eb_value, eb_h2d, eb_d2h = e2e_batched(torch, ps, calls, synth_host, d, w0)
    cpu_updates, cpu_s = reference_sample(calls, synth_host, d, "dssp", 3, 12, cfg.learning_rate,
                                          max_updates=args.cpu_updates)
    sweep = apply_sweep(torch, ps, hbm_peak) if not args.no_sweep else None
    c4 = c4_throttled(torch, ps) if not args.no_sweep else None
    c4_rt = c4_realtime(torch, ps) if not args.no_sweep else None
    tw = torch_workers(torch, ps) if not args.no_sweep else None
    clocks = sampler.summary()
    line = {
        "metric": METRIC,
        "value": head["updates_per_s"],
        "unit": "updates/s",
        "n_gpus": 1,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": head["ms_per_step"],
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": "C2 (BASELINE configs[1]): ResNet-20-sized server d=272474 fp32, "
                               "P=4 workers, gtx-mix schedule, DSSP(3,12); step = the server "
                               "serving the reference's recorded request stream of one run "
                               f"({n_apply} pushes, {n_pull} pulls, {n_apply} gate decisions) "
                               "in one device-resident kernel",
                   "d": d, "workers": P, "paradigm": "dssp", "s_lower": 3, "r_max": 12,
                   "updates_per_step": n_apply, "l2": "flushed between timed steps (256 MiB write)",
                   "parallelism": "single GPU"},
        "per_paradigm": per_paradigm,
        "device_simulation": device_sim,
        "parity": parity,
        # e2e: the headline workload (the same call stream and resident
        # updates as `value`) through the batch C-ABI call with host buffers
        "e2e": {"value": eb_value, "unit": "updates/s", "h2d_bytes_per_step": eb_h2d,
                "d2h_bytes_per_step": eb_d2h,
                "api": "DeviceReplay.run (C-ABI ps_replay_run) with host buffers: the call "
                       "stream and the resident updates H2D, every decision and the final "
                       "weights D2H, per step"},
        # the reference-compatible per-call path: every push's update H2D and
        # every pull D2H, one host round trip per reference call
        "e2e_per_call": {"value": e2e_value, "unit": "updates/s", "h2d_bytes_per_step": h2d,
                         "d2h_bytes_per_step": d2h,
                         "api": "ParameterServer drop-in (apply_gradient / decide_push / "
                                "handle_pull), pinned host buffers",
                         "updates_per_step": e2e_updates},
        "gpu_launches": 2 * args.steps,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": achieved / hbm_peak, "traffic": traffic, "peak_kind": peak_kind,
                     "kernel": "k_sim (replay mode)",
                     "bytes_model": "12 B/param per push-apply + 8 B/param per pull",
                     "note": "C2's 1 MB of weights stay in registers and its updates in L2 for "
                             "the whole stream (traffic = DRAM bytes per launch from ncu), so "
                             "frac can exceed 1: the kernel is bound by the latency of the "
                             "serial gate and per-call issue, not by HBM"},
        "cpu_baseline": {"value": cpu_updates / cpu_s, "unit": "updates/s", "cores": 1,
                         "kind": "port",
                         "sample": f"first {cpu_updates} updates of the same C2 request stream, "
                                   "oracle.RefPortServer (fp64 numpy + Python gate)",
                         "host_cpus": os.cpu_count()},
        "sweep": sweep,
        "c4_throttled": c4,
        "c4_free_running": c4_rt,
        "torch_workers": tw,
        "clocks": clocks,
    }
    print(json.dumps(line))
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="engine", choices=("engine", "reference"))
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--cpu-updates", type=int, default=3000)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference_arm(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1 or args.gpus > 1:
        from paper_1908_11848_b200 import sharded
        return sharded.bench_main(args, METRIC)
    return bench_single(args)


if __name__ == "__main__":
    sys.exit(main())
