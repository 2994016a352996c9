#!/usr/bin/env python
"""Benchmark of the parameter-server hot path (push-apply, pull, DSSP gate).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl engine|reference]

The headline at EVERY N is BASELINE.json configs[2] ("C3"): a ResNet-50-sized
server (d = 23,528,522 fp32) sharded by contiguous range across the N GPUs
(N = 1: the same server at G = 1), one homogeneous worker per GPU. One step is
one push group: every worker pushes its update, each shard owner applies the N
updates in ticket order (over NVLink P2P for N > 1), the replicated device
gate decides (DSSP(3,12) headline; SSP(3), BSP, ASP beside it) and every worker
pulls the new weights. Weak scaling: every GPU owns d/N parameters and applies
N updates to them per step. Inputs exceed L2 (94 MB update + 94 MB replica +
the double-buffered shard per GPU), so the HBM (N = 1) / NVLink (N > 1)
roofline is the bound that matters.

The line also carries:
  parity       decisions of every paradigm against the reference simulator's
               trace of the same schedule, and every shard / replica
               fingerprint against the fp32 replay of the same applies;
  e2e          the same step through the C-ABI with the update H2D from pinned
               host memory and the gate state D2H every step;
  roofline     k_shard_run against HBM (N = 1) or NVLink (N > 1);
  cpu_baseline the reference (stalesync, unmodified, staged into oracle/_ref;
               the oracle port if absent) on a bounded sample of the same
               workload, pinned to one host core;
  N = 1 only:  `c2` -- BASELINE configs[1] (ResNet-20-sized single-GPU server,
               P = 4, gtx-mix) served as the reference's recorded request
               stream in one kernel, reported as latency (us per call /
               decision; it is L2- and latency-bound), its e2e variants, the
               simulated run loop; `sweep` (configs[4], 1 MB - 1 GB);
               `c4_*` (configs[3]); torch workers.
  N > 1:       the sharded sweep (configs[4] at N GPUs), configs[3] across
               GPUs, ResNet-50 workers on the sharded server.
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
# free-running worker streams block on device flags: give every stream its own
# hardware queue (must precede CUDA initialization)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

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
# reference arm / cpu baseline: the reference's own CPU implementation
# ---------------------------------------------------------------------------

def load_fixture(name):
    """A committed fixture under tests/golden (recorded from the reference)."""
    import gzip
    path = os.path.join(ROOT, "tests", "golden", name)
    opener = gzip.open if name.endswith(".gz") else open
    with opener(path, "rt") as fh:
        return json.load(fh)


def reference_calls(paradigm="dssp"):
    """The C2 server-call sequence and trace recorded from the reference
    simulator itself (tests/golden/c2_schedule.json.gz, made by
    tests/golden/make_golden.py)."""
    for run in load_fixture("c2_schedule.json.gz")["runs"]:
        if run["name"] == f"c2_{paradigm}":
            calls = [tuple(c[:2]) if c[0] != "decide" else ("decide", c[1], c[2])
                     for c in run["calls"] if c[0] in ("pull", "apply", "decide")]
            return calls, run["trace"]
    raise KeyError(paradigm)


def pin_one_core():
    """Pin this process to one host core (the reference is single-threaded
    numpy): the highest-numbered core it may use, away from the ranks'
    launch threads. Returns (core, host cpu count)."""
    cores = sorted(os.sched_getaffinity(0))
    core = cores[-1]
    os.sched_setaffinity(0, {core})
    return core, os.cpu_count()


def reference_server_factory():
    """(kind, make(paradigm, P, s_lower, r_max, lr, d) -> server, GradientVector):
    the unmodified reference (stalesync, staged into oracle/_ref by
    oracle/stage_ref.sh) when present, else the oracle's port of it."""
    ref = os.path.join(ROOT, "oracle", "_ref")
    if os.path.isdir(os.path.join(ref, "stalesync")):
        if ref not in sys.path:
            sys.path.insert(0, ref)
        import stalesync
        from stalesync.config import make_config, validate_config

        def make(paradigm, P, s_lower, r_max, lr, d):
            cfg = validate_config(make_config(paradigm=paradigm, worker_count=P, s_lower=s_lower,
                                              r_max=r_max, learning_rate=lr, seed=0, dimension=d,
                                              timing_preset="homogeneous", compute_base=1.0,
                                              comm_delay=0.05, dataset_size=P, batch_size=1))
            return stalesync.ParameterServer(cfg, d)
        return "reference", make, stalesync.GradientVector
    import oracle

    def make(paradigm, P, s_lower, r_max, lr, d):
        return oracle.RefPortServer(paradigm, P, s_lower, r_max, lr, oracle.initial_weights_f64(0, d))

    class _G:
        def __new__(cls, values, source, source_iter=0):
            values = np.asarray(values, dtype=np.float64)
            values.flags.writeable = False
            return values
    return "port", make, _G


def reference_c3_groups(world, steps, warmup, time_budget_s=None):
    """The reference CPU server on the C3 workload with `world` homogeneous
    workers: one step = one push group (simnet.py:167-201): every worker's
    apply_gradient in seq order, then each decide_push, then every
    handle_pull. Returns (kind, seconds per step list)."""
    d = C3_DIM
    kind, make, GV = reference_server_factory()
    srv = make("dssp", world, 3, 12, 0.05, d)
    rng = np.random.default_rng(1000)
    # two distinct N(0,1) updates, alternated by worker; built once, outside
    # the timing (a GradientVector copies its values, config.py:48-51)
    grads = [GV(rng.standard_normal(d), p, 1) for p in range(min(world, 2))]
    from paper_1908_11848_b200.sharded import homogeneous_push_times
    times = homogeneous_push_times(1.0, 0.05, warmup + steps)

    def group(now):
        for p in range(world):
            srv.apply_gradient(grads[p % len(grads)])  # apply_gradient reads only .values
        for p in range(world):
            srv.decide_push(p, now)
        for p in range(world):
            srv.handle_pull(p)

    for i in range(warmup):
        group(times[i])
    out = []
    t_all = time.perf_counter()
    for i in range(steps):
        t0 = time.perf_counter()
        group(times[warmup + i])
        out.append(time.perf_counter() - t0)
        if time_budget_s and time.perf_counter() - t_all > time_budget_s and len(out) >= 2:
            break
    return kind, out


def run_reference_arm(args):
    """--impl reference: the reference's own CPU implementation on OUR arm's
    workload (C3 at N workers, DSSP(3,12)), rank 0 only, pinned to one core."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    core, ncpu = pin_one_core()
    kind, secs = reference_c3_groups(world, args.steps, args.warmup)
    total = sum(secs)
    value = len(secs) * world / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "updates/s",
        "n_gpus": args.gpus, "steps": len(secs), "warmup": args.warmup,
        "ms_per_step": 1e3 * total / len(secs), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"C3 (BASELINE configs[2]): d={C3_DIM}, {world} homogeneous worker(s), "
                               "DSSP(3,12); step = one push group (every worker's apply, decide, pull)",
                   "d": C3_DIM, "workers": world},
        "cpu_baseline": {"value": value, "unit": "updates/s", "cores": 1, "kind": kind,
                         "sample": f"{len(secs)} push groups of {world} updates, "
                                   + ("stalesync 0.1.0 unmodified (oracle/_ref)" if kind == "reference"
                                      else "oracle.RefPortServer (port)")
                                   + f", pinned to host core {core} of {ncpu}"},
        "e2e": {"value": value, "unit": "updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def cpu_sample_main(args):
    """Child process of the engine arm (the cpu_baseline leg and the weight
    checker; the only engine-arm code that touches oracle/): pinned to one
    core, times the reference on a bounded sample and prints one JSON line."""
    core, ncpu = pin_one_core()
    if args.cpu_sample == "c2":
        calls, _ = reference_calls("dssp")
        synth = synthetic_host(4, 2, C2_DIM)
        kind, make, GV = reference_server_factory()
        srv = make("dssp", 4, 3, 12, 0.05, C2_DIM)
        gv = [[GV(np.array(synth[p, k, :C2_DIM], dtype=np.float64), p, k) for k in range(2)]
              for p in range(4)]
        pushes, updates = {}, 0
        t0 = time.perf_counter()
        for call in calls:
            if call[0] == "apply":
                k = pushes.get(call[1], 0)
                pushes[call[1]] = k + 1
                srv.apply_gradient(gv[call[1]][k % 2])
                updates += 1
            elif call[0] == "decide":
                srv.decide_push(call[1], call[2])
            else:
                srv.handle_pull(call[1])
        dt = time.perf_counter() - t0
        print(json.dumps({"value": updates / dt, "unit": "updates/s", "cores": 1, "kind": kind,
                          "sample": f"the whole C2 request stream ({updates} updates, same as one "
                                    f"engine step), pinned to host core {core} of {ncpu}",
                          "host_cpus": ncpu, "us_per_update": 1e6 * dt / updates}))
        return 0
    # c3: reference timing + fp32 replay fingerprints of the engine's weights
    world, applies = args.world, args.applies
    kind, secs = reference_c3_groups(world, 50, 1, time_budget_s=12.0)
    value = len(secs) * world / sum(secs)
    import oracle
    from paper_1908_11848_b200.sharded import _fp32_checksums, host_update, shard_range
    d = C3_DIM
    w = oracle.initial_weights_f64(0, d).astype(np.float32)
    gs = [host_update(d, p) for p in range(world)]
    for i in range(applies):
        w = oracle.apply_f32(w, gs[i % world], 0.05)
    shards = []
    for r in range(world):
        lo, hi = shard_range(d, world, r)
        shards.append(_fp32_checksums(w[lo:hi]))
    extra = cpu_side_lines(world)
    print(json.dumps({"cpu_baseline": {
        **extra,
        "value": value, "unit": "updates/s", "cores": 1, "kind": kind,
        "sample": f"{len(secs)} push groups of {world} updates of the same C3 workload, "
                  + ("stalesync 0.1.0 unmodified (oracle/_ref)" if kind == "reference"
                     else "oracle.RefPortServer (port)") + f", pinned to host core {core} of {ncpu}",
        "host_cpus": ncpu},
        "fingerprints": {"shards": shards, "replica": _fp32_checksums(w)}}))
    return 0


def gate_check_main(path):
    """Child: feed every recorded free-running decision sequence to the CPU
    oracle gate (test infrastructure) and report which match."""
    import oracle
    runs = json.load(open(path))
    out = {}
    for key, run in runs.items():
        g = oracle.CGate(run["paradigm"], run["P"], run["s"], run["r"])
        ok = True
        for w, now, outcome, released in run["seq"]:
            if g.on_push(w, now) != (outcome, tuple(released)):
                ok = False
                break
        out[key] = ok
    print(json.dumps(out))
    return 0


def gate_check(runs):
    """{key: {paradigm, P, s, r, seq}} -> {key: decisions identical to the oracle gate}."""
    import tempfile
    with tempfile.NamedTemporaryFile("w", suffix=".json", delete=False) as fh:
        json.dump(runs, fh)
        path = fh.name
    try:
        return _run_cpu_child(["gate", "--log", path])
    finally:
        os.unlink(path)


def free_running(torch, ps, depth, P, mults, iters, batch=128, devices=None):
    """Real CIFAR ResNet-`depth` workers on ONE GPU gated by device flags
    (freerun.FreeRunningCluster): each worker's iteration -- forward/backward,
    throttle busy-wait, push kernel, stream wait on its go flag, pull kernel
    -- is one captured CUDA graph; all iterations are enqueued up front, one
    host sync at the end. `mults` are the per-worker slowdowns (the device
    busy-wait adds (m - 1) x the measured single-worker iteration time).
    Returns iterations/s, the fast worker's gate wait, defers, staleness and
    the oracle-gate parity per paradigm."""
    from paper_1908_11848_b200.engine import Engine
    from paper_1908_11848_b200.freerun import FreeRunningCluster
    from paper_1908_11848_b200.workers import CifarResNet, TorchWorker, synthetic_cifar
    torch.manual_seed(0)
    devices = devices or [0] * P
    workers = [TorchWorker(p, CifarResNet(depth), synthetic_cifar(1, batch, seed=p, device=f"cuda:{devices[p]}"),
                           device=f"cuda:{devices[p]}") for p in range(P)]
    d = workers[0].dimension
    w0 = workers[0].params[:d].detach().cpu().numpy().astype(np.float64)
    # single-worker iteration time (the throttle's unit)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for _ in range(3):
            workers[0].step()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            workers[0].step()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(10):
            g.replay()
        e1.record(st)
    torch.cuda.synchronize()
    base_ms = e0.elapsed_time(e1) / 10
    del g
    out, seqs = {}, {}
    for name, s, r in PARADIGMS:
        for wk in workers:
            wk.params.copy_(workers[0].params.to(wk.params.device))
        eng = Engine(name, P, s, r, 0.01, d, w0=w0, device=devices[0])
        cl = FreeRunningCluster(eng, workers, throttle_ns=[int((m - 1) * base_ms * 1e6) for m in mults])
        cl.capture(warmup=1)
        rep = cl.run(iters)
        seqs[name] = {"paradigm": name, "P": P, "s": s, "r": r,
                      "seq": [[w, now, o, list(rel)] for w, now, o, rel in rep.decision_sequence()]}
        out[name] = {"iters_per_s": rep.iters_per_s, "wall_s": rep.wall_s, "iterations": rep.pushes,
                     "fast_worker_wait_s": rep.wait_s(0), "defers": rep.defers(),
                     "max_staleness": rep.max_staleness(),
                     "final_weights_finite": bool(torch.isfinite(workers[0].params[:d]).all().item())}
        del cl
        eng.close()
    parity = gate_check(seqs)
    for name in out:
        out[name]["decisions_identical_to_oracle_gate"] = parity[name]
    return {"model": f"CIFAR ResNet-{depth} ({d:,} params)", "workers": P, "batch": batch,
            "worker_gpus": list(devices), "server_gpu": devices[0],
            "slowdowns": list(mults), "single_worker_iteration_ms": base_ms,
            "host_syncs_per_run": 1, "per_paradigm": out}


def cpu_side_lines(world):
    """BASELINE.md section 2's other CPU figures, on the same pinned core:
    the reference's end-to-end run_simulation of configs[0] ("C1",
    simnet.py:211-218), and -- labelled as NOT the reference -- an fp32
    numpy in-place restatement of the C3 push group (np.multiply into a
    temporary, np.subtract in place: bit-identical to the kernels' arithmetic)."""
    out = {}
    ref = os.path.join(ROOT, "oracle", "_ref")
    if os.path.isdir(os.path.join(ref, "stalesync")):
        if ref not in sys.path:
            sys.path.insert(0, ref)
        from stalesync.config import make_config, validate_config
        from stalesync.simnet import run_simulation
        cfg = validate_config(make_config(
            paradigm="dssp", worker_count=4, s_lower=3, r_max=12, timing_preset="gtx-mix",
            compute_base=1.0, comm_delay=0.05, model_kind="tiny_mlp", dimension=3072,
            dataset_size=512, batch_size=32, learning_rate=0.01, epochs=25, seed=0))
        t0 = time.perf_counter()
        _, report = run_simulation(cfg)
        dt = time.perf_counter() - t0
        out["reference_run_simulation_c1"] = {
            "seconds": dt, "updates": report.updates_total,
            "updates_per_s": report.updates_total / dt,
            "config": "BASELINE configs[0]: tiny_mlp 3072->8->1 (24,593 params), P=4, DSSP(3,12), "
                      "gtx-mix, 25 epochs (SURVEY.md 8(d))"}
    d = C3_DIM
    rng = np.random.default_rng(3)
    w = rng.uniform(-0.5, 0.5, d).astype(np.float32)
    g = rng.standard_normal(d, dtype=np.float32)
    tmp = np.empty_like(w)
    lr = np.float32(0.05)
    reps, t0 = 0, time.perf_counter()
    while time.perf_counter() - t0 < 3.0 or reps < 2:
        for _ in range(world):
            np.multiply(g, lr, out=tmp)
            np.subtract(w, tmp, out=w)
        reps += 1
    dt = time.perf_counter() - t0
    out["fp32_numpy_restatement_not_reference"] = {
        "updates_per_s": reps * world / dt, "gb_per_s": reps * world * 12 * d / dt / 1e9,
        "note": "numpy fp32 in place, 1 core, the C3 push group's applies only (no gate, no pull)"}
    return out


def _run_cpu_child(extra):
    out = subprocess.run([sys.executable, os.path.abspath(__file__), "--cpu-sample"] + extra,
                         capture_output=True, text=True, timeout=900)
    if out.returncode != 0:
        raise RuntimeError("cpu sample failed: " + out.stderr[-2000:])
    return json.loads(out.stdout.strip().splitlines()[-1])


def cpu_baseline_c3(world, applies):
    return _run_cpu_child(["c3", "--world", str(world), "--applies", str(applies)])


def shard_traffic():
    """DRAM bytes per step of k_shard_run at G = 1 from the committed ncu
    capture (profiles/k_shard_run_dram_bytes.json), or None."""
    tpath = os.path.join(ROOT, "profiles", "k_shard_run_dram_bytes.json")
    try:
        return json.load(open(tpath)).get("dram_bytes_per_step")
    except Exception:
        return None


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
        ap, pl, fl = [], [], []
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
                fl.append(eng.profile_floor_ms())
        eng.close()
        a_ms, p_ms, f_ms = statistics.median(ap), statistics.median(pl), statistics.median(fl)
        out.append({"mbytes": mb, "d": d,
                    "apply_ms": round(a_ms, 4), "apply_gbs": round(12 * d / a_ms / 1e6, 1),
                    "apply_frac": round(12 * d / a_ms / 1e6 / hbm_peak, 3),
                    "pull_ms": round(p_ms, 4), "pull_gbs": round(8 * d / p_ms / 1e6, 1),
                    "pull_frac": round(8 * d / p_ms / 1e6 / hbm_peak, 3),
                    # the same event bracket around an empty kernel: the launch
                    # floor inside every figure above
                    "empty_kernel_ms": round(f_ms, 4)})
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
        # host wall time inside the drop-in's calls (each ends in a stream sync,
        # so it includes waiting for the worker's own backward): an upper
        # bound on the server's share, not a device measurement
        out[name] = {"iters_per_s": done / wall, "host_time_in_server_calls_share": ps_s / wall,
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


def _safe(line, key, fn):
    """A side block of the line: its failure is recorded, not fatal to the
    headline (which is measured and checked before any side block runs)."""
    try:
        line[key] = fn()
    except Exception as exc:  # noqa: BLE001 -- reported in the line itself
        import traceback
        line[key] = {"error": f"{type(exc).__name__}: {exc}"[:500],
                     "where": traceback.format_exc().splitlines()[-3:]}


def single_gpu_extras(torch, ps, line):
    """N = 1 blocks beside the C3 headline (rank 0): BASELINE configs[1]
    ("C2") as the reference's recorded request stream served in one kernel,
    the simulated run loop, its e2e variants and CPU figure, the configs[4]
    sweep, configs[3] and the ResNet-20 torch workers."""
    from paper_1908_11848_b200.config import initial_weights_f64
    from paper_1908_11848_b200.engine import Engine
    from paper_1908_11848_b200.sim import DeviceReplay

    hbm_peak, _ = peaks()
    steps, warm = line["steps"], line["warmup"]
    d = C2_DIM
    P, K = 4, 2
    synth_host = synthetic_host(P, K, d)
    synth = torch.from_numpy(synth_host).cuda()
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    w0 = initial_weights_f64(c2_config("dssp", 3, 12), d)
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
        for _ in range(warm):
            replays[name].run(decisions=False)
            sim.run(read_weights=False, reset_gate=True)
    per_paradigm, device_sim, parity = {}, {}, {}
    for name, s, r in PARADIGMS:
        calls, _ = reference_calls(name)
        n_apply = sum(1 for c in calls if c[0] == "apply")
        n_dec = sum(1 for c in calls if c[0] == "decide")
        times, applied = [], 0
        for _ in range(steps):
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
        ms = total_ms / steps
        per_paradigm[name] = {"updates_per_s": applied / (total_ms * 1e-3),
                              "ms_per_step": ms,
                              "us_per_call": 1e3 * ms / len(calls),
                              "us_per_decision": 1e3 * ms / n_dec,
                              "decisions_per_s": n_dec / (ms * 1e-3),
                              "calls_per_step": len(calls), "updates_per_step": n_apply,
                              "defers_per_step": sum(1 for o, _ in check.decisions if o == "defer")}
        parity.setdefault("replay_decisions_identical_to_reference", {})[name] = got == want
    # the same data side with the control taken out (ps_replay_ceiling), on
    # this box: the roofline of the replay, which is latency-, not HBM-bound
    n_pull = sum(1 for c in reference_calls("dssp")[0] if c[0] == "pull")
    n_apply = sum(1 for c in reference_calls("dssp")[0] if c[0] == "apply")
    ceil_ms = replays["dssp"].engine.replay_ceiling_ms(n_pull, n_apply, reps=7)
    data_ceiling = {"ms": ceil_ms, "pulls": n_pull, "applies": n_apply,
                    "frac_of_step": ceil_ms / per_paradigm["dssp"]["ms_per_step"],
                    "what": "every data warp streams the step's pulls (stores of its register-resident "
                            "slice into 8 rotating replicas) and applies (L1-kept loads of 8 rotating "
                            "updates + w - lr*g) with no numbering, gate, verdicts or checkpoints, on the "
                            "replay's own grid and slices; frac_of_step = ceiling / DSSP step"}
    for name, s, r in PARADIGMS:
        cfg, sim = sims[name]
        times, applied = [], 0
        rep = None
        for _ in range(steps):
            flush_l2(torch, flush)
            torch.cuda.synchronize()
            rep = sim.run(read_weights=False, reset_gate=True)
            times.append(rep.device_ms)
            applied += rep.applied
        total_ms = sum(times)
        device_sim[name] = {"updates_per_s": applied / (total_ms * 1e-3),
                            "ms_per_step": total_ms / steps,
                            "virtual_duration_s": max(e.time for e in rep.entries)}
        parity.setdefault("simulation_trace_identical_to_reference", {})[name] = \
            ps.format_trace(rep.entries) == recorded[name]
    for name in replays:
        replays[name].engine.close()
        sims[name][1].engine.close()
    calls, _ = reference_calls("dssp")
    cfg = c2_config("dssp", 3, 12)
    e2e_value, h2d, d2h, e2e_updates = e2e_drop_in(torch, ps, cfg, calls, synth_host, d)
    eb_value, eb_h2d, eb_d2h = e2e_batched(torch, ps, calls, synth_host, d, w0)
    traffic = None
    try:
        traffic = json.load(open(os.path.join(ROOT, "profiles", "k_sim_dram_bytes.json"))).get(
            "dram_bytes_per_launch")
    except Exception:
        pass
    del synth, flush
    torch.cuda.empty_cache()
    line["c2"] = {
        "workload": "C2 (BASELINE configs[1]): ResNet-20-sized single-GPU server d=272474 fp32, "
                    "P=4, gtx-mix; step = the server serving the reference's recorded request "
                    "stream of one run (1,000 pushes, 1,004 pulls, 1,000 decisions) in one kernel",
        "bound": "latency: the 1 MB of weights live in registers and the updates in L1/L2 for "
                 "the whole stream (dram_bytes_per_launch from ncu), so it is reported per call and "
                 "per decision and against data_ceiling (the same loads and stores with no "
                 "control), not as an HBM fraction",
        "dram_bytes_per_launch": traffic,
        "data_ceiling": data_ceiling,
        "value": per_paradigm["dssp"]["updates_per_s"], "unit": "updates/s",
        "per_paradigm": per_paradigm, "device_simulation": device_sim, "parity": parity,
        "e2e": {"value": eb_value, "unit": "updates/s", "h2d_bytes_per_step": eb_h2d,
                "d2h_bytes_per_step": eb_d2h,
                "api": "DeviceReplay.run (C-ABI ps_replay_run) with host buffers: the call "
                       "stream and the resident updates H2D, every decision and the final "
                       "weights D2H, per step"},
        "e2e_per_call": {"value": e2e_value, "unit": "updates/s", "h2d_bytes_per_step": h2d,
                         "d2h_bytes_per_step": d2h, "updates_per_step": e2e_updates,
                         "api": "ParameterServer drop-in (apply_gradient / decide_push / "
                                "handle_pull), pinned host buffers"},
        "cpu_baseline": _run_cpu_child(["c2"]),
    }
    # configs[4] at N = 1: the push-apply / pull kernels 1 MB - 1 GB
    _safe(line, "sweep", lambda: apply_sweep(torch, ps, hbm_peak))
    _safe(line, "c4_throttled", lambda: c4_throttled(torch, ps))
    _safe(line, "c4_free_running", lambda: c4_realtime(torch, ps))
    _safe(line, "torch_workers_c2", lambda: torch_workers(torch, ps))
    # north star (4): real workers blocked and released by device flags, the
    # host out of the iteration loop -- C2-shaped (4 x ResNet-20, 2 of them
    # 2.2x slower like gtx-mix) and configs[3] (3 x ResNet-110 at 1x/2x/4x)
    _safe(line, "free_running_c2", lambda: free_running(torch, ps, 20, 4, (1.0, 1.0, 2.2, 2.2), 40))
    _safe(line, "free_running_c4", lambda: free_running(torch, ps, 110, 3, (1.0, 2.0, 4.0), 24))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="engine", choices=("engine", "reference"))
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--cpu-sample", choices=("c2", "c3", "gate"), default=None)
    ap.add_argument("--log", default=None)
    ap.add_argument("--world", type=int, default=1)
    ap.add_argument("--applies", type=int, default=0)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.cpu_sample == "gate":
        return gate_check_main(args.log)
    if args.cpu_sample:
        return cpu_sample_main(args)
    if args.impl == "reference":
        return run_reference_arm(args)
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    from paper_1908_11848_b200 import sharded
    return sharded.bench_main(args, METRIC, extras=single_gpu_extras if world == 1 else None)


if __name__ == "__main__":
    sys.exit(main())
