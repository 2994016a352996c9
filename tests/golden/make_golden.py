"""Generate the golden fixtures under tests/golden/ from the REFERENCE itself.

Runs only in the build container, where the read-only reference lives at
/root/reference (PYTHONPATH must reach pkg/src and pkg/tests). Nothing on
the GPU box imports this script; the GPU tests read the committed fixtures.

    PYTHONDONTWRITEBYTECODE=1 \
    PYTHONPATH=/root/reference/pkg/src:/root/reference/pkg/tests \
    python tests/golden/make_golden.py

Fixtures written (all deterministic; re-running reproduces them byte for byte):

  controller_tables.json   (latest_p, prev_p, latest_s, prev_s, r_max) -> r*
                           from stalesync.policy.synchronization_controller,
                           cross-checked against tests/oracles.py:10-28.
                           Same generators as tests/test_policy.py:82-99 and
                           tests/test_acceptance.py:96-134, plus edge cases.
  gate_sequences.json.gz   SyncPolicy.on_push decision streams
                           (stalesync/policy.py:152-206) for all paradigms.
  sim_corpus.json.gz       run_simulation traces (stalesync/simnet.py:127-201)
                           with the full server/worker call log of every run
                           and the fp64 final weights for the small models.
  apply_vectors.json       apply_update / apply_gradient known answers
                           (stalesync/server.py:29-69, tests/test_server.py).
  acceptance_corpora.json.gz  the acceptance suite's corpora at full scale
                           (criteria 1, 2, 4): trace digests, final weights.
  c4_sharded_schedule.json.gz  traces of the bench's throttled cluster across
                           GPUs (P = 2, 4, 8 at 1x/2x/4x, every paradigm).
  c3_schedule.json.gz      run_simulation traces of the bench's homogeneous
                           sharded workload (P = 1, 2, 4, 8, every paradigm).
  sim_throttle.json.gz     run_simulation with 1x/2x/4x throttled workers
                           (BASELINE configs[3]) through a TimingModel
                           subclass (ThrottledTimingModel below).
"""

from __future__ import annotations

import gzip
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

from oracles import controller_oracle  # reference tests/oracles.py
from stalesync.config import GradientVector, WeightVector, make_config, validate_config
from stalesync.policy import (IterationClockTable, ProtocolError, PushHistoryTable,
                              SyncPolicy, synchronization_controller)
from stalesync.server import DivergenceError, ParameterServer, apply_update, initial_weights
from stalesync.simnet import Simulation, TimingModel
from stalesync.trace import format_trace


def _dump(name, obj, gz=False):
    path = os.path.join(HERE, name)
    text = json.dumps(obj, sort_keys=True, separators=(",", ":"))
    if gz:
        with gzip.GzipFile(path, "wb", mtime=0) as fh:
            fh.write(text.encode())
    else:
        with open(path, "w") as fh:
            fh.write(text + "\n")
    print(f"wrote {name}: {os.path.getsize(path)} bytes")


# --------------------------------------------------------------------------
# controller tables
# --------------------------------------------------------------------------

def _two_worker_controller(latest_p, prev_p, latest_s, prev_s, r_max):
    """Same harness as tests/test_policy.py:159-170 (worker 1 slowest)."""
    history = PushHistoryTable(2)
    history.record(0, prev_p)
    history.record(1, prev_s)
    history.record(1, latest_s)
    clocks = IterationClockTable(2)
    for _ in range(5):
        clocks.increment(0)
    clocks.increment(1)
    return synchronization_controller(history, 0, latest_p, clocks, r_max)


def controller_tables():
    rows = []

    def add(lp, pp, ls, ps, r, source):
        got = _two_worker_controller(lp, pp, ls, ps, r)
        want = controller_oracle(lp, pp, ls, ps, r)
        assert got == want, (lp, pp, ls, ps, r)
        rows.append([lp, pp, ls, ps, r, got, source])

    # worked examples, tests/test_policy.py:39-54
    add(10.0, 9.0, 8.0, 4.0, 4, "worked")
    add(5.0, 4.0, 5.0, 4.0, 6, "tie")
    add(5.0, 4.0, 5.0, 4.0, 0, "rmax0")
    # degenerate intervals (floor 1e-9), tests/test_policy.py:67-79
    add(5.0, 5.0, 5.0, 5.0, 7, "zero-interval")
    add(5.0, 6.0, 5.0, 5.0, 7, "negative-interval")
    add(1e9, 1e9 - 1e-6, 1e9 + 0.5, 1e9 - 0.5, 12, "large-offset")
    # tests/test_policy.py:82-99 generator
    rng = np.random.default_rng(20260822)
    for trial in range(600):
        r_max = int(rng.integers(0, 16))
        if trial % 2:
            lp = float(rng.integers(5, 50)); pp = lp - float(rng.integers(1, 9))
            ls = float(rng.integers(5, 50)); ps = ls - float(rng.integers(1, 9))
        else:
            lp = float(rng.uniform(5, 50)); pp = lp - float(rng.uniform(0.01, 9))
            ls = float(rng.uniform(5, 50)); ps = ls - float(rng.uniform(0.01, 9))
        add(lp, pp, ls, ps, r_max, "test_policy")
    # tests/test_acceptance.py:96-134 generator (slowest chosen independently)
    rng = np.random.default_rng(303)
    for trial in range(1200):
        workers = int(rng.integers(2, 7))
        r_max = int(rng.integers(0, 13))
        history = PushHistoryTable(workers)
        latest, previous = {}, {}
        for w in range(workers):
            if trial % 2:
                first = float(rng.integers(1, 40)); second = first + float(rng.integers(1, 9))
            else:
                first = float(rng.uniform(1, 40)); second = first + float(rng.uniform(0.01, 9))
            history.record(w, first); history.record(w, second)
            previous[w], latest[w] = first, second
        clocks = IterationClockTable(workers)
        counts = rng.integers(1, 40, size=workers)
        for w in range(workers):
            for _ in range(int(counts[w])):
                clocks.increment(w)
        pusher = int(rng.integers(0, workers))
        push_time = latest[pusher] + (float(rng.integers(1, 9)) if trial % 2
                                      else float(rng.uniform(0.01, 9)))
        got = synchronization_controller(history, pusher, push_time, clocks, r_max)
        low = min(counts)
        slowest = min(w for w in range(workers) if counts[w] == low)
        previous[pusher], latest[pusher] = latest[pusher], push_time
        want = controller_oracle(latest[pusher], previous[pusher],
                                 latest[slowest], previous[slowest], r_max)
        assert got == want
        rows.append([latest[pusher], previous[pusher], latest[slowest],
                     previous[slowest], r_max, got, "acceptance"])
    # wide r_max and sub-microsecond intervals (device grid sizes)
    rng = np.random.default_rng(77)
    for trial in range(400):
        r_max = int(rng.integers(0, 65))
        base = float(rng.uniform(0, 1e4))
        lp = base + float(rng.uniform(0, 5)); pp = lp - float(rng.uniform(1e-7, 3))
        ls = base + float(rng.uniform(-5, 5)); ps = ls - float(rng.uniform(1e-7, 7))
        add(lp, pp, ls, ps, r_max, "wide")
    _dump("controller_tables.json", {
        "columns": ["latest_p", "prev_p", "latest_s", "prev_s", "r_max", "r_star", "source"],
        "rows": rows})


# --------------------------------------------------------------------------
# gate decision streams
# --------------------------------------------------------------------------

def gate_sequences():
    seqs = []
    rng = np.random.default_rng(4242)
    specs = []
    for paradigm in ("bsp", "asp", "ssp", "dssp"):
        for i in range(18):
            workers = int(rng.integers(1, 9))
            s_lower = int(rng.integers(0, 5))
            r_max = int(rng.integers(0, 13))
            specs.append((paradigm, workers, s_lower, r_max))
    # heavy DSSP: paper default (3, 12) with skewed arrival rates
    for workers in (2, 3, 4, 8):
        specs.append(("dssp", workers, 3, 12))
        specs.append(("dssp", workers, 1, 4))
    for k, (paradigm, workers, s_lower, r_max) in enumerate(specs):
        cfg = validate_config(make_config(paradigm=paradigm, worker_count=workers,
                                          s_lower=s_lower, r_max=r_max))
        policy = SyncPolicy(cfg)
        speeds = rng.uniform(0.2, 3.0, size=workers)
        next_at = {w: float(speeds[w]) for w in range(workers)}
        integer_times = (k % 3 == 0)
        steps = []
        for _ in range(160):
            ready = sorted(set(range(workers)) - policy.deferred)
            if not ready:
                break
            w = min(ready, key=lambda q: (next_at[q], q))
            now = next_at[w]
            if integer_times:
                now = float(round(now))
            d = policy.on_push(w, now)
            steps.append([w, now, d.outcome, list(d.released),
                          [policy.clocks[q] for q in range(workers)],
                          [policy.credits[q] for q in range(workers)],
                          sorted(policy.deferred)])
            next_at[w] = now + float(speeds[w]) * float(rng.uniform(0.5, 1.5))
            for q in d.released:
                next_at[q] = max(next_at[q], now) + float(speeds[q]) * 0.5
        seqs.append({"paradigm": cfg.paradigm, "worker_count": workers,
                     "s_lower": cfg.staleness.s_lower, "r_max": cfg.staleness.r_max,
                     "steps": steps})
    # protocol errors, stalesync/policy.py:153-156
    errors = []
    cfg = validate_config(make_config(paradigm="ssp", worker_count=2, s_lower=0))
    policy = SyncPolicy(cfg)
    errors.append(["ssp", 2, 0, 0, [[0, 0.0, "defer"], [0, 1.0, "ProtocolError"]]])
    try:
        policy.on_push(0, 0.0); policy.on_push(0, 1.0)
        raise AssertionError("expected ProtocolError")
    except ProtocolError:
        pass
    errors.append(["ssp", 2, 1, 0, [[5, 0.0, "ProtocolError"]]])
    _dump("gate_sequences.json.gz", {"sequences": seqs, "protocol_errors": errors}, gz=True)


# --------------------------------------------------------------------------
# simulator corpus with call logs
# --------------------------------------------------------------------------

class _Recorder:
    """Wraps one Simulation's server and workers to log every boundary call
    in order: pull (PULL_ARRIVE snapshot), adopt (PULL_RETURN), grad
    (COMPUTE_DONE), apply, decide."""

    def __init__(self, sim):
        self.log = []
        server = sim.server
        log = self.log
        orig_pull, orig_apply, orig_decide = (server.handle_pull, server.apply_gradient,
                                              server.decide_push)

        def handle_pull(p):
            snap = orig_pull(p)
            log.append(["pull", p, snap.version])
            return snap

        def apply_gradient(g):
            ok = orig_apply(g)
            log.append(["apply", g.source, bool(ok), server.weights.version])
            return ok

        def decide_push(p, now):
            d = orig_decide(p, now)
            log.append(["decide", p, now, d.outcome, list(d.released)])
            return d

        server.handle_pull = handle_pull
        server.apply_gradient = apply_gradient
        server.decide_push = decide_push
        for state in sim.workers:
            orig_begin, orig_adopt = state.begin_iteration, state.adopt

            def begin(state=state, orig=orig_begin):
                g = orig()
                log.append(["grad", state.worker, state.iterations])
                return g

            def adopt(w, state=state, orig=orig_adopt):
                log.append(["adopt", state.worker, w.version])
                return orig(w)

            state.begin_iteration = begin
            state.adopt = adopt


class ThrottledTimingModel(TimingModel):
    """BASELINE configs[3]'s heterogeneous cluster: worker w's compute base is
    multiplied by throttle[w % len(throttle)] (1x / 2x / 4x). The reference
    has no such preset (simnet.py:34-69); this subclass adds one without
    touching the reference: the presets' per-worker bases are scaled after
    construction, and every draw (constant, jitter, lognormal) then uses the
    scaled base exactly as TimingModel.compute_time does."""

    def __init__(self, spec, worker_count, seed, throttle):
        super().__init__(spec, worker_count, seed)
        self._bases = [b * float(throttle[w % len(throttle)]) for w, b in enumerate(self._bases)]


def _run_recorded(flat, keep_weights, throttle=None):
    cfg = validate_config(make_config(**flat))
    sim = Simulation(cfg)
    if throttle:
        sim.timing = ThrottledTimingModel(cfg.timing_model, cfg.worker_count, cfg.seed, throttle)
    rec = _Recorder(sim)
    entries, report = sim.run()
    out = {
        "config": flat,
        "normalized": {"paradigm": cfg.paradigm, "worker_count": cfg.worker_count,
                       "s_lower": cfg.staleness.s_lower, "r_max": cfg.staleness.r_max,
                       "dataset_size": cfg.dataset_size, "learning_rate": cfg.learning_rate,
                       "param_dim": int(sim.model.param_dim)},
        "trace": format_trace(entries),
        "calls": rec.log,
        "updates_total": report.updates_total,
        "duration_s": report.duration_s,
        "final_loss": report.final_loss,
        "final_version": sim.server.weights.version,
        "per_worker": {str(w): [m.iterations, m.epochs, m.wait_s, m.compute_s, m.comm_s]
                       for w, m in report.per_worker.items()},
    }
    if throttle:
        out["throttle"] = list(throttle)
    if keep_weights:
        out["final_weights"] = [float(x) for x in sim.server.weights.values]
        out["loss_curve"] = [[int(v), float(l)] for v, l in report.loss_curve]
    return out


def sim_corpus():
    runs = []
    # tests/test_simnet.py:45-73 golden (SSP(3), P=2, 1 s vs 4 s)
    runs.append(("golden_ssp_fast_slow", dict(
        paradigm="ssp", worker_count=2, s_lower=3, r_max=0, timing_preset="straggler",
        straggler_ratio=4.0, compute_base=1.0, comm_delay=0.0, model_kind="quadratic_bowl",
        dimension=4, dataset_size=16, batch_size=4, epochs=4, seed=1), True))
    # C1 (BASELINE configs[0]): tiny_mlp on 32x32x3-shaped inputs, P=4, DSSP(3,12)
    for preset in ("gtx-mix", "straggler", "lognormal"):
        for seed in ((0, 1, 2) if preset == "lognormal" else (0,)):
            runs.append((f"c1_{preset}_s{seed}", dict(
                paradigm="dssp", worker_count=4, s_lower=3, r_max=12, timing_preset=preset,
                compute_base=1.0, comm_delay=0.05, model_kind="tiny_mlp", dimension=3072,
                dataset_size=512, batch_size=32, learning_rate=0.01, epochs=25, seed=seed,
                loss_every=400), False))
    for paradigm, s, r in (("ssp", 3, 0), ("bsp", 0, 0), ("asp", 0, 0)):
        runs.append((f"c1_{paradigm}_gtx-mix_s0", dict(
            paradigm=paradigm, worker_count=4, s_lower=s, r_max=r, timing_preset="gtx-mix",
            compute_base=1.0, comm_delay=0.05, model_kind="tiny_mlp", dimension=3072,
            dataset_size=512, batch_size=32, learning_rate=0.01, epochs=25, seed=0,
            loss_every=400), False))
    # closed-loop quadratic-bowl runs: every paradigm x preset, several P
    presets = ("homogeneous", "jitter", "gtx-mix", "straggler", "lognormal")
    paradigms = (("bsp", 0, 0), ("asp", 0, 0), ("ssp", 3, 0), ("dssp", 3, 12),
                 ("dssp", 1, 4), ("ssp", 1, 0))
    k = 0
    for preset in presets:
        for paradigm, s, r in paradigms:
            workers = (2, 4, 8)[k % 3]
            runs.append((f"bowl_{paradigm}{s}_{r}_{preset}_p{workers}", dict(
                paradigm=paradigm, worker_count=workers, s_lower=s, r_max=r,
                timing_preset=preset, compute_base=1.0, comm_delay=(0.0, 0.05, 0.01)[k % 3],
                straggler_ratio=(2.0, 3.0, 4.0)[k % 3], model_kind="quadratic_bowl",
                dimension=(64, 257, 1024)[k % 3], dataset_size=16 * workers, batch_size=4,
                learning_rate=0.05, epochs=(6, 10, 8)[k % 3], seed=k), True))
            k += 1
    # criterion-1 style random corpus (tests/test_acceptance.py:50-75)
    rng = np.random.default_rng(101)
    for i in range(60):
        paradigm = "ssp" if i % 2 else "dssp"
        workers = int(rng.integers(2, 9))
        s_lower = int(rng.integers(0, 6))
        r_max = int(rng.integers(1, 9)) if paradigm == "dssp" else 0
        runs.append((f"corpus_{i}", dict(
            paradigm=paradigm, worker_count=workers, s_lower=s_lower, r_max=r_max,
            timing_preset=presets[i % 5], compute_base=1.0,
            comm_delay=(0.0, 0.01, 0.5)[i % 3], straggler_ratio=(1.5, 2.0, 3.0, 4.0)[i % 4],
            model_kind="quadratic_bowl", dimension=2, dataset_size=8 * workers,
            batch_size=4, epochs=int(rng.integers(1, 4)), seed=i), True))
    out = []
    for name, flat, keep in runs:
        rec = _run_recorded(flat, keep)
        rec["name"] = name
        out.append(rec)
    _dump("sim_corpus.json.gz", {"runs": out}, gz=True)


# --------------------------------------------------------------------------
# apply arithmetic
# --------------------------------------------------------------------------

def apply_vectors():
    cases = []

    def grad(values, source=0):
        return GradientVector(np.asarray(values, dtype=np.float64), source, 1)

    for w, g, lr in (([1.0, 2.0], [0.5, -1.0], 0.1), ([0.0, 0.0], [-1.0, -1.0], 0.5),
                     ([1.0, 2.0], [0.0, 0.0], 0.1)):
        out = apply_update(WeightVector(w), grad(g), lr)
        cases.append({"w": w, "g": g, "lr": lr, "out": [float(x) for x in out.values]})
    rng = np.random.default_rng(5)
    for n in (1, 3, 4, 5, 17, 64, 1000):
        w = rng.uniform(-0.5, 0.5, size=n)
        g = rng.normal(size=n)
        lr = float(rng.choice([0.05, 0.01, 0.3, 1.0]))
        out = apply_update(WeightVector(w), grad(g), lr)
        cases.append({"w": [float(x) for x in w], "g": [float(x) for x in g], "lr": lr,
                      "out": [float(x) for x in out.values]})
    # divergence and rejection, stalesync/server.py:38-41, :65-67
    try:
        apply_update(WeightVector([1e308, 0.0]), grad([-1e308, 0.0]), 10.0)
        diverged = False
    except DivergenceError:
        diverged = True
    assert diverged
    cfg = validate_config(make_config(paradigm="asp", worker_count=2, dimension=2, seed=99))
    server = ParameterServer(cfg, 2)
    ok = server.apply_gradient(grad([np.nan, 1.0]))
    init = {}
    for seed in (0, 1, 7, 99, 2 ** 40 + 3):
        c = validate_config(make_config(paradigm="bsp", worker_count=1, seed=seed))
        init[str(seed)] = [float(x) for x in initial_weights(c, 16).values]
    _dump("apply_vectors.json", {
        "cases": cases,
        "divergence": {"w": [1e308, 0.0], "g": [-1e308, 0.0], "lr": 10.0},
        "nan_rejected": {"applied": ok, "rejected_updates": server.rejected_updates},
        "initial_weights_16": init})


def c2_schedule():
    """bench.py's N=1 workload (BASELINE configs[1]): P=4, gtx-mix, 250
    iterations per worker, for each paradigm. The call log fixes the server
    call sequence the reference arm replays and the trace the device run loop
    must reproduce."""
    out = []
    for paradigm, s, r in (("dssp", 3, 12), ("ssp", 3, 0), ("bsp", 0, 0), ("asp", 0, 0)):
        flat = dict(paradigm=paradigm, worker_count=4, s_lower=s, r_max=r,
                    timing_preset="gtx-mix", compute_base=1.0, comm_delay=0.05,
                    model_kind="tiny_mlp", dimension=3072, dataset_size=4000, batch_size=16,
                    learning_rate=0.05, epochs=4, seed=0, loss_every=100000)
        rec = _run_recorded(flat, False)
        rec["name"] = f"c2_{paradigm}"
        out.append(rec)
    _dump("c2_schedule.json.gz", {"runs": out}, gz=True)


def c3_schedule():
    """bench.py's headline workload (BASELINE configs[2], "C3"): P homogeneous
    workers, one per GPU, for P = 1, 2, 4, 8 and every paradigm, 96 pushes
    per worker. The schedule (push instants, ticket order, decisions) does
    not depend on the parameter count, so these traces pin the sharded
    server's decisions at d = 23,528,522 too."""
    out = []
    for workers in (1, 2, 4, 8):
        for paradigm, s, r in (("dssp", 3, 12), ("ssp", 3, 0), ("bsp", 0, 0), ("asp", 0, 0)):
            flat = dict(paradigm=paradigm, worker_count=workers, s_lower=s, r_max=r,
                        timing_preset="homogeneous", compute_base=1.0, comm_delay=0.05,
                        model_kind="quadratic_bowl", dimension=2, dataset_size=96 * workers,
                        batch_size=1, learning_rate=0.05, epochs=1, seed=0, loss_every=100000)
            rec = _run_recorded(flat, False)
            rec["name"] = f"c3_{paradigm}_p{workers}"
            rec.pop("calls")
            out.append(rec)
    _dump("c3_schedule.json.gz", {"runs": out}, gz=True)


def acceptance_corpora():
    """The reference's acceptance corpora at full scale (tests/test_acceptance.py):
    criterion 1's 1000 randomized runs (:50-75), criterion 2's 100 seeds of
    SSP vs DSSP(r_max=0) (:78-93) and criterion 4's 4 ratios x 20 seeds of
    SSP(3) vs DSSP(3,12) (:137-160) -- the exact generators. Each run keeps
    its flat config, the SHA-256 of its rendered trace, its final version and
    fp64 final weights (d = 2 or 3), and criterion 4 the fast worker's wait."""
    import hashlib
    from stalesync.simnet import run_simulation
    presets = ("homogeneous", "jitter", "gtx-mix", "straggler", "lognormal")

    def rec(flat, extra=None):
        cfg = validate_config(make_config(**flat))
        sim = Simulation(cfg)
        entries, report = sim.run()
        text = format_trace(entries)
        out = {"config": flat, "sha256": hashlib.sha256(text.encode()).hexdigest(),
               "rows": len(entries), "final_version": sim.server.weights.version,
               "final_weights": [float(x) for x in sim.server.weights.values],
               "fast_wait_s": report.per_worker[0].wait_s}
        if extra:
            out.update(extra)
        return out

    crit1 = []
    rng = np.random.default_rng(101)
    for i in range(1000):
        paradigm = "ssp" if i % 2 else "dssp"
        workers = int(rng.integers(2, 9))
        s_lower = int(rng.integers(0, 6))
        r_max = int(rng.integers(1, 9)) if paradigm == "dssp" else 0
        crit1.append(rec(dict(
            paradigm=paradigm, mode="simulated", worker_count=workers,
            s_lower=s_lower, r_max=r_max, timing_preset=presets[i % 5],
            compute_base=1.0, comm_delay=(0.0, 0.01, 0.5)[i % 3],
            straggler_ratio=(1.5, 2.0, 3.0, 4.0)[i % 4],
            model_kind="quadratic_bowl", dimension=2,
            dataset_size=8 * workers, batch_size=4,
            epochs=int(rng.integers(1, 4)), seed=i)))
    crit2 = []
    for seed in range(100):
        base = dict(
            mode="simulated", worker_count=2 + seed % 5,
            s_lower=seed % 5, timing_preset=presets[seed % 5],
            compute_base=1.0, comm_delay=(0.0, 0.02)[seed % 2],
            straggler_ratio=2.0 + (seed % 3), model_kind="quadratic_bowl",
            dimension=2, dataset_size=8 * (2 + seed % 5), batch_size=4,
            epochs=2, seed=seed)
        crit2.append([rec(dict(paradigm="ssp", r_max=0, **base)),
                      rec(dict(paradigm="dssp", r_max=0, **base))])
    crit4 = []
    for ratio in (1.5, 2.0, 3.0, 4.0):
        for seed in range(20):
            base = dict(
                mode="simulated", worker_count=2, timing_preset="straggler",
                straggler_ratio=ratio, compute_base=1.0, comm_delay=0.0,
                model_kind="quadratic_bowl", dimension=3, dataset_size=16,
                batch_size=4, epochs=8, seed=seed)
            crit4.append([rec(dict(paradigm="ssp", s_lower=3, **base)),
                          rec(dict(paradigm="dssp", s_lower=3, r_max=12, **base))])
    _dump("acceptance_corpora.json.gz", {"criterion_1": crit1, "criterion_2": crit2,
                                         "criterion_4": crit4}, gz=True)


def sim_throttle():
    """BASELINE configs[3]: workers throttled 1x / 2x / 4x (ThrottledTimingModel),
    every paradigm. The bench's C4 schedule (P = 3, tiny_mlp-shaped budget),
    closed-loop quadratic-bowl runs with final weights at P = 3, 4 and 8
    (throttle cycling over the workers), and the seed-dependent presets
    (jitter, lognormal) under the same multipliers."""
    runs = []
    paradigms = (("dssp", 3, 12), ("ssp", 3, 0), ("bsp", 0, 0), ("asp", 0, 0))
    for paradigm, s, r in paradigms:
        runs.append((f"c4_{paradigm}", dict(
            paradigm=paradigm, worker_count=3, s_lower=s, r_max=r, timing_preset="homogeneous",
            compute_base=1.0, comm_delay=0.05, model_kind="tiny_mlp", dimension=3072,
            dataset_size=3 * 1600, batch_size=16, learning_rate=0.05, epochs=1, seed=0,
            loss_every=100000), False, (1, 2, 4)))
    k = 0
    for workers in (2, 3, 4, 8):
        for paradigm, s, r in paradigms + (("dssp", 1, 4),):
            preset = ("homogeneous", "jitter", "lognormal")[k % 3]
            runs.append((f"throttle_{paradigm}{s}_{r}_{preset}_p{workers}", dict(
                paradigm=paradigm, worker_count=workers, s_lower=s, r_max=r,
                timing_preset=preset, compute_base=1.0, comm_delay=(0.05, 0.01, 0.0)[k % 3],
                model_kind="quadratic_bowl", dimension=(64, 257, 1024)[k % 3],
                dataset_size=16 * workers * 3, batch_size=4, learning_rate=0.05,
                epochs=(2, 3, 2)[k % 3], seed=k + 11), True, (1, 2, 4)))
            k += 1
    out = []
    for name, flat, keep, throttle in runs:
        rec = _run_recorded(flat, keep, throttle)
        rec["name"] = name
        out.append(rec)
    _dump("sim_throttle.json.gz", {"runs": out}, gz=True)


def c4_sharded_schedule():
    """The schedule bench.py's configs[3]-across-GPUs block serves
    (sharded.throttled_bench): P = 2, 4, 8 workers throttled 1x/2x/4x
    (cycling), homogeneous base, every paradigm. The schedule does not
    depend on the parameter count, so a small bowl stands in for the
    ResNet-110-sized server; only the traces are kept."""
    out = []
    for workers in (2, 4, 8):
        throttle = tuple((1, 2, 4)[q % 3] for q in range(workers))
        for paradigm, s, r in (("dssp", 3, 12), ("ssp", 3, 0), ("bsp", 0, 0), ("asp", 0, 0)):
            flat = dict(paradigm=paradigm, worker_count=workers, s_lower=s, r_max=r,
                        timing_preset="homogeneous", compute_base=1.0, comm_delay=0.05,
                        model_kind="quadratic_bowl", dimension=64, dataset_size=workers * 400,
                        batch_size=16, learning_rate=0.05, epochs=1, seed=0, loss_every=100000)
            rec = _run_recorded(flat, False, throttle)
            rec["name"] = f"c4sh_{paradigm}_p{workers}"
            rec.pop("calls")
            out.append(rec)
    _dump("c4_sharded_schedule.json.gz", {"runs": out}, gz=True)


def sim_large():
    """Worker counts beyond the main corpus: P = 1 (serial SGD), and the
    lane-per-worker (9..32) and shared-memory (33..64) control-warp layouts
    of the device run loop, every paradigm, closed-loop quadratic bowl."""
    runs = []
    k = 0
    for workers in (1, 12, 33, 64):
        for paradigm, s, r in (("dssp", 2, 6), ("ssp", 2, 0), ("bsp", 0, 0), ("asp", 0, 0)):
            preset = ("lognormal", "gtx-mix", "straggler", "jitter")[k % 4]
            runs.append((f"large_{paradigm}_p{workers}_{preset}", dict(
                paradigm=paradigm, worker_count=workers, s_lower=s, r_max=r,
                timing_preset=preset, compute_base=1.0, comm_delay=(0.01, 0.05)[k % 2],
                straggler_ratio=3.0, model_kind="quadratic_bowl", dimension=(33, 130)[k % 2],
                dataset_size=8 * workers, batch_size=4, learning_rate=0.05, epochs=3, seed=40 + k),
                True))
            k += 1
    out = []
    for name, flat, keep in runs:
        rec = _run_recorded(flat, keep)
        rec["name"] = name
        out.append(rec)
    _dump("sim_large.json.gz", {"runs": out}, gz=True)


if __name__ == "__main__":
    which = sys.argv[1:] or ["controller", "gate", "sim", "apply", "c2", "large", "throttle", "c3", "acceptance", "c4sh"]
    if "throttle" in which:
        sim_throttle()
    if "c3" in which:
        c3_schedule()
    if "acceptance" in which:
        acceptance_corpora()
    if "c4sh" in which:
        c4_sharded_schedule()
    if "large" in which:
        sim_large()
    if "c2" in which:
        c2_schedule()
    if "controller" in which:
        controller_tables()
    if "gate" in which:
        gate_sequences()
    if "apply" in which:
        apply_vectors()
    if "sim" in which:
        sim_corpus()
