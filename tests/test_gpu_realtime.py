"""Free-running (wall-clock) mode of the device run loop.

Here the events fire when the GPU's global timer reaches them and each push
is decided at the instant it actually reached the control warp, the way the
reference's threaded runner drives the server (runner.py:168-291,
server.py:93-128). Schedules are therefore not reproducible run to run; what
is checked is that whatever order the run took, the server computed exactly
what the reference computes for that order:

* every recorded push decision equals the C oracle gate fed the same
  (worker, time) sequence (policy.py:108-206);
* the final weights equal, bit for bit, the fp32 replay of the recorded
  pull / adopt / compute / push order (server.py:29-91, engine.py:46-60);
* the deadline and the abort flag stop a run and report the workers still
  outstanding (runner.py:120-164, 294-298).
"""

import threading
import time

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

ps = pytest.importorskip("paper_1908_11848_b200")

CORPUS = [r for r in oracle.load_golden("sim_corpus.json.gz")["runs"]
          if r["config"].get("worker_count", 0) <= 8]
CASES = CORPUS[::4]


def _cfg(run):
    return ps.validate_config(ps.make_config(**run["config"]))


def _span(run):
    return float(run["trace"].strip().splitlines()[-1].split("\t")[0])


def _replay(cfg, entries, d):
    """fp32 quadratic-bowl replay of a trace in its recorded order."""
    seed = cfg.seed
    w = oracle.initial_weights_f64(seed, d).astype(np.float32)
    c = oracle.bowl_center_f64(seed, d).astype(np.float32)
    snap, rep, grad = {}, {}, {}
    applied = 0
    for e in entries:
        if e.kind == "pull_arrive":
            snap[e.worker] = w
        elif e.kind == "pull_return":
            rep[e.worker] = snap.pop(e.worker)
        elif e.kind == "compute_done":
            grad[e.worker] = np.subtract(rep[e.worker], c, dtype=np.float32)
        elif e.kind == "push_arrive":
            w = oracle.apply_f32(w, grad.pop(e.worker), cfg.learning_rate)
            applied += 1
    return w, applied


def _gate_tokens(cfg, entries):
    g = oracle.CGate(cfg.paradigm, cfg.worker_count, cfg.staleness.s_lower, cfg.staleness.r_max)
    out = []
    for e in entries:
        if e.kind == "push_arrive":
            kind, rel = g.on_push(e.worker, e.time)
            out.append(ps.trace.decision_token(kind == "grant", rel))
    return out


@pytest.mark.parametrize("run", CASES, ids=[r["name"] for r in CASES])
def test_free_running_matches_oracle_on_recorded_order(run):
    cfg = _cfg(run)
    d = run["normalized"]["param_dim"]
    scale = 0.03 / _span(run)  # ~30 ms of wall clock per run
    sim = ps.DeviceSimulation(cfg, dimension=d, grad="bowl")
    rep = sim.run(loss_every=0, realtime_scale=scale, deadline_s=20.0)
    assert rep.completed and rep.stuck == []
    entries = rep.entries
    # the loop is causal: times never go backwards
    times = [e.time for e in entries]
    assert all(b >= a for a, b in zip(times, times[1:]))
    pushes = [e for e in entries if e.kind == "push_arrive"]
    assert len(pushes) == cfg.worker_count * sim.budget
    assert [e.decision for e in pushes] == _gate_tokens(cfg, entries)
    w32, applied = _replay(cfg, entries, d)
    assert applied == rep.applied == rep.version
    assert np.array_equal(rep.final_weights.view(np.uint32), w32.view(np.uint32))
    # wall-clock paced: the run cannot finish before its schedule does
    assert rep.device_ms >= 0.9 * _span(run) * scale * 1e3


def test_deadline_reports_stuck_workers_and_engine_survives():
    run = next(r for r in CORPUS if r["name"].startswith("c1_ssp_gtx-mix"))
    cfg = _cfg(run)
    span = _span(run)
    sim = ps.DeviceSimulation(cfg, dimension=4096)
    t0 = time.perf_counter()
    rep = sim.run(loss_every=0, realtime_scale=1.0 / span, deadline_s=0.1)  # 1 s schedule
    assert time.perf_counter() - t0 < 5.0
    assert not rep.completed
    assert rep.stuck and set(rep.stuck) <= set(range(cfg.worker_count))
    pushes = [e for e in rep.entries if e.kind == "push_arrive"]
    assert 0 < len(pushes) < cfg.worker_count * sim.budget
    assert [e.decision for e in pushes] == _gate_tokens(cfg, rep.entries)
    # the same engine runs a full simulated schedule afterwards
    again = sim.run(loss_every=0, reset_gate=True)
    assert ps.format_trace(again.entries) == run["trace"]


def test_abort_from_another_thread():
    run = next(r for r in CORPUS if r["name"].startswith("c1_ssp_gtx-mix"))
    cfg = _cfg(run)
    sim = ps.DeviceSimulation(cfg, dimension=4096)
    timer = threading.Timer(0.2, sim.abort)
    timer.start()
    t0 = time.perf_counter()
    rep = sim.run(loss_every=0, realtime_scale=30.0 / _span(run))  # 30 s schedule, no deadline
    elapsed = time.perf_counter() - t0
    timer.join()
    assert not rep.completed and rep.stuck
    assert elapsed < 10.0


@pytest.mark.parametrize("workers,paradigm", [(12, "dssp"), (24, "ssp"), (32, "dssp")])
def test_free_running_lane_gate_for_larger_clusters(workers, paradigm):
    """9-32 workers run on the lane-per-worker control warp (ctl_lanes.cuh);
    the free-running mode there is held to the same oracle checks."""
    cfg = ps.validate_config(ps.make_config(
        paradigm=paradigm, worker_count=workers, s_lower=2, r_max=6 if paradigm == "dssp" else 0,
        timing_preset="lognormal", compute_base=1.0, comm_delay=0.05, model_kind="quadratic_bowl",
        dimension=257, dataset_size=workers * 8, batch_size=4, epochs=3, learning_rate=0.05, seed=3))
    sim = ps.DeviceSimulation(cfg, dimension=257, grad="bowl")
    ref = sim.run(loss_every=0)                  # simulated: the schedule's length
    span = max(e.time for e in ref.entries)
    sim2 = ps.DeviceSimulation(cfg, dimension=257, grad="bowl")
    rep = sim2.run(loss_every=0, realtime_scale=0.05 / span, deadline_s=20.0)
    assert rep.completed
    pushes = [e for e in rep.entries if e.kind == "push_arrive"]
    assert len(pushes) == workers * sim2.budget
    assert [e.decision for e in pushes] == _gate_tokens(cfg, rep.entries)
    w32, applied = _replay(cfg, rep.entries, 257)
    assert applied == rep.applied
    assert np.array_equal(rep.final_weights.view(np.uint32), w32.view(np.uint32))
