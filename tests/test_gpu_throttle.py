"""BASELINE configs[3] on the device run loop: a 1x/2x/4x throttled cluster.

The reference has no throttle preset; tests/golden/make_golden.py adds one as
a TimingModel subclass (ThrottledTimingModel: each worker's base scaled by
1x/2x/4x) and records the reference simulator's runs with it
(sim_throttle.json.gz). The device run loop must reproduce those traces byte
for byte, the weights bit-exact against the fp32 replay of the same call
log, and the replayed request streams decision for decision. The property
tests below (staleness ceiling, tests/test_acceptance.py:50-75; DSSP never
waits longer than SSP, :137-160) stay as a second route."""

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

ps = pytest.importorskip("paper_1908_11848_b200")

THROTTLED = oracle.load_golden("sim_throttle.json.gz")["runs"]


def _golden_cfg(run):
    return ps.validate_config(ps.make_config(**run["config"], throttle=tuple(run["throttle"])))


@pytest.mark.parametrize("run", THROTTLED, ids=[r["name"] for r in THROTTLED])
def test_throttled_trace_byte_identical_to_reference(run):
    cfg = _golden_cfg(run)
    d = run["normalized"]["param_dim"]
    rep = ps.DeviceSimulation(cfg, dimension=d, grad="bowl").run(loss_every=0)
    assert ps.format_trace(rep.entries) == run["trace"]
    assert rep.version == run["final_version"]
    if "final_weights" in run:
        w32, version = oracle.replay_bowl(run, dtype=np.float32)
        assert np.array_equal(rep.final_weights.view(np.uint32), w32.view(np.uint32))
        ref = np.array(run["final_weights"])
        err = np.max(np.abs(rep.final_weights - ref)) / max(np.max(np.abs(ref)), 1.0)
        assert err <= 1e-5, err


@pytest.mark.parametrize("run", THROTTLED[:4], ids=[r["name"] for r in THROTTLED[:4]])
def test_throttled_request_stream_replay(run):
    """The C4 (1x/2x/4x, ResNet-110-sized) request streams served by the
    device: every decision as the reference recorded it, weights bit-exact."""
    torch = pytest.importorskip("torch")
    from paper_1908_11848_b200.engine import Engine
    from paper_1908_11848_b200.sim import DeviceReplay
    norm = run["normalized"]
    P, K, d = norm["worker_count"], 2, 1_730_714
    dpad = (d + 3) // 4 * 4
    synth = np.zeros((P, K, dpad), dtype=np.float32)
    for p in range(P):
        for k in range(K):
            synth[p, k, :d] = oracle.synthetic_update(4, p, k, d)
    calls = [tuple(c[:2]) if c[0] != "decide" else ("decide", c[1], c[2])
             for c in run["calls"] if c[0] in ("pull", "apply", "decide")]
    eng = Engine(norm["paradigm"], P, norm["s_lower"], norm["r_max"], norm["learning_rate"], d,
                 w0=oracle.initial_weights_f64(0, d))
    rep = DeviceReplay(eng, calls, torch.from_numpy(synth).cuda(), K).run()
    assert rep.decisions == [(c[3], tuple(c[4])) for c in run["calls"] if c[0] == "decide"]
    w = oracle.initial_weights_f64(0, d).astype(np.float32)
    seen = {}
    for c in calls:
        if c[0] == "apply":
            k = seen.get(c[1], 0)
            seen[c[1]] = k + 1
            w = oracle.apply_f32(w, synth[c[1], k % K, :d], norm["learning_rate"])
    assert np.array_equal(eng.read()[0].view(np.uint32), w.view(np.uint32))
    eng.close()
from paper_1908_11848_b200.metrics import per_worker, staleness_histogram  # noqa: E402


def _cfg(paradigm, s, r, throttle=(1, 2, 4), seed=0):
    return ps.validate_config(ps.make_config(
        paradigm=paradigm, worker_count=3, s_lower=s, r_max=r, timing_preset="homogeneous",
        compute_base=1.0, comm_delay=0.05, throttle=throttle, model_kind="quadratic_bowl",
        dimension=64, dataset_size=3 * 160, batch_size=8, learning_rate=0.05, epochs=2,
        seed=seed))


def test_throttled_compute_times():
    rep = ps.run_device_simulation(_cfg("asp", 0, 0))
    last = {}
    for e in rep.entries:
        if e.kind == "pull_return":
            last[e.worker] = e.time
        elif e.kind == "compute_done":
            assert abs((e.time - last[e.worker]) - (1.0, 2.0, 4.0)[e.worker]) < 1e-9


def test_dssp_adapts_and_respects_ceiling():
    ssp = ps.run_device_simulation(_cfg("ssp", 3, 0))
    dssp = ps.run_device_simulation(_cfg("dssp", 3, 12))
    assert max(staleness_histogram(ssp.entries)) <= 3 + 1
    assert max(staleness_histogram(dssp.entries)) <= 3 + 12 + 1
    w_ssp = per_worker(ssp.entries)[0].wait_s
    w_dssp = per_worker(dssp.entries)[0].wait_s
    assert w_dssp <= w_ssp + 1e-9
    assert w_dssp < w_ssp  # the 4x straggler makes SSP stall the fast worker


def test_unit_throttle_is_homogeneous():
    a = ps.run_device_simulation(_cfg("dssp", 3, 12, throttle=(1, 1, 1)))
    b = ps.run_device_simulation(_cfg("dssp", 3, 12, throttle=()))
    assert ps.format_trace(a.entries) == ps.format_trace(b.entries)
