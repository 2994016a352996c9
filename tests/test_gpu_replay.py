"""Replay mode: the device serving the reference's recorded request streams.
Every decision must equal the one the reference recorded for that call, and
the weights the fp32 replay of the same applies."""

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
ps = pytest.importorskip("paper_1908_11848_b200")
from paper_1908_11848_b200.engine import Engine  # noqa: E402
from paper_1908_11848_b200.sim import DeviceReplay, read_replica  # noqa: E402


def _runs():
    # sim_large: P = 1, 12, 33 (the decision word carries at most 55 workers)
    large = [r for r in oracle.load_golden("sim_large.json.gz")["runs"]
             if r["normalized"]["worker_count"] <= 55]
    return oracle.load_golden("sim_corpus.json.gz")["runs"] + \
        oracle.load_golden("c2_schedule.json.gz")["runs"] + large


@pytest.mark.parametrize("d", [5, 4099, 272_474])
def test_replay_decisions_and_weights(d):
    K = 2
    for run in _runs()[:: (1 if d < 100_000 else 9)]:
        norm = run["normalized"]
        P = norm["worker_count"]
        calls = [tuple(c[:2]) if c[0] != "decide" else ("decide", c[1], c[2])
                 for c in run["calls"] if c[0] in ("pull", "apply", "decide")]
        dpad = (d + 3) // 4 * 4
        synth = np.zeros((P, K, dpad), dtype=np.float32)
        for p in range(P):
            for k in range(K):
                synth[p, k, :d] = oracle.synthetic_update(2, p, k, d)
        seed = run["config"].get("seed", 0)
        eng = Engine(norm["paradigm"], P, norm["s_lower"], norm["r_max"], norm["learning_rate"], d,
                     w0=oracle.initial_weights_f64(seed, d))
        rep = DeviceReplay(eng, calls, torch.from_numpy(synth).cuda(), K).run()
        want = [(c[3], tuple(c[4])) for c in run["calls"] if c[0] == "decide"]
        assert rep.decisions == want, run["name"]
        pulls = {}
        w, _, _ = _fp32_replay(calls, synth, d, norm["learning_rate"], seed=seed, pulls=pulls)
        got, _ = eng.read()
        assert np.array_equal(got.view(np.uint32), w.view(np.uint32)), run["name"]
        # every worker's last two pulls (pull k in replica buffer (k + 1) % 2), bit for bit
        _check_replicas(eng, pulls)
        eng.close()


def test_replay_rejects_protocol_violation():
    eng = Engine("ssp", 2, 0, 0, 0.1, 16)
    synth = torch.zeros(2, 1, 16, device="cuda")
    calls = [("apply", 0), ("decide", 0, 1.0), ("pull", 0)]  # worker 0 is deferred, then pulls
    with pytest.raises(ps.ProtocolError):
        DeviceReplay(eng, calls, synth, 1).run()


def _fp32_replay(calls, synth, d, lr, seed=0, reject=lambda p, k: False, pulls=None):
    """fp32 oracle of a replayed stream. With `pulls` (a dict) it also records,
    per worker, the snapshot of each of its pulls under key (worker, (k + 1) % 2):
    what that worker's replica buffer must hold after the run."""
    w = oracle.initial_weights_f64(seed, d).astype(np.float32)
    seen, npull = {}, {}
    applied = rejected = 0
    K = synth.shape[1]
    for c in calls:
        if c[0] == "pull" and pulls is not None:
            k = npull.get(c[1], 0)
            npull[c[1]] = k + 1
            pulls[(c[1], (k + 1) % 2)] = w
        if c[0] == "apply":
            k = seen.get(c[1], 0)
            seen[c[1]] = k + 1
            if reject(c[1], k % K):
                rejected += 1
                continue
            w = oracle.apply_f32(w, synth[c[1], k % K, :d], lr)
            applied += 1
    return w, applied, rejected


def _check_replicas(eng, pulls):
    assert pulls
    for (p, buf), snap in sorted(pulls.items()):
        got = read_replica(eng, p, buf)
        bad = np.flatnonzero(got.view(np.uint32) != snap.view(np.uint32))
        assert bad.size == 0, (p, buf, bad[:8])


def test_replay_stops_data_exactly_at_a_protocol_error():
    """The data warps run ahead of the gate warp but never past its validated
    watermark: a violation deep in the stream (call 70 of 100, applies after
    it) leaves exactly the applies before it in the weights."""
    d, K = 4099, 2
    dpad = (d + 3) // 4 * 4
    synth = np.zeros((2, K, dpad), dtype=np.float32)
    for p in range(2):
        for k in range(K):
            synth[p, k, :d] = oracle.synthetic_update(5, p, k, d)
    calls, t = [], 0.0
    while len(calls) < 69:
        for p in range(2):
            t += 1.0
            calls += [("apply", p), ("decide", p, t), ("pull", p)]
    calls = calls[:69]
    # ASP never defers: make the violation an unknown worker, then more applies
    bad = calls + [("pull", 7)] + [("apply", 0), ("decide", 0, t + 1.0), ("pull", 0)] * 10
    eng = Engine("asp", 2, 0, 0, 0.05, d, w0=oracle.initial_weights_f64(0, d))
    with pytest.raises(ps.ProtocolError):
        DeviceReplay(eng, bad, torch.from_numpy(synth).cuda(), K).run()
    got, _ = eng.read()
    want, applied, _ = _fp32_replay(calls, synth, d, 0.05)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    eng.refresh()
    assert eng.state.version == applied
    eng.close()


@pytest.mark.parametrize("d", [4099, 272_474, 500_000, 1_730_714])
def test_replay_rejects_nonfinite_updates_per_call(d):
    """One non-finite element in one worker's resident update rejects exactly
    the applies that use it (server.py:65-67), across chunk boundaries. The
    sizes cover every data-warp variant: speculative execution with rollback
    (1, 2 and 4 float4 of weights per lane) and the scan-ahead path (16)."""
    run = next(r for r in oracle.load_golden("c2_schedule.json.gz")["runs"] if r["name"] == "c2_dssp")
    norm = run["normalized"]
    K, P = 2, norm["worker_count"]
    dpad = (d + 3) // 4 * 4
    synth = np.zeros((P, K, dpad), dtype=np.float32)
    for p in range(P):
        for k in range(K):
            synth[p, k, :d] = oracle.synthetic_update(6, p, k, d)
    synth[1, 0, d - 99] = np.inf  # worker 1's even-numbered pushes
    calls = [tuple(c[:2]) if c[0] != "decide" else ("decide", c[1], c[2])
             for c in run["calls"] if c[0] in ("pull", "apply", "decide")]
    eng = Engine(norm["paradigm"], P, norm["s_lower"], norm["r_max"], norm["learning_rate"], d,
                 w0=oracle.initial_weights_f64(0, d))
    rep = DeviceReplay(eng, calls, torch.from_numpy(synth).cuda(), K).run()
    pulls = {}
    want, applied, rejected = _fp32_replay(calls, synth, d, norm["learning_rate"],
                                           reject=lambda p, k: p == 1 and k == 0, pulls=pulls)
    assert rep.rejected == rejected > 0 and rep.applied == applied
    got, _ = eng.read()
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    # pull contents: every worker's last two snapshots, bit for bit -- including
    # the pulls the speculative data warps re-executed after rolling back a
    # rejected update (server.py:65-67, :84-91)
    _check_replicas(eng, pulls)
    # decisions do not depend on the data
    assert rep.decisions == [(c[3], tuple(c[4])) for c in run["calls"] if c[0] == "decide"]
    eng.close()


def test_replay_empty_stream_and_worker_limit():
    eng = Engine("dssp", 4, 3, 12, 0.05, 64)
    synth = torch.zeros(4, 1, 64, device="cuda")
    rep = DeviceReplay(eng, [], synth, 1).run()
    assert rep.applied == 0 and rep.decisions == []
    eng.close()
    big = Engine("asp", 56, 0, 0, 0.05, 8)
    with pytest.raises(ValueError):
        DeviceReplay(big, [("pull", 0)], torch.zeros(56, 1, 8, device="cuda"), 1).run()
    big.close()


def test_resident_update_layout_is_validated():
    """The C-ABI takes the resident updates as a bare pointer: the Python side
    rejects anything but a contiguous fp32 [P, count, round_up(d,4)] CUDA
    tensor on the engine's device (misaligned float4 reads otherwise)."""
    eng = Engine("asp", 2, 0, 0, 0.05, 10)
    calls = [("apply", 0), ("decide", 0, 1.0)]
    for bad in (torch.zeros(2, 1, 10, device="cuda"),                  # d not padded to 12
                torch.zeros(2, 1, 12, device="cuda", dtype=torch.float64),
                torch.zeros(2, 2, 12, device="cuda"),                  # count mismatch
                torch.zeros(2, 1, 24, device="cuda")[:, :, ::2],       # not contiguous
                torch.zeros(2, 1, 12)):                                 # host tensor
        with pytest.raises(ValueError):
            DeviceReplay(eng, calls, bad, 1)
    DeviceReplay(eng, calls, torch.zeros(2, 1, 12, device="cuda"), 1).run()
    eng.close()


def test_replay_ceiling_probe():
    """ps_replay_ceiling (measurement export): the C2-shaped data side with no
    control runs, reports a positive time, grows with the call count, and
    refuses a bad request like every other export."""
    eng = Engine("dssp", 4, 3, 12, 0.05, 272_474)
    short = eng.replay_ceiling_ms(100, 100, reps=3)
    full = eng.replay_ceiling_ms(1004, 1000, reps=3)
    assert 0 < short < full
    with pytest.raises(ValueError):
        eng.replay_ceiling_ms(10, 10, reps=0)
    eng.close()
