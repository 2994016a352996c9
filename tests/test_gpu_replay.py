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
from paper_1908_11848_b200.sim import DeviceReplay  # noqa: E402


def _runs():
    return oracle.load_golden("sim_corpus.json.gz")["runs"] + \
        oracle.load_golden("c2_schedule.json.gz")["runs"]


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
        w = oracle.initial_weights_f64(seed, d).astype(np.float32)
        seen = {}
        for c in calls:
            if c[0] == "apply":
                k = seen.get(c[1], 0)
                seen[c[1]] = k + 1
                w = oracle.apply_f32(w, synth[c[1], k % K, :d], norm["learning_rate"])
        got, _ = eng.read()
        assert np.array_equal(got.view(np.uint32), w.view(np.uint32)), run["name"]
        eng.close()


def test_replay_rejects_protocol_violation():
    eng = Engine("ssp", 2, 0, 0, 0.1, 16)
    synth = torch.zeros(2, 1, 16, device="cuda")
    calls = [("apply", 0), ("decide", 0, 1.0), ("pull", 0)]  # worker 0 is deferred, then pulls
    with pytest.raises(ps.ProtocolError):
        DeviceReplay(eng, calls, synth, 1).run()
