"""The replay gate's two implementations against each other and the oracle.

For P <= 8 the replay gate warp evaluates a 32-call chunk's decisions at once
and keeps only the credit / deferred recurrence serial (gate_warp_replay_scan,
csrc/ps_sim.cu); PS_REPLAY_GATE_SCAN=0 selects the decision-at-a-time gate
(gate_on_push semantics, policy.py:152-206). Random request streams -- ties in
time, bursts of one worker, every paradigm, controller grids from r_max = 1 to
40 -- must give the oracle gate's decisions, and streams with
a protocol violation (a pull or push from a deferred worker, an unknown worker)
must stop at the same call with the same gate tables and weights under both.
"""

import ctypes

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
ps = pytest.importorskip("paper_1908_11848_b200")
from paper_1908_11848_b200.engine import Engine  # noqa: E402
from paper_1908_11848_b200.sim import DeviceReplay  # noqa: E402

D, K, LR = 1031, 2, 0.05


def _stream(rng, paradigm, P, s, r, n_decides, violation=None):
    """A protocol-following stream generated against the oracle gate, with
    its expected decisions. `violation` ("pull" | "decide" | "unknown") adds
    one bad call at a random point once a worker is deferred (unknown: any
    point) followed by more ordinary traffic."""
    gate = oracle.CGate(paradigm, P, s, r)
    calls, want = [], []
    t = 0.0
    speed = [1.0, 2.0, 4.0, 1.5, 3.0, 1.0, 2.5, 1.2, 5.0][:P] + [1.0] * max(0, P - 9)
    bad_at = int(rng.integers(n_decides // 4, n_decides)) if violation else -1
    injected = False
    for i in range(n_decides):
        free = [q for q in range(P) if q not in gate.deferred]
        if not free:
            break
        p = int(rng.choice(free)) if rng.random() < 0.7 else int(free[0])
        if rng.random() < 0.8:  # ~20 % of pushes tie with the previous one
            t += float(rng.exponential(0.5)) * speed[p]
        calls += [("apply", p), ("decide", p, t)]
        outcome, released = gate.on_push(p, t)
        want.append((outcome, tuple(released)))
        if outcome == "grant":
            calls.append(("pull", p))
        for q in released:
            calls.append(("pull", q))
        if violation and not injected and i >= bad_at:
            dq = sorted(gate.deferred)
            if violation == "unknown":
                calls.append(("pull", P + 3))
                injected = True
            elif dq:
                q = dq[0]
                calls.append(("pull", q) if violation == "pull" else ("decide", q, t + 1.0))
                injected = True
    return calls, want, injected


def _run(calls, paradigm, P, s, r, scan, monkeypatch):
    monkeypatch.setenv("PS_REPLAY_GATE_SCAN", "1" if scan else "0")
    dpad = (D + 3) // 4 * 4
    synth = np.zeros((P, K, dpad), dtype=np.float32)
    for p in range(P):
        for k in range(K):
            synth[p, k, :D] = oracle.synthetic_update(9, p, k, D)
    eng = Engine(paradigm, P, s, r, LR, D, w0=oracle.initial_weights_f64(3, D))
    err, dec = None, None
    try:
        dec = DeviceReplay(eng, calls, torch.from_numpy(synth).cuda(), K).run().decisions
    except ps.ProtocolError as e:
        err = type(e)
    st = eng.refresh()
    state = bytes(ctypes.string_at(ctypes.addressof(st), ctypes.sizeof(st)))
    w, _ = eng.read()
    eng.close()
    return err, dec, state, w


CONFIGS = [("dssp", 2, 3, 12), ("dssp", 3, 3, 12), ("dssp", 4, 3, 12), ("dssp", 4, 1, 4),
           ("dssp", 4, 0, 2), ("dssp", 5, 2, 1), ("dssp", 8, 3, 16), ("dssp", 8, 3, 17),
           ("dssp", 4, 2, 40), ("dssp", 9, 3, 12), ("ssp", 4, 2, 0), ("bsp", 3, 0, 0),
           ("asp", 4, 0, 0)]


@pytest.mark.parametrize("paradigm,P,s,r", CONFIGS)
def test_scan_gate_decisions_equal_oracle(paradigm, P, s, r, monkeypatch):
    rng = np.random.default_rng(P * 100 + r)
    for trial in range(4):
        calls, want, _ = _stream(rng, paradigm, P, s, r, 150 + 40 * trial)
        got = {}
        for scan in (1, 0):
            err, dec, state, w = _run(calls, paradigm, P, s, r, scan, monkeypatch)
            assert err is None
            assert dec == want, (paradigm, P, s, r, trial, scan)
            got[scan] = (state, w.view(np.uint32).copy())
        assert got[0][0] == got[1][0]
        assert np.array_equal(got[0][1], got[1][1])


@pytest.mark.parametrize("violation", ["pull", "decide", "unknown"])
@pytest.mark.parametrize("paradigm,P,s,r", [("dssp", 4, 3, 12), ("dssp", 3, 1, 4), ("ssp", 4, 1, 0),
                                            ("bsp", 2, 0, 0), ("dssp", 8, 2, 6)])
def test_scan_gate_protocol_errors_match_serial_gate(paradigm, P, s, r, violation, monkeypatch):
    rng = np.random.default_rng(7 + P + r)
    checked = 0
    for trial in range(6):
        calls, _, injected = _stream(rng, paradigm, P, s, r, 120, violation=violation)
        if not injected:
            continue
        a = _run(calls, paradigm, P, s, r, 1, monkeypatch)
        b = _run(calls, paradigm, P, s, r, 0, monkeypatch)
        assert a[0] is ps.ProtocolError and b[0] is ps.ProtocolError
        assert a[2] == b[2], (paradigm, P, violation, trial)  # gate tables, version, counters
        assert np.array_equal(a[3].view(np.uint32), b[3].view(np.uint32))
        checked += 1
    assert checked >= 2
