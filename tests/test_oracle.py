"""Pin the CPU oracle (test infrastructure) against golden vectors produced by
running the reference itself (tests/golden/make_golden.py)."""

import numpy as np
import pytest

import oracle


def test_controller_tables_c_and_python():
    data = oracle.load_golden("controller_tables.json")
    rows = data["rows"]
    assert len(rows) >= 2200
    for lp, pp, ls, ps, r, want, _src in rows:
        assert oracle.controller(lp, pp, ls, ps, r) == want
    for lp, pp, ls, ps, r, want, _src in rows[::7]:
        assert oracle.controller_py(lp, pp, ls, ps, r) == want


def test_controller_worked_examples():
    # tests/test_policy.py:39-54
    assert oracle.controller(10.0, 9.0, 8.0, 4.0, 4) == 2
    assert oracle.controller(5.0, 4.0, 5.0, 4.0, 6) == 1
    assert oracle.controller(5.0, 4.0, 5.0, 4.0, 0) == 0


@pytest.mark.parametrize("gate_cls", [oracle.CGate, oracle.PyGate])
def test_gate_sequences(gate_cls):
    data = oracle.load_golden("gate_sequences.json.gz")
    n = 0
    for seq in data["sequences"]:
        g = gate_cls(seq["paradigm"], seq["worker_count"], seq["s_lower"], seq["r_max"])
        for w, now, outcome, released, clocks, credits, deferred in seq["steps"]:
            got = g.on_push(w, now)
            assert got == (outcome, tuple(released)), (seq["paradigm"], n)
            assert list(g.clocks) == clocks
            assert list(g.credits) == credits
            assert sorted(g.deferred) == deferred
            n += 1
    assert n > 10000


@pytest.mark.parametrize("gate_cls", [oracle.CGate, oracle.PyGate])
def test_gate_protocol_errors(gate_cls):
    g = gate_cls("ssp", 2, 0, 0)
    assert g.on_push(0, 0.0) == ("defer", ())
    with pytest.raises(oracle.ProtocolViolation):
        g.on_push(0, 1.0)
    with pytest.raises(oracle.ProtocolViolation):
        gate_cls("ssp", 2, 1, 0).on_push(5, 0.0)


@pytest.mark.parametrize("fixture", ["sim_corpus.json.gz", "sim_large.json.gz", "sim_throttle.json.gz"])
def test_gate_replays_simulator_decisions(fixture):
    corpus = oracle.load_golden(fixture)
    for run in corpus["runs"]:
        norm = run["normalized"]
        g = oracle.CGate(norm["paradigm"], norm["worker_count"], norm["s_lower"], norm["r_max"])
        for call in run["calls"]:
            if call[0] == "decide":
                _, p, now, outcome, released = call
                assert g.on_push(p, now) == (outcome, tuple(released)), run["name"]


def test_apply_known_answers():
    data = oracle.load_golden("apply_vectors.json")
    for case in data["cases"]:
        out = oracle.apply_f64(case["w"], case["g"], case["lr"])
        assert np.array_equal(out, np.array(case["out"]))
    div = data["divergence"]
    assert not np.all(np.isfinite(oracle.apply_f64(div["w"], div["g"], div["lr"])))
    rc, _ = oracle.apply_f32_c([1e38, 0.0], [-1e38, 0.0], 10.0)
    assert rc == 2
    rc, _ = oracle.apply_f32_c([0.0, 0.0], [np.nan, 1.0], 0.1)
    assert rc == 1
    for seed, values in data["initial_weights_16"].items():
        assert np.array_equal(oracle.initial_weights_f64(int(seed), 16), np.array(values))


def test_apply_f32_c_matches_numpy_bitwise():
    rng = np.random.default_rng(3)
    w = rng.uniform(-0.5, 0.5, 1 << 16).astype(np.float32)
    g = rng.standard_normal(1 << 16).astype(np.float32)
    rc, out = oracle.apply_f32_c(w, g, 0.05)
    assert rc == 0
    assert np.array_equal(out.view(np.uint32), oracle.apply_f32(w, g, 0.05).view(np.uint32))


@pytest.mark.parametrize("fixture", ["sim_corpus.json.gz", "sim_large.json.gz", "sim_throttle.json.gz"])
def test_bowl_replay_reproduces_reference_fp64(fixture):
    corpus = oracle.load_golden(fixture)
    checked = 0
    for run in corpus["runs"]:
        if run["config"]["model_kind"] != "quadratic_bowl" or "final_weights" not in run:
            continue
        w, version = oracle.replay_bowl(run)
        assert version == run["final_version"]
        assert np.array_equal(w, np.array(run["final_weights"])), run["name"]
        w32, _ = oracle.replay_bowl(run, dtype=np.float32)
        ref = np.array(run["final_weights"])
        err = np.max(np.abs(w32 - ref)) / max(np.max(np.abs(ref)), 1.0)
        assert err <= 1e-5, (run["name"], err)
        checked += 1
    assert checked >= {"sim_corpus.json.gz": 80, "sim_large.json.gz": 16}.get(fixture, 15)


def test_throttled_schedule_matches_config_compute_times():
    """The host schedule generator (config.compute_time_table) reproduces the
    reference's throttled compute draws: every compute_done - pull_return gap
    in the reference traces equals the table entry (constant, jitter and
    lognormal presets scaled 1x/2x/4x)."""
    import paper_1908_11848_b200 as ps
    from paper_1908_11848_b200.config import compute_time_table, push_budget
    for run in oracle.load_golden("sim_throttle.json.gz")["runs"]:
        cfg = ps.validate_config(ps.make_config(**run["config"], throttle=tuple(run["throttle"])))
        table = compute_time_table(cfg, push_budget(cfg))
        last, k = {}, {}
        for line in run["trace"].splitlines()[1:]:
            t, w, kind = line.split("\t")[:3]
            t, w = float(t), int(w)
            if kind == "pull_return":
                last[w] = t
            elif kind == "compute_done":
                i = k.get(w, 0)
                k[w] = i + 1
                assert abs((t - last[w]) - table[w][i]) <= 1e-9 * max(1.0, t), (run["name"], w, i)
