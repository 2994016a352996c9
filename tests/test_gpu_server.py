"""Push-apply / pull parity through the C-ABI: bit-exact against the fp32
restatement of server.py:37, within 1e-5 (normwise) of the fp64 reference, and
the reference's own server tests restated against the drop-in."""

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

ps = pytest.importorskip("paper_1908_11848_b200")


@pytest.fixture(autouse=True, params=[0, 16], ids=["launch", "resident"])
def serving_mode(request, monkeypatch):
    """Every test runs twice: one launch + sync per call, and the resident
    per-call server (a persistent 16-CTA kernel behind a host-mapped mailbox,
    ps_set_resident)."""
    monkeypatch.setenv("PS_RESIDENT", str(request.param))
    return request.param


def _server(paradigm="asp", workers=2, dimension=2, **kw):
    cfg = ps.validate_config(ps.make_config(paradigm=paradigm, worker_count=workers,
                                            dimension=dimension, **kw))
    return ps.ParameterServer(cfg, dimension)


def _g(values, source=0, it=1):
    return ps.GradientVector(np.asarray(values, dtype=np.float64), source, it)


def _bits(a):
    return np.asarray(a, dtype=np.float32).view(np.uint32)


@pytest.mark.parametrize("d", [1, 2, 3, 4, 5, 17, 1023, 4096, 65537, (1 << 20) + 3])
def test_apply_bit_exact_vs_fp32_restatement(d):
    server = _server("asp", 2, d, learning_rate=0.05, seed=3)
    w = oracle.initial_weights_f64(3, d).astype(np.float32)
    for k in range(3):
        g = oracle.synthetic_update(0, k % 2, k, d)
        assert server.apply_gradient(ps.GradientVector(g, k % 2, k))
        w = oracle.apply_f32(w, g, 0.05)
        assert np.array_equal(_bits(server.weights.values), _bits(w))
    assert server.weights.version == 3


def test_apply_fp64_host_and_device_tensor_inputs():
    torch = pytest.importorskip("torch")
    d = 10_001
    server = _server("asp", 2, d, learning_rate=0.3, seed=5)
    w = oracle.initial_weights_f64(5, d).astype(np.float32)
    g64 = np.random.default_rng(1).standard_normal(d)
    server.apply_gradient(_g(g64))
    w = oracle.apply_f32(w, g64.astype(np.float32), 0.3)
    g32 = np.random.default_rng(2).standard_normal(d).astype(np.float32)
    server.apply_gradient(ps.GradientVector(torch.from_numpy(g32).cuda(), 1, 1))
    w = oracle.apply_f32(w, g32, 0.3)
    # an unaligned device view goes through the staging copy
    big = torch.from_numpy(np.concatenate([[0.0], g32]).astype(np.float32)).cuda()
    server.apply_gradient(ps.GradientVector(big[1:], 1, 2))
    w = oracle.apply_f32(w, g32, 0.3)
    assert np.array_equal(_bits(server.weights.values), _bits(w))


def test_normwise_tolerance_vs_fp64_reference_after_many_updates():
    d = 50_000
    server = _server("asp", 4, d, learning_rate=0.05, seed=0)
    w64 = oracle.initial_weights_f64(0, d)
    for k in range(200):
        g = oracle.synthetic_update(0, k % 4, k, d, dtype=np.float64)
        server.apply_gradient(_g(g, k % 4, k))
        w64 = oracle.apply_f64(w64, g, 0.05)
    err = np.max(np.abs(server.weights.values - w64)) / max(np.max(np.abs(w64)), 1.0)
    assert err <= 1e-5, err  # north-star tolerance, stated here


def test_apply_update_arithmetic_known_answers():
    data = oracle.load_golden("apply_vectors.json")
    for case in data["cases"]:
        out = ps.apply_update(ps.WeightVector(case["w"]), _g(case["g"]), case["lr"])
        want = oracle.apply_f32(np.float32(case["w"]), np.float32(case["g"]), case["lr"])
        assert np.array_equal(_bits(out.values), _bits(want))
        assert np.allclose(out.values, case["out"], rtol=1e-6, atol=1e-6)
    with pytest.raises(ps.DivergenceError):
        ps.apply_update(ps.WeightVector([1e38, 0.0]), _g([-1e38, 0.0]), 10.0)
    with pytest.raises(ValueError, match="dimension"):
        ps.apply_update(ps.WeightVector([1.0, 2.0]), _g([1.0, 2.0, 3.0]), 0.1)
    with pytest.raises(ValueError, match="learning_rate"):
        ps.apply_update(ps.WeightVector([1.0, 2.0]), _g([1.0, 2.0]), 0.0)


def test_zero_gradient_still_bumps_version():
    server = _server("asp", 2, 2)
    before = server.weights.values.copy()
    server.apply_gradient(_g([0.0, 0.0]))
    assert server.weights.version == 1
    assert np.array_equal(server.weights.values, before)


def test_non_finite_gradient_rejected_and_counted():
    # tests/test_server.py:91-98
    server = _server("asp")
    before = server.weights
    d = server.handle_push(_g([np.nan, 1.0]), now=0.0)
    assert d.granted
    assert server.rejected_updates == 1
    assert server.weights.version == 0
    assert np.array_equal(server.weights.values, before.values)
    big = _server("asp", 2, 100_003)
    g = np.zeros(100_003)
    g[77_777] = np.inf
    assert not big.apply_gradient(_g(g))
    assert big.weights.version == 0 and big.rejected_updates == 1


def test_divergence_leaves_weights_unchanged():
    server = _server("asp", 2, 8, learning_rate=10.0)
    before = server.weights.values.copy()
    with pytest.raises(ps.DivergenceError):
        server.apply_gradient(_g([-1e38] * 8))
    assert server.weights.version == 0
    assert np.array_equal(server.weights.values, before)


def test_ssp_defer_applies_and_parks():
    # tests/test_server.py:47-61
    server = _server("ssp", workers=2, s_lower=0)
    d = server.handle_push(_g([1.0, 1.0], source=0), now=1.0)
    assert not d.granted and server.weights.version == 1
    assert server.pending == {0: 1.0}
    with pytest.raises(ps.ProtocolError):
        server.handle_pull(0)
    r = server.handle_push(_g([1.0, 1.0], source=1), now=2.0)
    assert r.granted and r.released == (0,) and server.pending == {}
    assert server.handle_pull(0).version == 2


def test_simultaneous_pushes_aggregate_before_decisions():
    # tests/test_server.py:71-88
    server = _server("bsp", workers=2, learning_rate=1.0)
    before = server.weights.values.copy()
    server.apply_gradient(_g([1.0, 0.0], source=0))
    server.apply_gradient(_g([0.0, 1.0], source=1))
    d0 = server.decide_push(0, 3.0)
    d1 = server.decide_push(1, 3.0)
    assert server.weights.version == 2
    assert np.allclose(server.weights.values, before - np.array([1.0, 1.0]))
    assert not d0.granted and d1.granted and d1.released == (0,)
    assert server.handle_pull(0).version == 2


def test_snapshot_isolation_and_unknown_worker():
    server = _server("asp", dimension=2, seed=99)
    snap = server.handle_pull(1)
    server.handle_push(_g([1.0, 1.0], source=0), now=0.0)
    assert snap.version == 0 and server.weights.version == 1
    assert not np.array_equal(snap.values, server.weights.values)
    with pytest.raises(ps.ProtocolError):
        server.handle_pull(7)
    with pytest.raises(ValueError, match="dimension"):
        server.handle_push(_g([1.0, 2.0, 3.0]), now=0.0)


def test_pull_into_device_tensor():
    torch = pytest.importorskip("torch")
    server = _server("asp", 2, 1001, seed=4)
    out = torch.empty(1001, dtype=torch.float32, device="cuda")
    _, version = server.handle_pull(1, out=out)
    assert version == 0
    want = oracle.initial_weights_f64(4, 1001).astype(np.float32)
    assert np.array_equal(_bits(out.cpu().numpy()), _bits(want))
    out64 = torch.empty(1001, dtype=torch.float64, device="cuda")
    server.handle_pull(1, out=out64)
    assert np.array_equal(out64.cpu().numpy(), want.astype(np.float64))


def test_update_count_conservation():
    server = _server("asp", workers=3)
    rng = np.random.default_rng(0)
    for step in range(60):
        server.handle_push(_g(rng.normal(size=2), source=step % 3), float(step))
    assert server.weights.version == 60
    assert sum(server.clocks.counts.values()) == 60


def test_open_loop_replay_of_reference_call_logs():
    """Replay recorded simulator call sequences (tests/golden) through the
    drop-in with synthetic updates: every decision bit-exact, weights
    bit-exact against the fp32 restatement of the same sequence."""
    corpus = oracle.load_golden("sim_corpus.json.gz")
    runs = [r for r in corpus["runs"] if r["name"].startswith(("c1_", "golden", "bowl_dssp3"))]
    assert runs
    for run in runs:
        norm = run["normalized"]
        d = 4099
        cfg = ps.validate_config(ps.make_config(
            paradigm=norm["paradigm"], worker_count=norm["worker_count"],
            s_lower=norm["s_lower"], r_max=norm["r_max"], learning_rate=norm["learning_rate"],
            seed=run["config"].get("seed", 0)))
        server = ps.ParameterServer(cfg, d)
        pushes = {}
        for call in run["calls"]:
            kind, p = call[0], call[1]
            if kind == "apply":
                k = pushes.get(p, 0)
                pushes[p] = k + 1
                server.apply_gradient(ps.GradientVector(oracle.synthetic_update(0, p, k, d), p, k))
            elif kind == "decide":
                dcs = server.decide_push(p, call[2])
                assert (dcs.outcome, list(dcs.released)) == (call[3], call[4]), run["name"]
            elif kind == "pull":
                assert server.handle_pull(p).version == call[2], run["name"]
        want, _ = oracle.replay_open_loop(run, d, seed=0)
        assert np.array_equal(_bits(server.weights.values), _bits(want)), run["name"]


def test_resident_server_retires_when_idle_and_relaunches(serving_mode):
    """The persistent kernel retires after ~2 s without requests (nothing
    spins on the GPU forever) and the next call relaunches it; state reads
    and writes pause it in between."""
    if not serving_mode:
        pytest.skip("resident mode only")
    import time
    d = 4099
    server = _server("ssp", 2, d, s_lower=1, learning_rate=0.05, seed=1)
    w = oracle.initial_weights_f64(1, d).astype(np.float32)
    for k in range(4):
        g = oracle.synthetic_update(9, k % 2, k, d)
        server.handle_push(ps.GradientVector(g, k % 2, k), float(k))
        w = oracle.apply_f32(w, g, 0.05)
        if k == 1:
            time.sleep(2.6)          # the kernel retires here
        if k == 2:
            server.engine.refresh()  # ps_get_state pauses it
    assert np.array_equal(_bits(server.weights.values), _bits(w))
    assert server.weights.version == 4
