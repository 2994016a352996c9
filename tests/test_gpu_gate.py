"""Device gate parity: the CUDA controller and decision machine against the
reference's golden vectors (bit-exact), through the C-ABI."""

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

ps = pytest.importorskip("paper_1908_11848_b200")


def _policy(paradigm, workers, s_lower=0, r_max=0):
    cfg = ps.validate_config(ps.make_config(paradigm=paradigm, worker_count=workers,
                                            s_lower=s_lower, r_max=r_max))
    return ps.SyncPolicy(cfg)


def test_controller_grid_matches_every_golden_table():
    rows = oracle.load_golden("controller_tables.json")["rows"]
    got = ps.controller_batch([r[:4] for r in rows], [r[4] for r in rows])
    want = [r[5] for r in rows]
    bad = [i for i, (a, b) in enumerate(zip(got, want)) if a != b]
    assert not bad, [rows[i] for i in bad[:5]]


def test_controller_random_wide_grids_vs_oracle():
    rng = np.random.default_rng(11)
    n = 4000
    lp = rng.uniform(0, 1e3, n)
    tables = np.stack([lp, lp - rng.uniform(1e-9, 5, n), lp + rng.uniform(-5, 5, n),
                       lp - rng.uniform(1e-9, 9, n)], axis=1)
    tables[::3] = np.round(tables[::3])  # integer timestamps provoke ties
    r = rng.integers(0, 65, n)
    got = ps.controller_batch(tables, r)
    for i in range(n):
        assert got[i] == oracle.controller(*tables[i], int(r[i])), i


def test_worked_example_and_ties():
    # tests/test_policy.py:39-54 through the device grid
    assert list(ps.controller_batch([[10.0, 9.0, 8.0, 4.0], [5.0, 4.0, 5.0, 4.0],
                                     [5.0, 4.0, 5.0, 4.0]], [4, 6, 0])) == [2, 1, 0]


def test_gate_sequences_bit_exact():
    data = oracle.load_golden("gate_sequences.json.gz")
    for seq in data["sequences"]:
        pol = _policy(seq["paradigm"], seq["worker_count"], seq["s_lower"], seq["r_max"])
        for w, now, outcome, released, clocks, credits, deferred in seq["steps"]:
            d = pol.on_push(w, now)
            assert (d.outcome, list(d.released)) == (outcome, released)
            assert [pol.clocks[q] for q in range(seq["worker_count"])] == clocks
            assert [pol.credits[q] for q in range(seq["worker_count"])] == credits
            assert sorted(pol.deferred) == deferred


def test_protocol_errors():
    pol = _policy("ssp", 2, s_lower=0)
    assert pol.on_push(0, 0.0).outcome == ps.DEFER
    with pytest.raises(ps.ProtocolError):
        pol.on_push(0, 1.0)
    with pytest.raises(ps.ProtocolError):
        _policy("ssp", 2, s_lower=1).on_push(5, 0.0)


def test_ssp_defer_and_release():
    # tests/test_policy.py:116-127
    pol = _policy("ssp", 2, s_lower=3)
    for worker in (0, 1, 0, 1, 0, 0, 0):
        assert pol.on_push(worker, 0.0).granted
    assert pol.clocks.counts == {0: 5, 1: 2}
    assert pol.on_push(0, 1.0).outcome == ps.DEFER
    d = pol.on_push(1, 2.0)
    assert d.granted and d.released == (0,)


def test_bsp_barrier_three_workers():
    pol = _policy("bsp", 3)
    assert pol.on_push(0, 0.0).outcome == ps.DEFER
    assert pol.on_push(1, 0.5).outcome == ps.DEFER
    last = pol.on_push(2, 1.0)
    assert last.granted and last.released == (0, 1)


def test_dssp_credit_spend_and_mint():
    # tests/test_policy.py:156-190
    pol = _policy("dssp", 2, s_lower=3, r_max=12)
    pol.credits[0] = 2
    assert pol.on_push(0, 1.0).granted and pol.credits[0] == 1
    assert pol.on_push(0, 2.0).granted and pol.credits[0] == 0
    pol = _policy("dssp", 2, s_lower=1, r_max=4)
    for w, t in ((1, 2.0), (0, 2.5), (1, 4.0), (0, 5.0), (0, 6.0)):
        assert pol.on_push(w, t).granted
    assert pol.on_push(0, 7.0).granted and pol.credits[0] == 1
    assert pol.on_push(0, 8.0).granted and pol.credits[0] == 0


def test_dssp_headroom_cap_and_non_fastest():
    pol = _policy("dssp", 2, s_lower=1, r_max=4)
    for w, t in ((1, 2.0), (0, 2.5), (1, 4.0), (0, 5.0), (0, 6.0)):
        pol.on_push(w, t)
    granted, now = 0, 7.0
    while pol.on_push(0, now).granted:
        granted += 1
        now += 1.0
        assert granted < 50
    assert granted > 0 and pol.clocks[0] - pol.clocks[1] <= 1 + 4 + 1
    pol = _policy("dssp", 3, s_lower=1, r_max=8)
    pol.clocks.counts.update({0: 1, 1: 0, 2: 3})
    assert pol.on_push(0, 5.0).outcome == ps.DEFER
    assert pol.credits[0] == 0


def test_credit_table_rejects_negative():
    pol = _policy("dssp", 2, s_lower=1, r_max=2)
    with pytest.raises(ValueError):
        pol.credits[0] = -1


def test_degeneracy_dssp_zero_credit_equals_ssp():
    for seed in range(4):
        rng = np.random.default_rng(seed)
        ssp, dssp = _policy("ssp", 4, s_lower=2), _policy("dssp", 4, s_lower=2, r_max=0)
        now = 0.0
        for _ in range(120):
            ready = sorted(set(range(4)) - ssp.deferred)
            assert ready == sorted(set(range(4)) - dssp.deferred)
            w = int(rng.choice(ready))
            now += float(rng.uniform(0.01, 1.0))
            assert ssp.on_push(w, now) == dssp.on_push(w, now)
