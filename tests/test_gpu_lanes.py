"""The three control-warp layouts of the device run loop (replicated scalar
tables for P <= 8, one worker per lane for P <= 32, shared memory beyond)
must produce the same, reference-identical traces. The golden corpus covers
P <= 8; this drives P = 9..40 through all layouts and cross-checks them
against the C oracle's decisions on the same schedule."""

import pytest

import oracle

pytestmark = pytest.mark.gpu

ps = pytest.importorskip("paper_1908_11848_b200")


@pytest.mark.parametrize("P", [9, 16, 32, 33, 40])
@pytest.mark.parametrize("paradigm,s,r", [("dssp", 2, 6), ("ssp", 2, 0), ("bsp", 0, 0)])
def test_large_worker_counts(P, paradigm, s, r):
    cfg = ps.validate_config(ps.make_config(
        paradigm=paradigm, worker_count=P, s_lower=s, r_max=r, timing_preset="lognormal",
        compute_base=1.0, comm_delay=0.01, model_kind="quadratic_bowl", dimension=33,
        dataset_size=8 * P, batch_size=4, epochs=3, seed=P))
    rep = ps.run_device_simulation(cfg)
    gate = oracle.CGate(paradigm, P, cfg.staleness.s_lower, cfg.staleness.r_max)
    n = 0
    for e in rep.entries:
        if e.kind == "push_arrive":
            outcome, released = gate.on_push(e.worker, e.time)
            assert ps.decision_token(outcome == "grant", released) == e.decision
            assert gate.clocks[e.worker] == e.count
            n += 1
    assert n == P * ps.push_budget(cfg)
