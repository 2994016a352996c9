"""The reference's acceptance corpora at full scale on the device run loop
(tests/test_acceptance.py criteria 1, 2 and 4 -- 1000 randomized runs, 100
seeds of SSP vs DSSP(r_max=0), 4 ratios x 20 seeds of SSP(3) vs DSSP(3,12)),
recorded from the reference by tests/golden/make_golden.py. Every run's trace
must hash to the reference's (byte-identical decisions, clocks and times),
its final weights must be within the north-star 1e-5 of the reference's fp64
weights, and each criterion must hold on the device's own traces."""

import hashlib

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

ps = pytest.importorskip("paper_1908_11848_b200")
from paper_1908_11848_b200.metrics import per_worker  # noqa: E402

CORPORA = oracle.load_golden("acceptance_corpora.json.gz")


def _run(rec):
    cfg = ps.validate_config(ps.make_config(**rec["config"]))
    rep = ps.run_device_simulation(cfg)
    text = ps.format_trace(rep.entries)
    assert hashlib.sha256(text.encode()).hexdigest() == rec["sha256"], rec["config"]
    assert rep.version == rec["final_version"]
    ref = np.array(rec["final_weights"])
    err = np.max(np.abs(rep.final_weights - ref)) / max(np.max(np.abs(ref)), 1.0)
    assert err <= 1e-5, (rec["config"], err)
    return rep


def _max_gap_at_grants(entries):
    """tests/oracles.py:46-57 on the device trace: the clock gap at every
    granting push, max over the run."""
    clocks, worst = {}, 0
    for e in entries:
        if e.kind == "push_arrive":
            clocks[e.worker] = e.count
            if e.decision.startswith("grant"):
                worst = max(worst, e.count - min(clocks.get(q, 0) for q in range(max(clocks) + 1)))
    return worst


def test_criterion_01_staleness_safety_1000_runs():
    runs = CORPORA["criterion_1"]
    assert len(runs) == 1000
    for rec in runs:
        rep = _run(rec)
        c = rec["config"]
        ceiling = c["s_lower"] + 1 if c["paradigm"] == "ssp" else c["s_lower"] + c["r_max"] + 1
        clocks, worst = [0] * c["worker_count"], 0
        for e in rep.entries:
            if e.kind == "push_arrive":
                clocks[e.worker] = e.count
                if e.decision.startswith("grant"):
                    worst = max(worst, e.count - min(clocks))
        assert worst <= ceiling, (c, worst)


def test_criterion_02_dssp_rmax0_equals_ssp_100_seeds():
    for ssp, dssp in CORPORA["criterion_2"]:
        a, b = _run(ssp), _run(dssp)
        seq = lambda rep: [(e.worker, e.decision) for e in rep.entries if e.kind == "push_arrive"]
        assert seq(a) == seq(b), ssp["config"]["seed"]


def test_criterion_04_waiting_time_dominance_80_runs():
    total = strict = 0
    for ssp, dssp in CORPORA["criterion_4"]:
        a, b = _run(ssp), _run(dssp)
        wa, wb = per_worker(a.entries)[0].wait_s, per_worker(b.entries)[0].wait_s
        assert wa == pytest.approx(ssp["fast_wait_s"], abs=1e-9)
        assert wb == pytest.approx(dssp["fast_wait_s"], abs=1e-9)
        assert wb <= wa + 1e-9
        total += 1
        strict += wb < wa - 1e-9
    assert total == 80 and strict >= 0.8 * total
