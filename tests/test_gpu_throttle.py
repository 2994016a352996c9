"""BASELINE configs[3] on the device run loop: a 1x/2x/4x throttled cluster.
The reference has no throttle preset, so these check the schedule's defining
properties instead of a golden trace: the compute times are the throttled
ones, the staleness ceiling holds (tests/test_acceptance.py:50-75), and the
dynamic threshold never makes the fastest worker wait longer than SSP
(tests/test_acceptance.py:137-160)."""

import pytest

pytestmark = pytest.mark.gpu

ps = pytest.importorskip("paper_1908_11848_b200")
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
