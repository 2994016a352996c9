"""The drop-in driven by the REFERENCE's own code.

oracle/stage_ref.sh stages the unmodified stalesync 0.1.0 into oracle/_ref
(it travels to the GPU box with the snapshot; nothing here reads
/root/reference). The reference's own discrete-event simulator
(simnet.py:82-218) then runs with the engine plugged into its two seams:

  * the server seam -- ``sim.server = ParameterServer(...)`` (every
    handle_pull / apply_gradient / decide_push the simulator makes goes to
    the GPU: fp32 weights, device gate);
  * the policy seam -- ``Simulation(config, policy=SyncPolicy(config))``
    (the reference's fp64 server, decisions by the device gate).

Both must reproduce the reference's recorded traces byte for byte; with the
GPU server the closed-loop weights (workers compute on fp32 snapshots) stay
within the north-star 1e-5 of the reference's fp64 weights."""

import os
import sys

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

ps = pytest.importorskip("paper_1908_11848_b200")
REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref")
if not os.path.isdir(os.path.join(REF, "stalesync")):
    pytest.skip("oracle/_ref has no staged stalesync (run oracle/stage_ref.sh)", allow_module_level=True)
if REF not in sys.path:
    sys.path.insert(0, REF)
stalesync = pytest.importorskip("stalesync")
from stalesync.config import make_config, validate_config  # noqa: E402
from stalesync.simnet import Simulation  # noqa: E402
from stalesync.trace import format_trace  # noqa: E402

CORPUS = oracle.load_golden("sim_corpus.json.gz")["runs"]
RUNS = [r for r in CORPUS if r["name"].startswith(("golden", "c1_gtx", "c1_straggler", "c1_ssp", "c1_bsp"))]
RUNS += [r for r in CORPUS if r["name"].startswith("bowl_")][::5]


@pytest.mark.parametrize("run", RUNS, ids=[r["name"] for r in RUNS])
def test_reference_simulator_with_the_gpu_server(run):
    cfg = validate_config(make_config(**run["config"]))
    sim = Simulation(cfg)
    sim.server = ps.ParameterServer(cfg, sim.model.param_dim)
    entries, report = sim.run()
    assert format_trace(entries) == run["trace"]
    assert sim.server.weights.version == run["final_version"]
    if "final_weights" in run:
        ref = np.array(run["final_weights"])
        got = np.asarray(sim.server.weights.values, dtype=np.float64)
        err = np.max(np.abs(got - ref)) / max(np.max(np.abs(ref)), 1.0)
        assert err <= 1e-5, err


@pytest.mark.parametrize("run", RUNS[:6], ids=[r["name"] for r in RUNS[:6]])
def test_reference_simulator_with_the_device_gate_as_policy(run):
    cfg = validate_config(make_config(**run["config"]))
    sim = Simulation(cfg, policy=ps.SyncPolicy(cfg))
    entries, _ = sim.run()
    assert format_trace(entries) == run["trace"]
    if "final_weights" in run:  # the reference's own fp64 server: exact
        assert np.array_equal(np.asarray(sim.server.weights.values), np.array(run["final_weights"]))
