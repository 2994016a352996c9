"""Multi-GPU parity of the sharded server (needs >= 2 GPUs; run with
`gpurun --gpus 2`). Each rank replays the reference's homogeneous schedules:
decisions byte-identical to the reference trace, every shard and every
pulled replica bit-exact against the fp32 oracle."""

import glob
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _gpus():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.parametrize("world,gmax", [(2, 0), (4, 0), (2, 8), (4, 16)])
def test_sharded_parity(tmp_path, world, gmax):
    """gmax > 0 runs the G <= 8 / G <= 16 kernel instantiations on this box's
    GPUs (PS_SHARD_GMAX), the code the 8-GPU runs execute."""
    if _gpus() < world:
        pytest.skip(f"needs {world} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr", "127.0.0.1",
           "--master-port", str(29400 + world + gmax), os.path.join(ROOT, "tests", "_sharded_worker.py"),
           str(tmp_path)]
    env = dict(os.environ, PS_SHARD_GMAX=str(gmax))
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env)
    _check_verdicts(tmp_path, res, world)


def _check_verdicts(tmp_path, res, world):
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    files = sorted(glob.glob(str(tmp_path / "rank*.json")))
    assert len(files) == world
    for f in files:
        v = json.load(open(f))
        assert v["checks"], v
        for c in v["checks"]:
            assert c["trace"] and c["shard"] and c["replica"], json.dumps(c)
            assert c["version"] == c["steps"] * world


@pytest.mark.parametrize("world", [2, 4])
def test_torch_workers_on_the_sharded_server(tmp_path, world):
    """Real ResNet-20 workers whose parameters live in the server's replica
    and whose gradients live in its update buffer: every step's weights equal
    the fp32 replay of all workers' gradients in the gate's ticket order."""
    if _gpus() < world:
        pytest.skip(f"needs {world} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr", "127.0.0.1",
           "--master-port", str(29470 + world), os.path.join(ROOT, "tests", "_sharded_torch_worker.py"),
           str(tmp_path)]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    for f in sorted(glob.glob(str(tmp_path / "torch_rank*.json"))):
        for c in json.load(open(f)):
            assert c["ok"], c
            assert c["version"] == 6 * world, c


def test_sharded_parity_eight_ranks_on_four_gpus(tmp_path):
    """G = 8 (the driver's scaling run) on a 4-GPU box: two ranks per GPU,
    host plumbing over gloo. Every rank runs k_shard_run<8> with seven peers:
    reference traces, shards, replicas, rejection and divergence as above."""
    if _gpus() < 4:
        pytest.skip("needs 4 GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           "--nproc-per-node=8", "--master-addr", "127.0.0.1", "--master-port", "29488",
           os.path.join(ROOT, "tests", "_sharded_worker.py"), str(tmp_path)]
    env = dict(os.environ, PS_SHARD_OVERSUBSCRIBE="1", PS_SHARD_CTAS_PER_SM="1")
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env)
    _check_verdicts(tmp_path, res, 8)


@pytest.mark.parametrize("world", [2, 4])
def test_many_short_lived_servers(world):
    """60 create / run / verify / close cycles of varying sizes: every
    replica bit-exact (guards the initialization ordering of ps_shard_create
    and the collective shutdown)."""
    if _gpus() < world:
        pytest.skip(f"needs {world} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr", "127.0.0.1",
           "--master-port", str(29520 + world), os.path.join(ROOT, "tools", "shard_stress.py"), "60"]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    assert f"stress: 60 servers x {world} ranks, 0 replica mismatches" in res.stdout, res.stdout[-3000:]


@pytest.mark.parametrize("world", [2, 4])
def test_heterogeneous_schedules_on_the_sharded_server(tmp_path, world):
    """Reference runs with stragglers, mixed speeds and jitter: any push group
    and any set of pulling workers per step (ps_shard_run_groups). Decisions
    byte-identical to the reference, every shard the fp32 replay, every
    replica the weights after the group of that worker's last pull."""
    if _gpus() < world:
        pytest.skip(f"needs {world} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr", "127.0.0.1",
           "--master-port", str(29560 + world), os.path.join(ROOT, "tests", "_sharded_groups_worker.py"),
           str(tmp_path)]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    files = sorted(glob.glob(str(tmp_path / "groups_rank*.json")))
    assert len(files) == world
    n = 0
    for f in files:
        for c in json.load(open(f)):
            assert c["trace"] and c["shard"] and c["replica"], json.dumps(c)
            assert c["version"] == c["pushes"], c
            n += 1
    assert n > 0
