"""CPU checks of the sharded server's host logic: shard ranges, the schedule
timestamps, and the torch.distributed plumbing (gloo, world_size 2)."""

import os

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1908_11848_b200 import sharded


@pytest.mark.parametrize("d", [1, 3, 4, 5, 1023, 272_474, 23_528_522])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_shard_ranges_partition_contiguously(d, world):
    lo_prev = 0
    for r in range(world):
        lo, hi = sharded.shard_range(d, world, r)
        assert lo == lo_prev and lo <= hi and (lo % 4 == 0 or lo == d)
        lo_prev = hi
    assert lo_prev == d


def test_homogeneous_push_times_match_reference_traces():
    for run in oracle.load_golden("sim_corpus.json.gz")["runs"]:
        if run["config"].get("timing_preset") != "homogeneous":
            continue
        times = sorted({float(l.split("\t")[0]) for l in run["trace"].splitlines()
                        if l.split("\t")[2] == "push_arrive"})
        cfg = run["config"]
        got = sharded.homogeneous_push_times(cfg["compute_base"], cfg["comm_delay"], len(times))
        assert got == times, run["name"]


def _gloo_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    blobs = sharded.exchange_blobs(bytes([rank]) * (7 + rank))
    m = sharded.max_over_ranks(1.5 * (rank + 1))
    out[rank] = (blobs == [bytes([r]) * (7 + r) for r in range(world)]) and m == 1.5 * world
    dist.destroy_process_group()


def test_plumbing_gloo_world2():
    manager = mp.Manager()
    out = manager.dict()
    mp.spawn(_gloo_worker, args=(2, 29511, out), nprocs=2, join=True)
    assert out[0] and out[1]
