"""One rank of the heterogeneous-schedule check of the sharded server
(launched by tests/test_gpu_sharded.py under torchrun). Replays reference
runs with stragglers / mixed speeds / jitter -- any push group, any set of
pulling workers per step -- and checks decisions, shards and replicas."""

import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import paper_1908_11848_b200 as ps  # noqa: E402
from paper_1908_11848_b200.sharded import ShardedServer, groups_from_trace  # noqa: E402
from paper_1908_11848_b200.trace import TraceEntry  # noqa: E402


def _entries(text):
    out = []
    for line in text.splitlines():
        t, w, kind, c, dec = line.split("\t")
        out.append(TraceEntry(float(t), int(w), kind, int(c), dec))
    return out


def main(out_dir):
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    runs = [r for r in oracle.load_golden("sim_corpus.json.gz")["runs"]
            if r["config"].get("timing_preset") != "homogeneous"
            and r["normalized"]["worker_count"] == world
            and r["config"].get("model_kind") == "quadratic_bowl"]
    # BASELINE configs[3]: the reference's runs with 1x/2x/4x throttled workers
    runs += [r for r in oracle.load_golden("sim_throttle.json.gz")["runs"]
             if r["normalized"]["worker_count"] == world]
    checks = []
    for d in (5, 100_003):
        for run in runs:
            cfg = ps.validate_config(ps.make_config(**run["config"],
                                                    throttle=tuple(run.get("throttle", ()))))
            entries = _entries(run["trace"])
            groups = groups_from_trace(entries)
            w0 = oracle.initial_weights_f64(cfg.seed, d)
            srv = ShardedServer(cfg, d, rank, world, local, w0_host=w0)
            gs = [oracle.synthetic_update(4, p, 0, d) for p in range(world)]
            srv.update[:d].copy_(torch.from_numpy(gs[rank]))
            torch.cuda.synchronize()
            dist.barrier()
            # two runs: the trace and the gate carry over (and the trace
            # buffer grows between them)
            srv.run_groups(groups[:3])
            srv.run_groups(groups[3:])
            got = [e.render().split("\t") for e in srv.trace()]
            want = [line.split("\t") for line in run["trace"].splitlines()
                    if line.split("\t")[2] == "push_arrive"]
            # fp32 replay: every group's updates in ticket order; a worker's
            # replica holds the weights after the group of its last pull
            w = w0.astype(np.float32)
            mine = w.copy()
            for _, order, pulls in groups:
                for p in order:
                    w = oracle.apply_f32(w, gs[p], cfg.learning_rate)
                if rank in pulls:
                    mine = w.copy()
            shard, rep = srv.read_shard(), srv.read_replica()
            checks.append({
                "run": run["name"], "d": d, "groups": len(groups),
                "trace": got == want,
                "shard": bool(np.array_equal(shard.view(np.uint32), w[srv.lo:srv.hi].view(np.uint32))),
                "replica": bool(np.array_equal(rep.view(np.uint32), mine.view(np.uint32))),
                "version": int(srv.state().version), "pushes": len(want)})
            torch.cuda.synchronize()
            dist.barrier()
            srv.close()
    # a pusher first seen late in a run with a non-finite update: the
    # pipelined run_groups must judge its first group in full (redo without
    # it) and skip it afterwards -- rejected at every push (server.py:65-67)
    d = 100_003
    cfg = ps.validate_config(ps.make_config(paradigm="asp", worker_count=world, dimension=d,
                                            learning_rate=0.05, seed=8))
    w0 = oracle.initial_weights_f64(8, d)
    srv = ShardedServer(cfg, d, rank, world, local, w0_host=w0)
    late = world - 1
    gs = [oracle.synthetic_update(11, p, 0, d) for p in range(world)]
    gs[late][d // 2] = np.nan
    srv.update[:d].copy_(torch.from_numpy(gs[rank]))
    torch.cuda.synchronize()
    dist.barrier()
    early = list(range(world - 1))
    groups = []
    for i in range(9):
        order = early + ([late] if i in (3, 6, 7) else [])
        groups.append((float(i + 1), order, list(order)))
    srv.run_groups(groups)
    w = w0.astype(np.float32)
    mine = w.copy()
    for _, order, pulls in groups:
        for p in order:
            if p != late:
                w = oracle.apply_f32(w, gs[p], cfg.learning_rate)
        if rank in pulls:
            mine = w.copy()
    st = srv.state()
    checks.append({
        "run": "late_pusher_rejected", "d": d, "groups": len(groups),
        "trace": int(st.rejected) == 3,
        "shard": bool(np.array_equal(srv.read_shard().view(np.uint32), w[srv.lo:srv.hi].view(np.uint32))),
        "replica": bool(np.array_equal(srv.read_replica().view(np.uint32), mine.view(np.uint32))),
        "version": int(st.version) + int(st.rejected), "pushes": sum(len(g[1]) for g in groups)})
    torch.cuda.synchronize()
    dist.barrier()
    srv.close()
    with open(os.path.join(out_dir, f"groups_rank{rank}.json"), "w") as fh:
        json.dump(checks, fh)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1])
