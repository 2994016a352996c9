"""One rank of the multi-GPU parity check (launched by tests/test_gpu_sharded.py
under torchrun). Replays reference homogeneous schedules (tests/golden) on
the sharded server and writes this rank's verdict as JSON."""

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
from paper_1908_11848_b200.sharded import ShardedServer  # noqa: E402


def main(out_dir):
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ["LOCAL_RANK"])
    # PS_SHARD_OVERSUBSCRIBE=1: more ranks than GPUs (ranks share GPUs round-
    # robin, host plumbing over gloo) -- exercises G = 8 on a 4-GPU box
    if os.environ.get("PS_SHARD_OVERSUBSCRIBE") == "1":
        local = local % torch.cuda.device_count()
        torch.cuda.set_device(local)
        dist.init_process_group("gloo")
    else:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    verdict = {"rank": rank, "checks": []}
    runs = [r for r in oracle.load_golden("sim_corpus.json.gz")["runs"]
            if r["config"].get("timing_preset") == "homogeneous"
            and r["normalized"]["worker_count"] == world]
    only = os.environ.get("PS_TEST_ONLY_RUN")  # diagnosis: one run, one size
    if only:
        runs = [r for r in runs if r["name"] == only]
    # C3 at full size (BASELINE configs[2]: d = 23,528,522, the bench's shard
    # size, CTA-count trim and redo geometry) on the first homogeneous run
    from paper_1908_11848_b200.sharded import C3_DIM
    sizes = (100_003,) if only else (5, 100_003, C3_DIM)
    for d in sizes:
        for run in (runs[:1] if d == C3_DIM else runs):
            cfg = ps.validate_config(ps.make_config(**run["config"]))
            rows = [line.split("\t") for line in run["trace"].splitlines()]
            pushes = [r for r in rows if r[2] == "push_arrive"]
            times = sorted({float(r[0]) for r in pushes})
            w0 = oracle.initial_weights_f64(cfg.seed, d)
            srv = ShardedServer(cfg, d, rank, world, local, w0_host=w0)
            g = oracle.synthetic_update(0, rank, 0, d)
            srv.update[:d].copy_(torch.from_numpy(g))
            torch.cuda.synchronize()
            dist.barrier()
            srv.run(times)
            got = [e.render().split("\t") for e in srv.trace()]
            want = [[r[0], r[1], r[2], r[3], r[4]] for r in pushes]
            # oracle: every group applies its updates in the reference's ticket
            # order (the order of the group's push rows in the reference trace)
            w = w0.astype(np.float32)
            gs = [oracle.synthetic_update(0, p, 0, d) for p in range(world)]
            for r in pushes:
                w = oracle.apply_f32(w, gs[int(r[1])], cfg.learning_rate)
            shard = srv.read_shard()
            rep = srv.read_replica()
            ok_trace = got == want
            ok_shard = bool(np.array_equal(shard.view(np.uint32), w[srv.lo:srv.hi].view(np.uint32)))
            ok_rep = bool(np.array_equal(rep.view(np.uint32), w.view(np.uint32)))
            st = srv.state()
            diff = [(a, b) for a, b in zip(got, want) if a != b][:3]
            if not ok_rep:
                bad = np.nonzero(rep.view(np.uint32) != w.view(np.uint32))[0]
                diff = {"replica_mismatches": int(bad.size), "first": int(bad[0]), "last": int(bad[-1]),
                        "lo_hi": [srv.lo, srv.hi],
                        "got": float(rep[bad[0]]), "want": float(w[bad[0]]),
                        "w0": float(w0[bad[0]]),
                        "stale_equals_w0": bool(np.all(rep[bad] == w0[bad].astype(np.float32)))}
            verdict["checks"].append({"run": run["name"], "d": d, "trace": ok_trace,
                                      "diff": diff, "n_got": len(got), "n_want": len(want),
                                      "shard": ok_shard, "replica": ok_rep,
                                      "version": int(st.version), "steps": len(times)})
            torch.cuda.synchronize()
            dist.barrier()
            srv.close()
    # rejection across shards: worker 1's update is non-finite in ONE element,
    # inside shard 0 only; every owner must reject it whole (server.py:65-67)
    d = 100_003
    cfg = ps.validate_config(ps.make_config(paradigm="asp", worker_count=world, dimension=d,
                                            learning_rate=0.05, seed=3))
    w0 = oracle.initial_weights_f64(3, d)
    srv = ShardedServer(cfg, d, rank, world, local, w0_host=w0)
    g = oracle.synthetic_update(1, rank, 0, d)
    if rank == 1:
        g[7] = np.nan
    srv.update[:d].copy_(torch.from_numpy(g))
    torch.cuda.synchronize()
    dist.barrier()
    srv.run([1.0, 2.0])
    w = w0.astype(np.float32)
    for _ in range(2):
        for p in range(world):
            if p != 1:
                w = oracle.apply_f32(w, oracle.synthetic_update(1, p, 0, d), 0.05)
    st = srv.state()
    rep = srv.read_replica()
    bad = np.nonzero(rep.view(np.uint32) != w.view(np.uint32))[0]
    verdict["checks"].append({
        "run": "reject", "d": d, "trace": True,
        "diff": {} if bad.size == 0 else {"replica_mismatches": int(bad.size), "first": int(bad[0]),
                                          "last": int(bad[-1]), "lo_hi": [srv.lo, srv.hi],
                                          "stale_equals_w0": bool(np.all(rep[bad] == w0[bad].astype(np.float32)))},
        "shard": bool(np.array_equal(srv.read_shard().view(np.uint32), w[srv.lo:srv.hi].view(np.uint32))),
        "replica": bool(np.array_equal(srv.read_replica().view(np.uint32), w.view(np.uint32))),
        "version": int(st.version) + int(st.rejected), "steps": 2,
        "rejected": int(st.rejected)})
    assert int(st.rejected) == 2, int(st.rejected)
    torch.cuda.synchronize()
    dist.barrier()
    srv.close()
    # divergence: finite updates whose result overflows in ONE element of
    # shard 0 -> DivergenceError on every rank, weights unchanged
    # (server.py:38-41), and the run ends without a watchdog
    cfg = ps.validate_config(ps.make_config(paradigm="asp", worker_count=world, dimension=d,
                                            learning_rate=0.5, seed=3))
    w0 = oracle.initial_weights_f64(3, d)
    w0[7] = 3.0e38
    srv = ShardedServer(cfg, d, rank, world, local, w0_host=w0)
    g = oracle.synthetic_update(1, rank, 0, d)
    if rank == 1:
        g[7] = -3.4e38
    srv.update[:d].copy_(torch.from_numpy(g))
    torch.cuda.synchronize()
    dist.barrier()
    diverged = False
    try:
        srv.run([1.0])
    except ps.DivergenceError:
        diverged = True
    w = w0.astype(np.float32)
    verdict["checks"].append({
        "run": "diverge", "d": d, "trace": diverged,
        "shard": bool(np.array_equal(srv.read_shard().view(np.uint32), w[srv.lo:srv.hi].view(np.uint32))),
        "replica": True, "version": int(srv.state().version), "steps": 0})
    torch.cuda.synchronize()
    dist.barrier()
    srv.close()
    # the lagged pipeline (runs of > 2 steps: step k starts once every owner
    # finished step k-2): a rejected update over 6 steps, rejected at every
    # push, and a divergence at step 15 of 20 -- every rank stops there with
    # the weights of step 14 (server.py:38-41, :65-67)
    cfg = ps.validate_config(ps.make_config(paradigm="asp", worker_count=world, dimension=d,
                                            learning_rate=0.05, seed=5))
    w0 = oracle.initial_weights_f64(5, d)
    srv = ShardedServer(cfg, d, rank, world, local, w0_host=w0)
    g = oracle.synthetic_update(7, rank, 0, d)
    if rank == world - 1:
        g[d - 3] = np.inf
    srv.update[:d].copy_(torch.from_numpy(g))
    torch.cuda.synchronize()
    dist.barrier()
    srv.run([float(i + 1) for i in range(6)])
    w = w0.astype(np.float32)
    for _ in range(6):
        for p in range(world - 1):
            w = oracle.apply_f32(w, oracle.synthetic_update(7, p, 0, d), 0.05)
    st = srv.state()
    verdict["checks"].append({
        "run": "reject_lagged", "d": d, "trace": int(st.rejected) == 6,
        "shard": bool(np.array_equal(srv.read_shard().view(np.uint32), w[srv.lo:srv.hi].view(np.uint32))),
        "replica": bool(np.array_equal(srv.read_replica().view(np.uint32), w.view(np.uint32))),
        "version": int(st.version) + int(st.rejected), "steps": 6})
    torch.cuda.synchronize()
    dist.barrier()
    srv.close()
    cfg = ps.validate_config(ps.make_config(paradigm="asp", worker_count=world, dimension=d,
                                            learning_rate=0.5, seed=5))
    w0 = oracle.initial_weights_f64(5, d)
    w0[11] = 2.0e38
    srv = ShardedServer(cfg, d, rank, world, local, w0_host=w0)
    g = oracle.synthetic_update(8, rank, 0, d)
    g[11] = -2.0e37 if rank == 0 else 0.0
    srv.update[:d].copy_(torch.from_numpy(g))
    torch.cuda.synchronize()
    dist.barrier()
    diverged = False
    try:
        srv.run([float(i + 1) for i in range(20)])
    except ps.DivergenceError:
        diverged = True
    gs = [oracle.synthetic_update(8, p, 0, d) for p in range(world)]
    for p in range(world):
        gs[p][11] = -2.0e37 if p == 0 else 0.0
    w = w0.astype(np.float32)
    steps_ok = 0
    while True:
        nxt = w
        for p in range(world):
            nxt = oracle.apply_f32(nxt, gs[p], 0.5)
        if not np.all(np.isfinite(nxt)):
            break
        w = nxt
        steps_ok += 1
    verdict["checks"].append({
        "run": "diverge_lagged", "d": d, "trace": diverged and steps_ok < 20,
        "shard": bool(np.array_equal(srv.read_shard().view(np.uint32), w[srv.lo:srv.hi].view(np.uint32))),
        "replica": True, "version": int(srv.state().version), "steps": steps_ok,
        "steps_before_divergence": steps_ok})
    torch.cuda.synchronize()
    dist.barrier()
    srv.close()
    # divergence at the pipeline's boundaries: the first lagged resolve
    # (steps 1 and 2 of a run), and the run's last step -- the weights must
    # be the input of the failing step on every rank
    for start, n_steps in ((3.25e38, 6), (3.15e38, 6), (2.9e38, 6), (2.3e38, 8)):
        cfg = ps.validate_config(ps.make_config(paradigm="asp", worker_count=world, dimension=d,
                                                learning_rate=0.5, seed=6))
        w0 = oracle.initial_weights_f64(6, d)
        w0[13] = start
        srv = ShardedServer(cfg, d, rank, world, local, w0_host=w0)
        g = oracle.synthetic_update(9, rank, 0, d)
        g[13] = -2.0e37 if rank == 0 else 0.0
        srv.update[:d].copy_(torch.from_numpy(g))
        torch.cuda.synchronize()
        dist.barrier()
        diverged = False
        try:
            srv.run([float(i + 1) for i in range(n_steps)])
        except ps.DivergenceError:
            diverged = True
        gs = [oracle.synthetic_update(9, p, 0, d) for p in range(world)]
        for p in range(world):
            gs[p][13] = -2.0e37 if p == 0 else 0.0
        w = w0.astype(np.float32)
        ok_steps = 0
        while ok_steps < n_steps:
            nxt = w
            for p in range(world):
                nxt = oracle.apply_f32(nxt, gs[p], 0.5)
            if not np.all(np.isfinite(nxt)):
                break
            w = nxt
            ok_steps += 1
        verdict["checks"].append({
            "run": f"diverge_at_{ok_steps}_of_{n_steps}", "d": d,
            "trace": diverged == (ok_steps < n_steps),
            "shard": bool(np.array_equal(srv.read_shard().view(np.uint32), w[srv.lo:srv.hi].view(np.uint32))),
            "replica": True, "version": int(srv.state().version), "steps": ok_steps})
        torch.cuda.synchronize()
        dist.barrier()
        srv.close()
    with open(os.path.join(out_dir, f"rank{rank}.json"), "w") as fh:
        json.dump(verdict, fh)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1])
