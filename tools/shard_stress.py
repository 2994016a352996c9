"""Stress the sharded server's pull path: many short-lived servers, each run
checked bit for bit against the fp32 replay; on a mismatch, re-read the
replica after a pause to tell late-landing writes from lost ones.
Run under torchrun (G >= 2)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist

import oracle
import paper_1908_11848_b200 as ps
from paper_1908_11848_b200.sharded import ShardedServer

rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 100
sizes = [5, 100_003, 4099, 100_003, 1 << 20, 100_003]
cache = {}
bad = 0
for it in range(iters):
    d = sizes[it % len(sizes)]
    if d not in cache:
        gs = [oracle.synthetic_update(9, p, 0, d) for p in range(world)]
        w0 = oracle.initial_weights_f64(5, d)
        w = w0.astype(np.float32)
        for _ in range(2):
            for p in range(world):
                w = oracle.apply_f32(w, gs[p], 0.05)
        cache[d] = (gs, w0, w)
    gs, w0, want = cache[d]
    cfg = ps.validate_config(ps.make_config(paradigm="asp", worker_count=world, dimension=d,
                                            learning_rate=0.05, seed=5))
    srv = ShardedServer(cfg, d, rank, world, local, w0_host=w0)
    srv.update[:d].copy_(torch.from_numpy(gs[rank]))
    torch.cuda.synchronize()
    dist.barrier()
    srv.run([1.0, 2.0])
    rep = srv.read_replica()
    if not np.array_equal(rep.view(np.uint32), want.view(np.uint32)):
        idx = np.nonzero(rep.view(np.uint32) != want.view(np.uint32))[0]
        time.sleep(0.5)
        rep2 = srv.read_replica()
        later = int(np.count_nonzero(rep2.view(np.uint32) != want.view(np.uint32)))
        bad += 1
        print(f"[rank {rank}] iter {it} d={d}: {idx.size} mismatches at {idx[0]}..{idx[-1]} "
              f"(shard {srv.lo}..{srv.hi}); after 0.5 s: {later}; got {rep[idx[0]]} want {want[idx[0]]} "
              f"w0 {w0[idx[0]]:.6f}", flush=True)
    torch.cuda.synchronize()
    dist.barrier()
    srv.close()
t = torch.tensor([bad], device="cuda")
dist.all_reduce(t)
if rank == 0:
    print(f"stress: {iters} servers x {world} ranks, {int(t.item())} replica mismatches", flush=True)
dist.destroy_process_group()
