"""NVLink byte counters of the sharded step's streaming pass (one-sided: rank
0 runs ps_shard_stream_probe while the other ranks idle), for a
multi-process ncu capture that needs no cross-GPU flags:
  ncu --target-processes all --metrics nvlrx__bytes.sum,nvltx__bytes.sum,...
      -k regex:k_shard_stream_probe python -m torch.distributed.run ... this
Each probe launch = one step's worth of this owner's traffic: (G-1) update
slices in over NVLink, the new slice out to G-1 replicas."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist
from paper_1908_11848_b200.sharded import ShardedServer, c3_config, C3_DIM, shard_range
rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("gloo")
d = C3_DIM
srv = ShardedServer(c3_config("asp", 0, 0, world), d, rank, world, local)
srv.update[:d].normal_()
torch.cuda.synchronize()
dist.barrier()
if rank == 0:
    ms = ctypes.c_double(0)
    for _ in range(3):
        srv._check(srv.lib.ps_shard_stream_probe(srv._h, 1, ctypes.byref(ms)))
    lo, hi = shard_range(d, world, rank)
    S = hi - lo
    print(f"G={world} probe_ms={ms.value:.4f} algorithmic per step: in {(world-1)*S*4} B (update slices), "
          f"out {(world-1)*S*4} B (replica slices); {2*(world-1)*S*4/(ms.value*1e-3)/1e9:.0f} GB/s one-sided",
          flush=True)
dist.barrier()
srv.close()
dist.destroy_process_group()
