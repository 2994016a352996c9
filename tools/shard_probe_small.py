"""A short sharded run for a multi-process ncu capture of the NVLink byte
counters of k_shard_run (torchrun, one rank per GPU, a few metrics only)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist
from paper_1908_11848_b200.sharded import ShardedServer, c3_config, homogeneous_push_times, C3_DIM
rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("gloo")
d = int(sys.argv[1]) if len(sys.argv) > 1 else C3_DIM
srv = ShardedServer(c3_config("asp", 0, 0, world), d, rank, world, local)
srv.update[:d].normal_()
times = homogeneous_push_times(1.0, 0.05, 8)
dist.barrier()
ms = srv.run(times[:4])
print(f"rank {rank} d={d} step_ms={ms / 4:.4f}", flush=True)
dist.barrier()
srv.close()
dist.destroy_process_group()
