"""Timing of the sharded C3 step alone (torchrun, one rank per GPU; or plain
python for G = 1): warm-up run, then 20 timed steps in one launch; prints the
max-over-ranks ms per step and the NVLink / HBM figure of merit."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29771")
os.environ.setdefault("RANK", "0")
os.environ.setdefault("WORLD_SIZE", "1")
os.environ.setdefault("LOCAL_RANK", "0")
import torch, torch.distributed as dist
from paper_1908_11848_b200.sharded import (ShardedServer, c3_config, homogeneous_push_times, C3_DIM,
                                           max_over_ranks, shard_range)
rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
d = C3_DIM
srv = ShardedServer(c3_config("dssp", 3, 12, world), d, rank, world, local)
srv.update[:d].normal_()
times = homogeneous_push_times(1.0, 0.05, 64)
srv.run(times[:5])
dist.barrier(); torch.cuda.synchronize()
ms = max_over_ranks(srv.run(times[5:25])) / 20
lo, hi = shard_range(d, world, rank)
if rank == 0:
    tag = os.environ.get("TAG", "")
    if world == 1:
        print(f"{tag} G=1 step_us={ms*1e3:.1f} hbm_gbs={16*d/(ms*1e-3)/1e9:.0f}")
    else:
        print(f"{tag} G={world} step_us={ms*1e3:.1f} nvlink_gbs={2*(world-1)*(hi-lo)*4/(ms*1e-3)/1e9:.0f}")
dist.barrier(); torch.cuda.synchronize()
srv.close()
dist.destroy_process_group()
