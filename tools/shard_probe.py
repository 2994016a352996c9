"""Per-kernel timing of the sharded step (run under torchrun)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, torch.distributed as dist
from paper_1908_11848_b200.sharded import ShardedServer, c3_config, homogeneous_push_times, max_over_ranks, C3_DIM

rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
d = int(sys.argv[1]) if len(sys.argv) > 1 else C3_DIM
srv = ShardedServer(c3_config("asp", 0, 0, world), d, rank, world, local)
srv.update[:d].normal_()
times = homogeneous_push_times(1.0, 0.05, 100)
srv.run(times[:5])
dist.barrier()
ms = srv.run(times[5:25])
ms = max_over_ranks(ms)
srv.lib.ps_shard_set_profiling(srv._h, 1)
dist.barrier()
srv.run(times[25:45])
ph = (ctypes.c_double * 3)()
srv.lib.ps_shard_phase_ms(srv._h, ph)
if rank == 0:
    print(f"world={world} d={d} step_ms={ms/20:.4f} profiled apply_kernel={ph[0]/20:.4f} then_wait_pull={ph[1]/20:.4f}")
dist.barrier()
srv.close()
dist.destroy_process_group()
