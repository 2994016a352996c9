"""The sharded step's kernel in one process (world = 1, gloo plumbing), for an
ncu capture of k_shard_run's streaming loop (ncu must not run multi-rank
commands). At G = 1 the step is local: read the update and the shard, write
the shard and the replica -- 16 B/param of HBM traffic, no NVLink."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29711")
import torch, torch.distributed as dist
from paper_1908_11848_b200.sharded import ShardedServer, c3_config, homogeneous_push_times, C3_DIM

dist.init_process_group("gloo", rank=0, world_size=1)
torch.cuda.set_device(0)
d = int(sys.argv[1]) if len(sys.argv) > 1 else C3_DIM
srv = ShardedServer(c3_config("asp", 0, 0, 1), d, 0, 1, 0)
srv.update[:d].normal_()
times = homogeneous_push_times(1.0, 0.05, 64)
for i in range(4):
    ms = srv.run(times[i * 8:(i + 1) * 8])
print(f"d={d} step_ms={ms / 8:.4f} -> {16 * d / (ms / 8 * 1e-3) / 1e9:.1f} GB/s (16 B/param)")
srv.close()
dist.destroy_process_group()
