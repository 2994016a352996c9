"""NVLink traffic of the engine's P2P kernels, measurable under ncu in ONE
process: the server on cuda:0, one free-running worker on cuda:1 whose push
kernel applies its update to the server's weights over NVLink (reads w,
writes w': 8 B/param over the link + 4 B/param local gradient reads) and
whose pull kernel copies the weights back over NVLink (4 B/param).
A single worker takes every ticket in stream order, so ncu's serialized
replay cannot deadlock it. Usage: python tools/nvlink_probe.py [d] [iters]
(without ncu: per-iteration wall time of the steady state, after 3 warm-up
iterations)"""
import os, sys
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1908_11848_b200.engine import Engine
from paper_1908_11848_b200.freerun import FreeRunningCluster
from paper_1908_11848_b200.workers import SyntheticWorker

d = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 24
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
dpad = (d + 3) // 4 * 4
ring = torch.randn(1, dpad, device="cuda:1") * 1e-3
eng = Engine("asp", 1, 0, 0, 0.05, d, device=0)
cl = FreeRunningCluster(eng, [SyntheticWorker(ring, device="cuda:1")], graphs=False)
cl.run(3)  # first launches (module loading, peer mappings) out of the timing
rep = cl.run(iters)
print(f"d={d} pushes={rep.pushes} wall_ms={rep.wall_s * 1e3:.3f} "
      f"per_iter_us={rep.wall_s * 1e6 / iters:.1f} link_bytes_per_iter={12 * d} "
      f"link_GBps={12 * d * iters / rep.wall_s / 1e9:.1f}")
