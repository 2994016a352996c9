"""A few push-apply (+pull) launches at one size, for ncu captures."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1908_11848_b200 as ps

mb = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
d = mb * (1 << 20) // 4
eng = ps.engine.Engine("asp", 1, 0, 0, 0.05, d)
eng.set_profiling(True)
g = torch.randn(d, device="cuda")
dst = torch.empty(d, device="cuda")
for _ in range(5):
    eng.apply(0, g)
    eng.read(out=dst)
print("apply ms", eng.last_kernel_ms())
