"""A few device replays of the C2 DSSP request stream (for ncu captures)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import oracle
from paper_1908_11848_b200.engine import Engine
from paper_1908_11848_b200.sim import DeviceReplay
from bench import synthetic_host, reference_calls, C2_DIM

d = C2_DIM
calls, _ = reference_calls("dssp")
eng = Engine("dssp", 4, 3, 12, 0.05, d, w0=oracle.initial_weights_f64(0, d))
rp = DeviceReplay(eng, calls, torch.from_numpy(synthetic_host(4, 2, d)).cuda(), 2)
for _ in range(5):
    r = rp.run(decisions=False)
print("ms", r.device_ms)
