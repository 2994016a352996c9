"""One small device run (for ncu source-level profiling of the control warp)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1908_11848_b200 as ps
from bench import c2_config, synthetic_host

d = int(sys.argv[1]) if len(sys.argv) > 1 else 16
ctas = int(sys.argv[2]) if len(sys.argv) > 2 else 1
synth = torch.from_numpy(synthetic_host(4, 2, d)).cuda()
sim = ps.DeviceSimulation(c2_config("dssp", 3, 12), dimension=d, grad="synthetic")
sim.set_synthetic(synth, 2)
for _ in range(4):
    r = sim.run(read_weights=False, reset_gate=True, data_ctas=ctas)
print("ms", r.device_ms, "control", r.control_ms)
