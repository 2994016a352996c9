"""Timing probe of the device run loop: control vs data critical path."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1908_11848_b200 as ps
from bench import c2_config, synthetic_host, C2_DIM

d = int(sys.argv[1]) if len(sys.argv) > 1 else C2_DIM
synth = torch.from_numpy(synthetic_host(4, 2, d)).cuda()
for name, s, r in (("dssp", 3, 12), ("asp", 0, 0)):
    cfg = c2_config(name, s, r)
    for ctas in (0, 74, 37, 16):
        sim = ps.DeviceSimulation(cfg, dimension=d, grad="synthetic")
        sim.set_synthetic(synth, 2)
        for _ in range(3):
            sim.run(read_weights=False, reset_gate=True)
        rs = [sim.run(read_weights=False, reset_gate=True, data_ctas=ctas) for _ in range(5)]
        print(json.dumps({"paradigm": name, "d": d, "ctas": ctas,
                          "ms": round(float(np.median([x.device_ms for x in rs])), 3),
                          "control_ms": round(float(np.median([x.control_ms for x in rs])), 3),
                          "data_ms": round(float(np.median([x.data_ms for x in rs])), 3)}))
        sim.engine.close()
