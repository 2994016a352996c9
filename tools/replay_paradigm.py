"""Device replays of the C2 request stream of one paradigm (argv[1], default
dssp): device ms per stream; with the profiling build (DSSP_PS_LIB=
tools/libdssp_ps_prof.so) the gate warp prints its cycle accounting."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1908_11848_b200.config import initial_weights_f64
from paper_1908_11848_b200.engine import Engine
from paper_1908_11848_b200.sim import DeviceReplay
from bench import synthetic_host, reference_calls, c2_config, C2_DIM, PARADIGMS

name = sys.argv[1] if len(sys.argv) > 1 else "dssp"
s, r = {p: (a, b) for p, a, b in PARADIGMS}[name]
d = C2_DIM
calls, _ = reference_calls(name)
mode = sys.argv[2] if len(sys.argv) > 2 else "full"
if mode == "gate":      # decides only: the gate warp alone
    calls = [c for c in calls if c[0] == "decide"]
elif mode == "data":    # pulls and applies only: the data warps alone
    calls = [c for c in calls if c[0] != "decide"]
elif mode == "pulls":   # the pulls alone
    calls = [c for c in calls if c[0] == "pull"]
elif mode == "applies":  # the applies alone
    calls = [c for c in calls if c[0] == "apply"]
eng = Engine(name, 4, s, r, 0.05, d, w0=initial_weights_f64(c2_config(name, s, r), d))
rp = DeviceReplay(eng, calls, torch.from_numpy(synthetic_host(4, 2, d)).cuda(), 2)
ctas = int(sys.argv[3]) if len(sys.argv) > 3 else 0  # data CTAs (0: one per SM after the gate's)
for _ in range(3):
    rr = rp.run(decisions=False, data_ctas=ctas)
print(name, mode, "ctas", ctas, "device_ms", round(rr.device_ms, 4), "gate_ms", round(rr.control_ms, 4), "data_ms", round(rr.data_ms, 4),
      "decides", sum(1 for c in calls if c[0] == "decide"), "calls", len(calls))
