"""Where the replay's time goes: the C2 DSSP request stream vs the same
stream with only its decides (pure gate) and only its pulls/applies (pure
data side + op emission)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import statistics
import torch
import oracle
from paper_1908_11848_b200.engine import Engine
from paper_1908_11848_b200.sim import DeviceReplay
from bench import synthetic_host, reference_calls, C2_DIM

d = int(sys.argv[1]) if len(sys.argv) > 1 else C2_DIM
calls, _ = reference_calls("dssp")
synth = torch.from_numpy(synthetic_host(4, 2, d)).cuda()
variants = {
    "full": calls,
    "decides_only": [c for c in calls if c[0] == "decide"],
    "pull_apply_only": [c for c in calls if c[0] != "decide"],
    "apply_only": [c for c in calls if c[0] == "apply"],
    "pull_only": [c for c in calls if c[0] == "pull"],
}
for name, cs in variants.items():
    eng = Engine("dssp", 4, 3, 12, 0.05, d, w0=oracle.initial_weights_f64(0, d))
    rp = DeviceReplay(eng, cs, synth, 2)
    ts = []
    for _ in range(7):
        r = rp.run(decisions=False)
        ts.append(r.device_ms)
    print(f"d={d} {name:16s} calls={len(cs):5d} median_ms={statistics.median(ts[2:]):.3f} "
          f"us_per_call={1e3 * statistics.median(ts[2:]) / len(cs):.3f}")
    eng.close()
