"""Throughput of the device replay (server serving the recorded C2 request stream)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle
from paper_1908_11848_b200.engine import Engine
from paper_1908_11848_b200.sim import DeviceReplay
from bench import synthetic_host, C2_DIM

d = int(sys.argv[1]) if len(sys.argv) > 1 else C2_DIM
synth = torch.from_numpy(synthetic_host(4, 2, d)).cuda()
for run in oracle.load_golden("c2_schedule.json.gz")["runs"]:
    norm = run["normalized"]
    calls = [tuple(c[:2]) if c[0] != "decide" else ("decide", c[1], c[2]) for c in run["calls"] if c[0] in ("pull", "apply", "decide")]
    eng = Engine(norm["paradigm"], 4, norm["s_lower"], norm["r_max"], 0.05, d, w0=oracle.initial_weights_f64(0, d))
    rp = DeviceReplay(eng, calls, synth, 2)
    for _ in range(3):
        rp.run(decisions=False)
    ms = [rp.run(decisions=False).device_ms for _ in range(5)]
    r = rp.run()
    ok = r.decisions == [(c[3], tuple(c[4])) for c in run["calls"] if c[0] == "decide"]
    print(json.dumps({"paradigm": norm["paradigm"], "d": d, "ms": round(float(np.median(ms)), 3),
                      "updates_per_s": round(r.applied / (np.median(ms) * 1e-3)), "decisions_match": ok}))
    eng.close()
