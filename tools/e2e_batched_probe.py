"""Where the time of one e2e_batched step goes (host view, perf_counter)."""
import os, sys, time, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle
from paper_1908_11848_b200.engine import Engine
from paper_1908_11848_b200.sim import DeviceReplay
from bench import synthetic_host, reference_calls, C2_DIM

d = C2_DIM
calls, _ = reference_calls("dssp")
synth_host = synthetic_host(4, 2, d)
eng = Engine("dssp", 4, 3, 12, 0.05, d, w0=oracle.initial_weights_f64(0, d))
pinned = torch.from_numpy(np.ascontiguousarray(synth_host)).pin_memory()
dev = torch.empty(pinned.shape, dtype=torch.float32, device="cuda")
out_w = torch.empty(d, dtype=torch.float32).pin_memory().numpy()
rp = DeviceReplay(eng, calls, dev, 2)
T = {"h2d": [], "run": [], "read": [], "total": []}
for it in range(30):
    t0 = time.perf_counter()
    dev.copy_(pinned, non_blocking=True)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    r = rp.run(decisions=True)
    t2 = time.perf_counter()
    eng.read(out=out_w)
    t3 = time.perf_counter()
    if it >= 5:
        T["h2d"].append(t1 - t0); T["run"].append(t2 - t1); T["read"].append(t3 - t2); T["total"].append(t3 - t0)
        T.setdefault("kernel", []).append(r.device_ms * 1e-3)
for k, v in T.items():
    print(f"{k:8s} median {statistics.median(v)*1e3:.3f} ms  min {min(v)*1e3:.3f}  max {max(v)*1e3:.3f}")
