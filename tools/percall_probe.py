"""Per-call latency of the reference-shaped API (ParameterServer drop-in /
Engine per-op calls) at C2 size: device vs pinned-host gradients, device vs
host pulls, decide alone. Wall-clock per call, median of many."""
import os, sys, time, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1908_11848_b200.engine import Engine

d = int(sys.argv[1]) if len(sys.argv) > 1 else 272_474
eng = Engine("asp", 4, 0, 0, 0.05, d)
if int(os.environ.get("PS_RESIDENT", "0") or 0):
    eng.set_resident(int(os.environ["PS_RESIDENT"]))
g_dev = torch.randn(d, device="cuda") * 1e-3
g_host = torch.randn(d).mul_(1e-3).pin_memory().numpy()
out_dev = torch.empty(d, device="cuda")
out_host = torch.empty(d).pin_memory().numpy()
torch.cuda.synchronize()

def timeit(fn, n=400):
    for _ in range(20):
        fn()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return 1e6 * statistics.median(ts)

now = [0.0]
def push_dev():
    now[0] += 1.0
    eng.push(0, g_dev, now[0])
def push_host():
    now[0] += 1.0
    eng.push(0, g_host, now[0])
def apply_dev():
    eng.apply(0, g_dev)
def decide():
    now[0] += 1.0
    eng.decide(0, now[0])
def pull_dev():
    eng.read(out=out_dev, worker=0)
def pull_host():
    eng.read(out=out_host, worker=0)
for name, fn in (("push_dev", push_dev), ("push_host", push_host), ("apply_dev", apply_dev),
                 ("decide", decide), ("pull_dev", pull_dev), ("pull_host", pull_host)):
    print(f"{name:10s} {timeit(fn):8.2f} us")
