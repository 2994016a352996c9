"""configs[4] small end: push-apply / pull device time at 1-64 MB through the
Engine's profiling events (the bench's apply_sweep), for A/B of apply knobs."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_1908_11848_b200 as ps
hbm, _ = bench.peaks()
rows = bench.apply_sweep(torch, ps, hbm)
for r in rows[:4]:
    print(os.environ.get("PS_APPLY_SMALL_U", "1"), json.dumps(r))
