"""Per-call latency of the reference-facing path (C-ABI and drop-in)."""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1908_11848_b200 as ps
from paper_1908_11848_b200 import _lib

d = int(sys.argv[1]) if len(sys.argv) > 1 else 272_474
N = 300
cfg = ps.validate_config(ps.make_config(paradigm="asp", worker_count=4, dimension=d, learning_rate=0.05))
server = ps.ParameterServer(cfg, d)
eng = server.engine
lib = eng.lib
h = eng.handle
g_pin = torch.randn(d).pin_memory()
g_np = g_pin.numpy()
g_page = np.array(g_np)
out_pin = torch.empty(d).pin_memory().numpy()
out_page = np.empty(d, dtype=np.float32)
applied = ctypes.c_int32()
granted = ctypes.c_int32()
rel = ctypes.c_uint64()
ver = ctypes.c_int64()


def t(label, fn):
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(N):
        fn()
    dt = (time.perf_counter() - t0) / N * 1e6
    print(f"{label:40s} {dt:8.1f} us")


t("ps_apply pinned f32", lambda: lib.ps_apply(h, 0, g_np.ctypes.data, 0, 0, ctypes.byref(applied)))
t("ps_apply pageable f32", lambda: lib.ps_apply(h, 0, g_page.ctypes.data, 0, 0, ctypes.byref(applied)))
t("ps_decide", lambda: lib.ps_decide(h, 0, 1.0, ctypes.byref(granted), ctypes.byref(rel)))
t("ps_push pinned", lambda: lib.ps_push(h, 0, g_np.ctypes.data, 0, 0, 1.0, ctypes.byref(applied),
                                         ctypes.byref(granted), ctypes.byref(rel)))
t("ps_read_weights -> pinned", lambda: lib.ps_read_weights(h, out_pin.ctypes.data, 0, 0, ctypes.byref(ver)))
t("ps_read_weights -> pageable", lambda: lib.ps_read_weights(h, out_page.ctypes.data, 0, 0, ctypes.byref(ver)))
gv = ps.GradientVector(g_np, 0, 0)
t("drop-in apply_gradient", lambda: server.apply_gradient(gv))
t("drop-in decide_push", lambda: server.decide_push(0, 1.0))
t("drop-in handle_push", lambda: server.handle_push(gv, 1.0))
t("drop-in handle_pull(out=pinned)", lambda: server.handle_pull(1, out=out_pin))
t("drop-in handle_pull()", lambda: server.handle_pull(1))
dev = torch.empty(d, device="cuda")
t("torch H2D pinned copy", lambda: (dev.copy_(g_pin, non_blocking=True), torch.cuda.synchronize()))
