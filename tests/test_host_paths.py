"""CPU checks of host-side logic around the engine: the server-call sequence
derived from a trace equals the reference's recorded boundary calls, and the
PyTorch worker flattening keeps parameters and gradients as views."""

import oracle
from paper_1908_11848_b200.sim import calls_from_trace
from paper_1908_11848_b200.trace import TraceEntry


def _entries(text):
    out = []
    for line in text.splitlines():
        t, w, kind, c, dec = line.split("\t")
        out.append(TraceEntry(float(t), int(w), kind, int(c), dec))
    return out


def test_calls_from_trace_equal_recorded_boundary_calls():
    runs = oracle.load_golden("sim_corpus.json.gz")["runs"] + \
        oracle.load_golden("c2_schedule.json.gz")["runs"]
    for run in runs:
        want = []
        for c in run["calls"]:
            if c[0] == "pull":
                want.append(("pull", c[1]))
            elif c[0] == "apply":
                want.append(("apply", c[1]))
            elif c[0] == "decide":
                want.append(("decide", c[1], c[2]))
        assert calls_from_trace(_entries(run["trace"])) == want, run["name"]


def test_flatten_makes_views():
    import torch
    from paper_1908_11848_b200.workers import CifarResNet, flatten_
    model = CifarResNet(20)
    flat_p, flat_g, n = flatten_(model, device="cpu")
    assert n == 272_474 and flat_p.numel() % 4 == 0
    flat_p[:n] = torch.arange(n, dtype=torch.float32)
    off = 0
    for p in model.parameters():
        k = p.numel()
        assert p.data.data_ptr() == flat_p[off:off + k].data_ptr()
        assert p.grad.data_ptr() == flat_g[off:off + k].data_ptr()
        assert float(p.data.reshape(-1)[0]) == float(off)
        off += k
