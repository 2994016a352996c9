"""CPU checks of host-side logic around the engine: the server-call sequence
derived from a trace equals the reference's recorded boundary calls, and the
PyTorch worker flattening keeps parameters and gradients as views."""

import os

import oracle
from paper_1908_11848_b200.sim import calls_from_trace

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
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


def test_decision_words_decode_like_the_reference_tokens():
    """ps_replay_decisions words ((released << 8) | outcome) decode into the
    reference's SyncDecision shape (policy.py:33-40): outcome, released ids
    ascending."""
    from paper_1908_11848_b200.sim import decode_decisions
    words = [0, 1, (0b1011 << 8) | 0, (1 << 54) << 8]
    assert decode_decisions(words) == [("grant", ()), ("defer", ()), ("grant", (0, 1, 3)),
                                       ("grant", (54,))]


def test_replay_call_array_layout_matches_the_c_abi():
    """DeviceReplay packs calls as ps_replay_call {double now; int32 kind;
    int32 worker} (include/dssp_ps.h)."""
    import ctypes
    from paper_1908_11848_b200 import sim
    assert sim._CALL_DTYPE.itemsize == 16
    assert [sim._CALL_DTYPE.fields[k][1] for k in ("now", "kind", "worker")] == [0, 8, 12]
    assert (sim.CALL_PULL, sim.CALL_APPLY, sim.CALL_DECIDE) == (0, 1, 2)
    header = open(os.path.join(ROOT, "include", "dssp_ps.h")).read()
    for name in ("PS_CALL_PULL", "PS_CALL_APPLY", "PS_CALL_DECIDE"):
        assert name in header
    assert ctypes.sizeof(ctypes.c_double) + 2 * ctypes.sizeof(ctypes.c_int32) == 16


def test_groups_from_trace_partition_pushes_and_pulls():
    """groups_from_trace (the sharded server's schedule input) covers every
    push once, in trace order, groups same-instant pushes exactly like
    calls_from_trace, and gives every pull after the first group a home."""
    from paper_1908_11848_b200.sharded import groups_from_trace
    for run in oracle.load_golden("sim_corpus.json.gz")["runs"][:40]:
        entries = _entries(run["trace"])
        groups = groups_from_trace(entries)
        pushes = [(e.time, e.worker) for e in entries if e.kind == "push_arrive"]
        assert [(t, w) for t, order, _ in groups for w in order] == pushes
        calls = calls_from_trace(entries)
        decide_groups, cur = [], []
        for c in calls:
            if c[0] == "apply":
                cur.append(c[1])
            elif c[0] == "decide" and cur:
                decide_groups.append(cur)
                cur = []
        assert [order for _, order, _ in groups] == decide_groups
        first = next(i for i, e in enumerate(entries) if e.kind == "push_arrive")
        late_pulls = sum(1 for e in entries[first:] if e.kind == "pull_arrive")
        assert sum(len(p) for _, _, p in groups) == late_pulls
