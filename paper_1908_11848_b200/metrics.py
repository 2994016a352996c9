"""Per-worker accounting from a device trace (the reference's summarize,
metrics.py:84-149, restricted to what the hot path produces).

A worker's time splits into compute (PULL_RETURN -> COMPUTE_DONE), wait (a
deferred push -> the granting push that releases it) and communication (the
rest). The staleness of an applied update is the frontier clock minus the
pusher's clock at its push (metrics.py:152-164).
"""

from __future__ import annotations

from dataclasses import dataclass


@dataclass
class WorkerTimes:
    iterations: int = 0
    wait_s: float = 0.0
    compute_s: float = 0.0
    comm_s: float = 0.0
    finish_s: float = 0.0


def per_worker(entries):
    ids = sorted({e.worker for e in entries})
    out = {w: WorkerTimes() for w in ids}
    last = {w: 0.0 for w in ids}
    deferred_at = {}
    released_at = {}
    for e in entries:
        w = out[e.worker]
        if e.kind == "push_arrive":
            if "[" in e.decision:
                inner = e.decision[e.decision.index("[") + 1:e.decision.index("]")]
                for tok in inner.split(","):
                    released_at[int(tok)] = e.time
            if e.decision == "defer":
                deferred_at[e.worker] = e.time
            w.iterations = e.count
        if e.kind == "compute_done":
            w.compute_s += e.time - last[e.worker]
        elif e.kind == "grant_deliver" and e.worker in deferred_at:
            rel = released_at.pop(e.worker)
            w.wait_s += rel - deferred_at.pop(e.worker)
            w.comm_s += e.time - rel
        else:
            w.comm_s += e.time - last[e.worker]
        last[e.worker] = e.time
        w.finish_s = e.time
    return out


def staleness_histogram(entries):
    counts = {}
    hist = {}
    for e in entries:
        if e.kind != "push_arrive":
            continue
        counts[e.worker] = e.count
        gap = max(counts.values()) - e.count
        hist[gap] = hist.get(gap, 0) + 1
    return hist
