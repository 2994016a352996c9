"""Event-trace rows in the reference's TSV format (trace.py:1-72).

``time<TAB>worker<TAB>kind<TAB>t_p<TAB>decision``: time printed with repr so
it round-trips, ``decision`` is ``grant``, ``defer``, ``grant[i,j]`` or ``-``.
The device loop writes fixed-size rows (ps_trace_row); this module renders
them byte-identically to ``stalesync.trace.format_trace``.
"""

from __future__ import annotations

from dataclasses import dataclass

from ._lib import EVENT_KINDS

COMPUTE_DONE, PUSH_ARRIVE, GRANT_DELIVER, PULL_ARRIVE, PULL_RETURN = EVENT_KINDS


@dataclass(frozen=True)
class TraceEntry:
    time: float
    worker: int
    kind: str
    count: int
    decision: str = "-"

    def render(self) -> str:
        return f"{self.time!r}\t{self.worker}\t{self.kind}\t{self.count}\t{self.decision}"


def decision_token(granted: bool, released=()) -> str:
    if not granted:
        return "defer"
    if released:
        return "grant[" + ",".join(str(w) for w in released) + "]"
    return "grant"


def format_trace(entries) -> str:
    return "".join(entry.render() + "\n" for entry in entries)


def rows_to_entries(rows, n):
    out = []
    for i in range(n):
        r = rows[i]
        if r.decision < 0:
            token = "-"
        else:
            released = tuple(q for q in range(64) if (r.released >> q) & 1)
            token = decision_token(r.decision == 0, released)
        out.append(TraceEntry(float(r.time), int(r.worker), EVENT_KINDS[r.kind], int(r.count), token))
    return out
