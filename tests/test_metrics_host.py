"""The trace accounting (metrics.py) against the reference's own report
(summarize, metrics.py:84-149) stored with every golden simulator run."""

import oracle
from paper_1908_11848_b200.metrics import per_worker, staleness_histogram
from paper_1908_11848_b200.trace import TraceEntry


def _entries(text):
    out = []
    for line in text.splitlines():
        t, w, kind, c, dec = line.split("\t")
        out.append(TraceEntry(float(t), int(w), kind, int(c), dec))
    return out


def test_per_worker_times_match_reference_reports():
    for run in oracle.load_golden("sim_corpus.json.gz")["runs"]:
        got = per_worker(_entries(run["trace"]))
        for w, (iters, _epochs, wait, compute, comm) in run["per_worker"].items():
            g = got[int(w)]
            assert g.iterations == iters, run["name"]
            assert g.wait_s == wait and g.compute_s == compute and g.comm_s == comm, run["name"]


def test_staleness_histogram_totals():
    for run in oracle.load_golden("sim_corpus.json.gz")["runs"][:20]:
        hist = staleness_histogram(_entries(run["trace"]))
        assert sum(hist.values()) == run["updates_total"]
