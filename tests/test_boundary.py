"""CPU checks of the drop-in boundary: the C-ABI library loads and exports
every entry point include/dssp_ps.h declares; the host-side mirror of the
reference interface behaves like the reference without touching a GPU."""

import ctypes
import os

import numpy as np
import pytest

import oracle
from paper_1908_11848_b200 import _lib, config as pcfg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    assert os.path.exists(_lib.LIB_PATH), "run __graft_entry__.build() first"
    lib = ctypes.CDLL(_lib.LIB_PATH)
    declared = _lib.declared_symbols()
    assert len(declared) >= 18
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    assert set(declared) <= set(_lib.SIGNATURES), "binding table lags the header"


def test_ctypes_struct_layouts_match_header():
    assert ctypes.sizeof(_lib.PSConfig) == 4 * 4 + 8 + 8 + 4 + 28
    assert ctypes.sizeof(_lib.PSGateState) == 24 + 64 * 8 * 5 + 8 * 4
    assert ctypes.sizeof(_lib.PSTraceRow) == 40


def test_engine_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(_lib.EngineUnavailable):
        _lib.load(require_gpu=True)


def test_validate_config_matches_reference_normalization():
    for run in oracle.load_golden("sim_corpus.json.gz")["runs"]:
        cfg = pcfg.validate_config(pcfg.make_config(**run["config"]))
        norm = run["normalized"]
        assert cfg.paradigm == norm["paradigm"]
        assert (cfg.staleness.s_lower, cfg.staleness.r_max) == (norm["s_lower"], norm["r_max"])
        assert cfg.dataset_size == norm["dataset_size"]


def test_compute_time_table_reproduces_reference_schedule():
    """Every COMPUTE_DONE in a reference trace happens exactly at the
    preceding PULL_RETURN plus the k-th draw of our precomputed table."""
    for run in oracle.load_golden("sim_corpus.json.gz")["runs"]:
        cfg = pcfg.validate_config(pcfg.make_config(**run["config"]))
        budget = pcfg.push_budget(cfg)
        table = pcfg.compute_time_table(cfg, budget)
        last_return = {}
        k = {}
        for line in run["trace"].splitlines():
            t, w, kind, _, _ = line.split("\t")
            t, w = float(t), int(w)
            if kind == "pull_return":
                last_return[w] = t
            elif kind == "compute_done":
                i = k.get(w, 0)
                assert t == last_return[w] + table[w, i], (run["name"], w, i)
                k[w] = i + 1


def test_initial_weights_and_center_match_reference_streams():
    data = oracle.load_golden("apply_vectors.json")
    for seed, values in data["initial_weights_16"].items():
        cfg = pcfg.make_config(seed=int(seed))
        assert np.array_equal(pcfg.initial_weights_f64(cfg, 16), np.array(values))


def test_trace_rendering_matches_reference_format():
    from paper_1908_11848_b200.trace import TraceEntry, format_trace
    run = oracle.load_golden("sim_corpus.json.gz")["runs"][0]
    entries = []
    for line in run["trace"].splitlines():
        t, w, kind, c, dec = line.split("\t")
        entries.append(TraceEntry(float(t), int(w), kind, int(c), dec))
    assert format_trace(entries) == run["trace"]
