"""Vectorised trace/summary CSV emission (paper_2601_14476_b200.traces) is
byte-identical to the reference CLI writers (cli.py:146-168), pinned by
golden files the reference itself wrote (tests/golden/make_trace_golden.py)."""

from __future__ import annotations

import csv
import io
from types import SimpleNamespace

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2601_14476_b200 import traces


def _restated(results) -> bytes:
    """Row-by-row restatement of cli._trace_rows + cli._write_csv."""
    fh = io.StringIO(newline="")
    w = csv.writer(fh, lineterminator="\n")
    w.writerow(traces.TRACE_COLUMNS)
    for t, r in enumerate(results):
        for c in range(r.i0_trace.size):
            cut = None if r.cut_trace is None else int(r.cut_trace[c])
            w.writerow([traces.fmt(x) for x in (t, c, float(r.i0_trace[c]),
                                                float(r.energy_trace[c]), cut)])
    return fh.getvalue().encode()


def test_synthetic_traces_match_reference_golden():
    z = np.load(GOLDEN / "traces.npz")
    res = []
    for k in range(5):
        cut = z[f"s{k}_cut"]
        res.append(SimpleNamespace(i0_trace=z[f"s{k}_i0"], energy_trace=z[f"s{k}_e"],
                                   cut_trace=None if cut.size == 0 else cut.astype(np.int64)))
    want = (GOLDEN / "trace_synth.csv").read_bytes()
    assert traces.trace_csv_bytes(res) == want
    assert _restated(res) == want


def test_random_traces_match_row_by_row_restatement():
    rng = np.random.default_rng(3)
    res = []
    for k in range(40):
        C = int(rng.integers(1, 60))
        i0 = np.exp(rng.uniform(-8, 4, C))
        kind = k % 4
        if kind == 0:
            e = -np.round(rng.uniform(0, 1e6, C))
        elif kind == 1:
            e = rng.standard_normal(C) * 10.0 ** rng.integers(-5, 18, C)
        elif kind == 2:
            e = np.round(rng.uniform(-1e17, 1e17, C))
        else:
            e = rng.choice([0.0, -0.0, 1e16, 9999999999999998.0, -1e16, 5e-324, np.inf], C)
        cut = None if k % 5 == 0 else rng.integers(-2 ** 62, 2 ** 62, C)
        res.append(SimpleNamespace(i0_trace=i0, energy_trace=e, cut_trace=cut))
    assert traces.trace_csv_bytes(res) == _restated(res)
    assert traces.trace_csv_bytes([]) == b"trial,cycle,i0,energy,cut\n"


def test_summary_row_format_matches_reference_golden():
    want = (GOLDEN / "summary_g1.csv").read_text().splitlines()
    fields = next(csv.reader([want[1]]))
    spec = SimpleNamespace(graph="G1", algo=SimpleNamespace(kind=SimpleNamespace(value="psa")),
                           variability=SimpleNamespace(sigma_lambda=0.0, sigma_delta=0.0,
                                                       sigma_nu=0.5),
                           cycles=30, trials=6, base_seed=0)
    summ = SimpleNamespace(mean_cut=float(fields[8]), std_cut=float(fields[9]),
                           normalized_mean_cut=float(fields[10]),
                           mean_final_energy=float(fields[11]), anneal_seconds=float(fields[12]))
    got = traces.summary_csv_bytes([traces.summary_row(spec, summ)]).decode().splitlines()
    assert got == want


@pytest.mark.gpu
def test_gpu_run_reproduces_the_reference_trace_csv(tmp_path):
    """End to end: this package's run_trials on the device, then the vectorised
    writer, gives the reference CLI's --trace-out file byte for byte; the
    summary row equals the reference's except the wall-clock column."""
    from paper_2601_14476_b200 import benchmarks, engine
    from paper_2601_14476_b200.annealer import Algorithm, AlgorithmConfig
    from paper_2601_14476_b200.pbit import VariabilityConfig
    graph, _ = benchmarks.load("G1")
    spec = engine.ExperimentSpec(graph="G1", algo=AlgorithmConfig(Algorithm.PSA),
                                 variability=VariabilityConfig(0.0, 0.0, 0.5), cycles=30, trials=6)
    summary = engine.run_trials(spec, {"G1": graph}, {"G1": 11605})
    traces.write_trace_csv(str(tmp_path / "t.csv"), summary.results)
    assert (tmp_path / "t.csv").read_bytes() == (GOLDEN / "trace_g1.csv").read_bytes()
    traces.write_summary_csv(str(tmp_path / "s.csv"), spec, summary)
    got = (tmp_path / "s.csv").read_text().splitlines()
    want = (GOLDEN / "summary_g1.csv").read_text().splitlines()
    assert got[0] == want[0]
    assert got[1].rsplit(",", 1)[0] == want[1].rsplit(",", 1)[0]


def test_native_formatter_equals_numpy_path(monkeypatch):
    """pbsa_format_trace_csv (library host code) and the numpy path give the
    same bytes on a batch-shaped input (shared i0, integral energies)."""
    rng = np.random.default_rng(8)
    C = 37
    i0 = np.exp(rng.uniform(-6, 3, C))
    res = [SimpleNamespace(i0_trace=i0, energy_trace=-np.round(rng.uniform(-5e4, 9e15, C)),
                           cut_trace=rng.integers(-5, 2 ** 50, C)) for _ in range(23)]
    fast = traces._native_rows(res)
    assert fast is not None
    assert b"trial,cycle,i0,energy,cut\n" + fast == _restated(res)
    monkeypatch.setattr(traces, "_native_rows", lambda r: None)
    assert traces.trace_csv_bytes(res) == _restated(res)
    nocut = [SimpleNamespace(i0_trace=i0, energy_trace=r.energy_trace, cut_trace=None) for r in res]
    assert traces.trace_csv_bytes(nocut) == _restated(nocut)
