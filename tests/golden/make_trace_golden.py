"""Golden CSV files from the REFERENCE CLI writers (cli.py:146-168).

Run in the build container (the only place /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/nc PYTHONPATH=/root/reference/pkg/src \\
        python tests/golden/make_trace_golden.py

Writes tests/golden/traces.npz (the inputs) and the reference's bytes:
  trace_synth.csv   cli._write_csv(TRACE_COLUMNS, cli._trace_rows(...)) of
                    synthetic traces with the awkward values (fractions,
                    -0.0, 1e16, no graph, huge ints)
  trace_g1.csv      the same for the reference's own run_trials on a small
                    G1 spec (pSA, sigma_nu = 0.5, 6 trials x 30 cycles);
                    this repository's GPU run must reproduce it byte for byte
  summary_g1.csv    cli._summary_row of that run (anneal_seconds excluded
                    from comparison: it is a wall time)
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF_TESTS = Path("/root/reference/pkg/tests")
sys.path.insert(0, str(REF_TESTS))

from pbitsa import cli  # noqa: E402
from pbitsa.annealer import Algorithm, AlgorithmConfig  # noqa: E402
from pbitsa.engine import ExperimentSpec, run_trials  # noqa: E402
from pbitsa.pbit import VariabilityConfig  # noqa: E402

import analogs  # noqa: E402

OUT = Path(__file__).resolve().parent


class _R:
    def __init__(self, i0, e, cut):
        self.i0_trace, self.energy_trace, self.cut_trace = i0, e, cut

    @property
    def trace(self):
        from pbitsa.annealer import TraceRecord
        return [TraceRecord(c, float(self.i0_trace[c]), float(self.energy_trace[c]),
                            None if self.cut_trace is None else int(self.cut_trace[c]))
                for c in range(self.i0_trace.size)]


class _S:
    def __init__(self, results):
        self.results = results


def main() -> None:
    rng = np.random.default_rng(7)
    C = 25
    i0 = 0.01 * (1.0 / 0.9) ** np.arange(C)
    synth = []
    arrays = {}
    for k in range(5):
        e = -np.round(rng.uniform(0, 5e4, C))
        if k == 1:
            e = rng.standard_normal(C) * 1e3          # fractional energies
        if k == 2:
            e[:4] = [-0.0, 0.0, 1e16, -2.5e17]        # repr edge cases
        cut = rng.integers(0, 2 ** 40, C) if k != 3 else None
        synth.append(_R(i0 if k != 4 else i0 * 1.5, e, cut))
        arrays[f"s{k}_i0"], arrays[f"s{k}_e"] = synth[-1].i0_trace, e
        arrays[f"s{k}_cut"] = np.array([]) if cut is None else cut
    cli._write_csv(str(OUT / "trace_synth.csv"), cli.TRACE_COLUMNS, cli._trace_rows(_S(synth)))

    from pbitsa.gset import to_graph
    graph = to_graph(analogs.make_analog("G1"))
    spec = ExperimentSpec(graph="G1", algo=AlgorithmConfig(Algorithm.PSA),
                          variability=VariabilityConfig(0.0, 0.0, 0.5), cycles=30, trials=6)
    summary = run_trials(spec, {"G1": graph}, {"G1": 11605})
    cli._write_csv(str(OUT / "trace_g1.csv"), cli.TRACE_COLUMNS, cli._trace_rows(summary))
    cli._write_csv(str(OUT / "summary_g1.csv"), cli.SUMMARY_COLUMNS, [cli._summary_row(spec, summary)])
    np.savez_compressed(OUT / "traces.npz", **arrays)
    print("wrote", sorted(p.name for p in OUT.glob("*.csv")))


if __name__ == "__main__":
    main()
