"""Trace and summary CSV emission, vectorised.

The reference writes its per-cycle traces row by row: ``cli._trace_rows``
(/root/reference/pkg/src/pbitsa/cli.py:163-168) builds one list of ``_fmt``
strings per (trial, cycle) -- ``repr`` for floats, ``str`` for ints, "" for
None (cli.py:36-41) -- and ``csv.writer`` (cli.py:155-159) writes them with
"\\n" line ends.  For 4096 trials x 1000 cycles that is ~11 s of Python
(SURVEY §8(f)).  This module produces byte-identical files from whole arrays:

* integer columns (trial, cycle, cut) are rendered digit-by-digit with numpy
  into one byte buffer;
* ``i0`` is the same schedule for every trial of a batch, so each distinct
  i0 trace is ``repr``-ed once and its byte strings are reused;
* energies of MAX-CUT models are integral, and ``repr`` of an integral
  float with magnitude < 1e16 is its integer digits + ".0", so they take the
  integer path; any other value (fractions, -0.0, huge) falls back to
  ``repr`` for exactly those entries.

The common case (a batch: one i0 trace, integral energies) is formatted by
the CUDA library's host-side formatter ``pbsa_format_trace_csv`` on all host
threads (no GPU involved); the numpy path covers everything else.

``write_trace_csv`` / ``write_summary_csv`` mirror the reference CLI's
``--trace-out`` / ``--summary-out`` files (cli.py:190-197, 213-224).
"""

from __future__ import annotations

import csv
import io
from typing import Sequence

import numpy as np

SUMMARY_COLUMNS = [
    "graph", "algo", "sigma_lambda", "sigma_delta", "sigma_nu",
    "cycles", "trials", "seed", "mean_cut", "std_cut",
    "normalized_mean_cut", "mean_final_energy", "anneal_seconds",
]
TRACE_COLUMNS = ["trial", "cycle", "i0", "energy", "cut"]

_CHUNK = 1 << 18  # rows assembled per pass (bounds the index temporaries)


def fmt(x: object) -> str:
    """cli.py:36-41"""
    if x is None:
        return ""
    if isinstance(x, float):
        return repr(x)
    return str(x)


def _itoa(v: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """Decimal text of int64 values: ([N, W] bytes, left-aligned) and lengths;
    W is the widest value's width (one digit pass per digit actually present)."""
    v = np.asarray(v, dtype=np.int64)
    neg = v < 0
    mag = np.where(neg, -(v + 1), v).astype(np.uint64) + neg.astype(np.uint64)  # |v|, INT64_MIN safe
    top = int(mag.max()) if mag.size else 0
    ndig = len(str(top))
    small = top < 2 ** 31  # 32-bit division is much faster than 64-bit
    x = mag.astype(np.uint32 if small else np.uint64)
    nd = np.ones(v.shape, np.int64)
    t = x // 10
    for _ in range(ndig - 1):
        nd += t > 0
        t //= 10
    width = nd + neg
    W = ndig + 1
    out = np.zeros(v.shape + (W,), np.uint8)
    rows = np.arange(v.size)
    for j in range(ndig):  # j-th digit from the right
        d = (x % 10).astype(np.uint8) + 48
        x //= 10
        pos = width - 1 - j
        ok = j < nd
        out[rows[ok], pos[ok]] = d[ok]
    out[neg, 0] = ord("-")
    return out, width


def _float_strs(vals: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """repr() text of float64 values as ([N, W] bytes, lengths); integral
    values below 1e16 take the integer digits + '.0' path."""
    vals = np.asarray(vals, dtype=np.float64)
    integral = np.isfinite(vals) & (vals == np.trunc(vals)) & (np.abs(vals) < 1e16) & ~(
        (vals == 0.0) & np.signbit(vals))
    ints = np.where(integral, vals, 0.0).astype(np.int64)
    digits, w = _itoa(ints)
    out = np.zeros((vals.size, max(26, digits.shape[1] + 2)), np.uint8)
    out[:, :digits.shape[1]] = digits
    rows = np.arange(vals.size)
    out[rows, w] = ord(".")
    out[rows, w + 1] = ord("0")
    lens = w + 2
    for k in np.nonzero(~integral)[0]:  # the rest: exact repr, entry by entry
        s = repr(float(vals[k])).encode()
        out[k, :] = 0
        out[k, :len(s)] = np.frombuffer(s, np.uint8)
        lens[k] = len(s)
    return out, lens


def _native_rows(results: Sequence) -> bytes | None:
    """The common case -- one shared i0 trace, integral energies, cuts on every
    trial or on none -- formatted by the CUDA library's host-side formatter
    (pbsa_format_trace_csv, all host threads); None when it does not apply
    or the library is absent (then the numpy path below runs)."""
    i0 = np.asarray(results[0].i0_trace, dtype=np.float64)
    if any(r.i0_trace.shape != i0.shape or not np.array_equal(r.i0_trace, i0) for r in results):
        return None
    cuts_none = [r.cut_trace is None for r in results]
    if any(cuts_none) and not all(cuts_none):
        return None
    e = np.stack([np.asarray(r.energy_trace, dtype=np.float64) for r in results])
    if not (np.all(np.isfinite(e)) and np.all(e == np.trunc(e)) and np.all(np.abs(e) < 1e16)
            and not np.any((e == 0.0) & np.signbit(e))):
        return None
    try:
        from . import _native
        _native.load()
    except (RuntimeError, OSError):
        return None
    cut = None if cuts_none[0] else np.stack([np.asarray(r.cut_trace, dtype=np.int64) for r in results])
    return _native.format_trace_rows([repr(float(x)).encode() for x in i0], e.astype(np.int64), cut)


def trace_csv_bytes(results: Sequence) -> bytes:
    """The bytes cli._write_csv(path, TRACE_COLUMNS, cli._trace_rows(summary))
    writes for ``summary.results == results`` (objects with ``i0_trace``,
    ``energy_trace`` and ``cut_trace`` (or None), like TrialResult)."""
    head = (",".join(TRACE_COLUMNS) + "\n").encode()
    if not results:
        return head
    fast = _native_rows(results)
    if fast is not None:
        return head + fast
    parts = [head]
    # i0: one repr per distinct trace, reused by every trial sharing it
    i0_cache: dict[bytes, tuple[np.ndarray, np.ndarray]] = {}
    rows_t, rows_c, i0_txt, i0_len, energies, cuts, has_cut = [], [], [], [], [], [], []
    for t, r in enumerate(results):
        i0 = np.ascontiguousarray(r.i0_trace, dtype=np.float64)
        key = i0.tobytes()
        if key not in i0_cache:
            i0_cache[key] = _float_strs(i0)
        txt, ln = i0_cache[key]
        C = i0.size
        rows_t.append(np.full(C, t, np.int64))
        rows_c.append(np.arange(C, dtype=np.int64))
        i0_txt.append(txt)
        i0_len.append(ln)
        energies.append(np.asarray(r.energy_trace, dtype=np.float64))
        if r.cut_trace is None:
            cuts.append(np.zeros(C, np.int64))
            has_cut.append(np.zeros(C, bool))
        else:
            cuts.append(np.asarray(r.cut_trace, dtype=np.int64))
            has_cut.append(np.ones(C, bool))
    cols = [np.concatenate(x) for x in (rows_t, rows_c, energies, cuts, has_cut)]
    i0_txt = np.concatenate(i0_txt)
    i0_len = np.concatenate(i0_len)
    N = cols[0].size
    for lo in range(0, N, _CHUNK):
        hi = min(N, lo + _CHUNK)
        fields = [_itoa(cols[0][lo:hi]), _itoa(cols[1][lo:hi]), (i0_txt[lo:hi], i0_len[lo:hi]),
                  _float_strs(cols[2][lo:hi])]
        ct, cl = _itoa(cols[3][lo:hi])
        fields.append((ct, np.where(cols[4][lo:hi], cl, 0)))
        n = hi - lo
        row_len = sum(f[1] for f in fields) + len(fields)  # 4 commas + newline
        off = np.zeros(n + 1, np.int64)
        np.cumsum(row_len, out=off[1:])
        buf = np.full(int(off[-1]), ord(","), np.uint8)
        buf[off[1:] - 1] = ord("\n")
        pos = off[:-1].copy()
        for txt, ln in fields:
            w = txt.shape[1]
            idx = pos[:, None] + np.arange(w)[None, :]
            m = np.arange(w)[None, :] < ln[:, None]
            buf[idx[m]] = txt[m]
            pos += ln + 1
        parts.append(buf.tobytes())
    return b"".join(parts)


def write_trace_csv(path: str, results: Sequence) -> None:
    """cli.py:196 (``--trace-out``), byte-identical."""
    with open(path, "wb") as fh:
        fh.write(trace_csv_bytes(results))


def summary_row(spec, summary) -> list[str]:
    """cli._summary_row (cli.py:146-152)."""
    v = spec.variability
    return [fmt(x) for x in [
        spec.graph, spec.algo.kind.value, v.sigma_lambda, v.sigma_delta, v.sigma_nu,
        spec.cycles, spec.trials, spec.base_seed, summary.mean_cut, summary.std_cut,
        summary.normalized_mean_cut, summary.mean_final_energy, summary.anneal_seconds,
    ]]


def summary_csv_bytes(rows: Sequence[Sequence[str]], extra_columns: Sequence[str] = ()) -> bytes:
    """csv.writer output of SUMMARY_COLUMNS (+ the sweep's "axis", "value")
    and the given rows (cli.py:155-159, 194, 222)."""
    fh = io.StringIO(newline="")
    w = csv.writer(fh, lineterminator="\n")
    w.writerow(list(SUMMARY_COLUMNS) + list(extra_columns))
    w.writerows(rows)
    return fh.getvalue().encode()


def write_summary_csv(path: str, spec, summary) -> None:
    """cli.py:194 (``--summary-out`` of ``run``)."""
    with open(path, "wb") as fh:
        fh.write(summary_csv_bytes([summary_row(spec, summary)]))


def write_sweep_summary_csv(path: str, specs: Sequence, summaries: Sequence, axis: str,
                            values: Sequence[float]) -> None:
    """cli.py:213-222 (``--summary-out`` of ``sweep``): one row per point plus
    the axis name and value."""
    rows = [summary_row(s, m) + [fmt(axis), fmt(float(v))]
            for s, m, v in zip(specs, summaries, values)]
    with open(path, "wb") as fh:
        fh.write(summary_csv_bytes(rows, ["axis", "value"]))
