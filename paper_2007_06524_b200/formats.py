"""Wire formats on either side of the solve.

Input side: realizations travel as the reference's JSON document
(``Realization.to_json`` / ``from_json``, lattice.py:229-250, in lattice.py
here).  Output side: the per-iteration trace of a ``PcgReport`` as the rows the
reference CLI writes (``trace.csv``: ``iteration,rel_residual``, cells
formatted by ``_fmt`` = repr for floats, cli.py:264-267,281-287,358-360), so a
GPU solve can be dropped under the reference tooling with identical bytes.
The CLI itself, its TOML configuration and the Kronecker-rank report fields are
outside the hot path and not rebuilt.
"""

from __future__ import annotations

from pathlib import Path


def fmt_cell(value) -> str:
    """cli.py:264-267."""
    if isinstance(value, float):
        return repr(value)
    return str(value)


def trace_rows(report) -> list:
    """(iteration, relative residual) pairs of a PcgReport, 1-based (cli.py:358-360)."""
    return list(enumerate(report.residuals, start=1))


def trace_csv_lines(report, header_lines=()) -> list:
    """Lines of ``trace.csv`` (cli.py:281-287): optional ``# key = value`` header
    lines, the column line, one row per iteration."""
    lines = list(header_lines)
    lines.append("iteration,rel_residual")
    for row in trace_rows(report):
        lines.append(",".join(fmt_cell(v) for v in row))
    return lines


def write_trace_csv(path, report, header_lines=()) -> None:
    Path(path).write_text("\n".join(trace_csv_lines(report, header_lines)) + "\n")


def batch_reports(result, name: str) -> list:
    """Per-realization ``PcgReport`` objects of a batched solve (BatchResult)."""
    return [result.report(b, name) for b in range(len(result.iterations))]
