"""Run-artefact CSVs byte-identical to the reference's writers (experiment.py:641-675);
goldens written by the reference itself (oracle/make_golden_reports.py). Host-only."""

import os
import sys
import types

import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden", "reports")
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from oracle.make_golden_reports import rows  # noqa: E402  (the fixed inputs)


def _read(name):
    with open(os.path.join(GOLD, name), "rb") as fh:
        return fh.read()


def test_writers_match_reference_bytes(tmp_path):
    from paper_1609_04104_b200 import reports as R

    metrics, mask_rows, mask_entries, budget, trace = rows()
    R.write_metrics_csv(tmp_path / "m.csv", [R.MetricRow(*m) for m in metrics])
    assert (tmp_path / "m.csv").read_bytes() == _read("metrics.csv")
    R.write_mask_csv(tmp_path / "r.csv", mask_rows)
    assert (tmp_path / "r.csv").read_bytes() == _read("mask_rows.csv")
    R.write_mask_csv(tmp_path / "e.csv", mask_entries)
    assert (tmp_path / "e.csv").read_bytes() == _read("mask_entries.csv")
    R.write_mask_csv(tmp_path / "z.csv", [])
    assert (tmp_path / "z.csv").read_bytes() == _read("mask_empty.csv")
    R.write_budget_csv(tmp_path / "b.csv", budget)
    assert (tmp_path / "b.csv").read_bytes() == _read("budget.csv")
    reps = [types.SimpleNamespace(t=t, instantaneous_cost=f, step_size=m, gamma=g, residual=r) for t, f, m, g, r in trace]
    R.write_trace_csv(tmp_path / "t.csv", reps)
    assert (tmp_path / "t.csv").read_bytes() == _read("trace.csv")
