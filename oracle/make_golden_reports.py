"""Golden run-artefact CSVs written by the reference's own writers
(experiment.py:641-675) for fixed rows. Test infrastructure only: run in the
build container; the files are committed under tests/golden/reports/.
scikit-image is absent here, so a stub `skimage.metrics` is registered before
importing the reference's experiment module; the writers do not
use it.
"""

from __future__ import annotations

import importlib
import os
import sys
import types

import numpy as np

REF_PKG = "/root/reference/pkg/src/tensortrack"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden", "reports")


def rows():
    """The fixed inputs (shared with tests/test_reports.py)."""
    metrics = [(0, 0.125, 0.9, 256), (1, 1.0 / 3.0, 0.5 + 1e-17, 64), (2, 1e-300, -0.0, 0), (3, 2.5e10, 1.0, 7)]
    mask_rows = [(0, -1), (1, 0), (1, 5), (2, 255)]
    mask_entries = [(4, 1, 2), (4, 0, 0), (5, 7, 9)]
    budget = [(5, 64, 47, 47.123456789012345), (6, 64, 50, 1.0 / 7.0)]
    trace = [(1, 0.5, 0.01, np.array([1 + 2j, -0.5j]), np.array([0.1, 0.2 - 0.3j, 1e-9])),
             (2, 1.0 / 3.0, 0.0, np.array([0j]), np.zeros(0, complex))]
    return metrics, mask_rows, mask_entries, budget, trace


def main():
    if "tensortrack" not in sys.modules:
        pkg = types.ModuleType("tensortrack")
        pkg.__path__ = [REF_PKG]
        sys.modules["tensortrack"] = pkg
    sk = types.ModuleType("skimage")
    skm = types.ModuleType("skimage.metrics")
    skm.structural_similarity = lambda *a, **k: 0.0
    sk.metrics = skm
    sys.modules.setdefault("skimage", sk)
    sys.modules.setdefault("skimage.metrics", skm)
    ex = importlib.import_module("tensortrack.experiment")
    me = importlib.import_module("tensortrack.metrics")
    metrics, mask_rows, mask_entries, budget, trace = rows()
    os.makedirs(OUT, exist_ok=True)
    ex.write_metrics_csv(os.path.join(OUT, "metrics.csv"), [me.MetricRow(*m) for m in metrics])
    ex.write_mask_csv(os.path.join(OUT, "mask_rows.csv"), mask_rows)
    ex.write_mask_csv(os.path.join(OUT, "mask_entries.csv"), mask_entries)
    ex.write_mask_csv(os.path.join(OUT, "mask_empty.csv"), [])
    ex.write_budget_csv(os.path.join(OUT, "budget.csv"), budget)
    reps = [types.SimpleNamespace(t=t, instantaneous_cost=f, step_size=m, gamma=g, residual=r) for t, f, m, g, r in trace]
    ex.write_trace_csv(os.path.join(OUT, "trace.csv"), reps)
    print("wrote", sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main()
