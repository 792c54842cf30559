"""CPU: checkpoint files of a host TrackerState (A, B, t, alpha_bar over CTEN + state.json) round-trip
exactly; the manifest writer follows run_experiment's format (experiment.py:727-741)."""

import json
import os

import numpy as np
import pytest

import paper_1609_04104_b200 as tt
from paper_1609_04104_b200 import checkpoint


def test_tracker_state_round_trip(tmp_path):
    rng = np.random.default_rng(3)
    A = rng.standard_normal((12, 3)) + 1j * rng.standard_normal((12, 3))
    B = rng.standard_normal((9, 3)) + 1j * rng.standard_normal((9, 3))
    cfg = tt.StepConfig(0.05, 3, tt.HessianBound(1e-3, 1e9), norm_cap=7.5)
    st = tt.TrackerState(tt.TensorSubspace((A, B)), cfg, t=17, alpha_bar=0.1 + 1e-17 * 3)
    checkpoint.save_state(st, tmp_path / "ck")
    back = checkpoint.load_state(tmp_path / "ck")
    np.testing.assert_array_equal(back.subspace.factors[0], A)  # float64 pairs: exact
    np.testing.assert_array_equal(back.subspace.factors[1], B)
    assert back.t == 17 and back.alpha_bar == st.alpha_bar
    assert back.config.lam == 0.05 and back.config.rank == 3 and back.config.norm_cap == 7.5
    assert isinstance(back.config.step, tt.HessianBound) and back.config.step.c_cap == 1e9
    meta = json.loads((tmp_path / "ck" / "state.json").read_text())
    assert meta["kind"] == "state" and meta["domain"] == "image"
    with pytest.raises(ValueError):
        checkpoint.load_engine(None, tmp_path / "ck")  # not an engine checkpoint


def test_checkpoint_version_is_checked(tmp_path):
    st = tt.TrackerState(tt.TensorSubspace((np.ones((4, 2)), np.ones((3, 2)))), tt.StepConfig(0.1, 2))
    checkpoint.save_state(st, tmp_path)
    p = tmp_path / "state.json"
    meta = json.loads(p.read_text())
    meta["version"] = 99
    p.write_text(json.dumps(meta))
    with pytest.raises(ValueError, match="version"):
        checkpoint.load_state(tmp_path)


def test_manifest_format(tmp_path):
    path = tmp_path / "manifest.json"
    m = tt.write_manifest(path, "adaptive", "in.cten", {"seed": 7, "lam": 0.05}, [1.23456, 2.0], [0.5, 0.25], 1.5,
                          commit="abc")
    text = path.read_text()
    assert text.endswith("}\n")
    assert text == json.dumps(m, indent=2, sort_keys=True) + "\n"
    assert m["timings"]["per_frame_ms"] == [1.235, 2.0] and m["mean_nmse"] == 0.375
    assert sorted(m) == ["commit", "config", "input", "mean_nmse", "mode", "timings"]
