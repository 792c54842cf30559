"""The per-patch tracker oracle (oracle.patched_run, restating experiment._run_tracking_patched,
experiment.py:332-441) against the reference's own outputs (tests/golden/patched_*.npz, written by
oracle/make_golden_patched.py, which runs the reference's run_tracking with a PatchConfig)."""

import os

import numpy as np
import pytest

from oracle import tt_oracle as O

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def load_case(name):
    z = np.load(os.path.join(GOLDEN, f"{name}.npz"), allow_pickle=False)
    c = {k: z[k] for k in z.files}
    c["entries_list"] = [c["entries"][t, :c["counts"][t]].astype(np.int64) for t in range(int(c["T"]))]
    kind = str(c["step_kind"])
    c["step"] = ("fixed", float(c["step_par"][0])) if kind == "fixed" else ("hessian", *map(float, c["step_par"]))
    return c


def replay_rng(c):
    """The reference's generator after its inits and masks (experiment.py:346-381), ready for the
    reshuffle permutations: random_subspace draws two (n, rho) normals per mode per patch,
    variable_density_rows one uniform per row after the DC line."""
    n1, n2, rho = (int(x) for x in c["patch"])
    rng = np.random.default_rng(int(c["seed"]))
    for _ in range(len(c["A0s"])):
        for n in (n1, n2):
            rng.standard_normal((n, rho))
            rng.standard_normal((n, rho))
    for t in range(int(c["warm_n"]), int(c["T"])):
        rng.random(len(np.unique(c["entries_list"][t][:, 0])) - 1)
    return rng


def run_oracle(c, power=True):
    n1, n2, rho = (int(x) for x in c["patch"])
    return O.patched_run(c["frames"], c["A0s"], c["B0s"], float(c["lam"]), c["step"], n1, n2, c["entries_list"],
                         int(c["warm_n"]), int(c["warm_epochs"]), int(c["epochs"]), rng=replay_rng(c),
                         reshuffle=bool(c["reshuffle"]), power=power)


@pytest.mark.parametrize("name", ["patched_vd", "patched_uniform"])
def test_patched_oracle_matches_reference(name):
    c = load_case(name)
    out = run_oracle(c)
    np.testing.assert_array_equal(np.concatenate(out["orders"]), c["orders"])
    for k, st in enumerate(out["trace"]):
        np.testing.assert_allclose(st["gamma"], c["trace_gamma"][k], rtol=1e-9, atol=1e-12)
        np.testing.assert_allclose(st["residual"], c["trace_resid"][k, :c["trace_resid_len"][k]], rtol=1e-9, atol=1e-12)
        assert st["cost"] == pytest.approx(c["trace_cost"][k], rel=1e-10)
        assert st["mu"] == pytest.approx(c["trace_mu"][k], rel=1e-10)
        assert st["t"] == c["trace_t"][k]
    np.testing.assert_allclose(out["recon"], c["recon"], rtol=1e-9, atol=1e-12)


def test_patch_split_and_assemble():
    """patch_batches' stable filter and patch_assemble (mri.py:151-177): the 4x4 frame / 2x2 patch
    quadrants of the reference's test (test_mri.py:147-154), entries kept in measurement order."""
    frame = np.arange(16).reshape(4, 4)
    ent = np.array([[3, 3], [0, 1], [2, 0], [0, 0], [1, 2]])
    parts = O.patch_split(ent, frame[ent[:, 0], ent[:, 1]], 4, 4, 2, 2)
    np.testing.assert_array_equal(parts[0][0], [[0, 1], [0, 0]])
    np.testing.assert_array_equal(parts[0][1], [1, 0])
    np.testing.assert_array_equal(parts[1][0], [[1, 0]])
    np.testing.assert_array_equal(parts[2][0], [[0, 0]])
    np.testing.assert_array_equal(parts[3][0], [[1, 1]])
    tiles = [frame[p * 2:(p + 1) * 2, q * 2:(q + 1) * 2] for p in range(2) for q in range(2)]
    np.testing.assert_array_equal(tiles[1], [[2, 3], [6, 7]])
    np.testing.assert_array_equal(O.patch_assemble(tiles, 4, 4, 2, 2), frame)
