"""GPU parity of the per-patch trackers (run_tracking_patched, restating experiment._run_tracking_patched,
experiment.py:332-441) against the reference's own outputs (tests/golden/patched_*.npz) and the oracle:
per-step gammas / costs / step sizes / residuals within 1e-4 relative, the assembled reconstructions
within 1e-4, NRMSE trajectory within 1e-3 absolute, reshuffle orders and t exact."""

import numpy as np
import pytest

from conftest import rel
from oracle import tt_oracle as O
from test_patched_oracle import load_case, replay_rng

pytestmark = pytest.mark.gpu


def _grid_step(c):
    import paper_1609_04104_b200 as tt

    n1, n2, rho = (int(x) for x in c["patch"])
    grid = tt.PatchGrid(tuple(int(x) for x in c["shape"]), n1, n2, rho)
    kind, par = c["step"][0], c["step"][1:]
    step = tt.Fixed(par[0]) if kind == "fixed" else tt.HessianBound(par[0], par[1])
    return grid, step


@pytest.mark.parametrize("name", ["patched_vd", "patched_uniform"])
def test_patched_matches_reference(name):
    import paper_1609_04104_b200 as tt

    c = load_case(name)
    grid, step = _grid_step(c)
    res = tt.run_tracking_patched(c["frames"], grid, float(c["lam"]), step, c["entries_list"], warm_n=int(c["warm_n"]),
                                  warm_epochs=int(c["warm_epochs"]), epochs=int(c["epochs"]), rng=replay_rng(c),
                                  reshuffle=bool(c["reshuffle"]), A0s=c["A0s"], B0s=c["B0s"], keep_residual=True)
    np.testing.assert_array_equal(np.concatenate(res.orders), c["orders"])
    np.testing.assert_array_equal(res.step_t, c["trace_t"])
    assert len(res.step_gamma) == len(c["trace_gamma"])
    for k in range(len(res.step_gamma)):
        assert rel(res.step_gamma[k], c["trace_gamma"][k]) < 1e-4, k
        assert rel(res.step_cost[k], c["trace_cost"][k]) < 1e-4, k
        assert rel(res.step_mu[k], c["trace_mu"][k]) < 1e-4, k
        want = c["trace_resid"][k, :c["trace_resid_len"][k]]
        assert res.step_residual[k].shape == want.shape
        assert rel(res.step_residual[k], want) < 1e-4, k
    for t in range(int(c["T"])):
        assert rel(res.recon[t], c["recon"][t]) < 1e-4, t
    assert np.max(np.abs(np.sqrt(res.nmse) - np.sqrt(c["nmse"]))) < 1e-3
    np.testing.assert_array_equal(res.samples, c["counts"])


def test_patched_larger_grid_vs_oracle():
    """64 x 64 frames, 16 x 16 patches of rank 4, VD rows, HessianBound steps (closed form on both
    sides), two reshuffled epochs: device == oracle restatement."""
    import paper_1609_04104_b200 as tt

    N, n, rho, T, warm = 64, 16, 4, 8, 2
    grid = tt.PatchGrid((N, N), n, n, rho)
    rng = np.random.Generator(np.random.Philox(5))  # device VD draws index the Philox stream
    A0s, B0s = tt.init_patch_factors(grid, rng)
    masks = [tt.full_entries((N, N))] * warm + [tt.draw_frame_entries("variable_density", (N, N), rng, 0.3)
                                                 for _ in range(T - warm)]
    g = np.random.default_rng(6)
    u = g.standard_normal((N, 2)) + 1j * g.standard_normal((N, 2))
    frames = np.stack([(u * [1.0, 0.3 * np.cos(0.5 * t)]) @ u.T / N + 0.01 * (g.standard_normal((N, N)) + 1j * g.standard_normal((N, N)))
                       for t in range(T)])
    state = rng.bit_generator.state
    res = tt.run_tracking_patched(frames, grid, 0.05, tt.HessianBound(1e-3, 1e9), masks, warm_n=warm, warm_epochs=2,
                                  epochs=2, rng=rng, reshuffle=True, A0s=A0s, B0s=B0s)
    rng2 = np.random.Generator(np.random.Philox(5))
    rng2.bit_generator.state = state
    ref = O.patched_run(frames, A0s, B0s, 0.05, ("hessian", 1e-3, 1e9), n, n, masks, warm, 2, 2, rng=rng2,
                        reshuffle=True, power=False)
    assert [list(o) for o in res.orders] == [list(o) for o in ref["orders"]]
    for k, st in enumerate(ref["trace"]):
        assert rel(res.step_gamma[k], st["gamma"]) < 1e-4, k
        assert rel(res.step_cost[k], st["cost"]) < 1e-4, k
        assert rel(res.step_mu[k], st["mu"]) < 1e-4, k
    assert rel(res.recon, ref["recon"]) < 1e-4
    for p, (A, B, t, ab) in enumerate(ref["final"]):
        assert rel(res.final_A[p], A) < 1e-4 and rel(res.final_B[p], B) < 1e-4
        assert res.t == t


def test_patched_errors_and_edges():
    import paper_1609_04104_b200 as tt

    N = 16
    grid = tt.PatchGrid((N, N), 8, 8, 2)
    rng = np.random.default_rng(1)
    A0s, B0s = tt.init_patch_factors(grid, rng)
    frames = np.ones((3, N, N), np.complex64)
    full = tt.full_entries((N, N))
    dup = np.concatenate([full[:10], full[3:4]])
    with pytest.raises(ValueError, match="duplicate"):
        tt.run_tracking_patched(frames, grid, 0.1, tt.Fixed(0.01), [full, dup, full], warm_n=1, A0s=A0s, B0s=B0s)
    bad = np.array([[0, 0], [N, 1]])
    with pytest.raises(ValueError, match="out of range"):
        tt.run_tracking_patched(frames, grid, 0.1, tt.Fixed(0.01), [full, bad, full], warm_n=1, A0s=A0s, B0s=B0s)
    with pytest.raises(TypeError):
        g17 = tt.PatchGrid((N, N), 8, 8, 17)
        a17, b17 = tt.init_patch_factors(g17, rng)
        tt.run_tracking_patched(frames, g17, 0.1, tt.Fixed(0.01), [full] * 3, A0s=a17, B0s=b17)
    with pytest.raises(ValueError):
        tt.PatchGrid((N, N), 5, 8, 2)
    # all frames warm: no main steps, every frame still re-projected; an empty frame mask is a zero step
    res = tt.run_tracking_patched(frames, grid, 0.1, tt.Fixed(0.01), [full, np.zeros((0, 2)), full], warm_n=3,
                                  A0s=A0s, B0s=B0s)
    assert res.step_gamma.shape == (0, 4 * 2) and res.recon.shape == (3, N, N)
    ref = O.patched_run(frames, A0s, B0s, 0.1, ("fixed", 0.01), 8, 8, [full, np.zeros((0, 2), np.int64), full], 3, 1, 1)
    assert rel(res.recon, ref["recon"]) < 1e-4
    assert np.all(res.gamma[1] == 0)
