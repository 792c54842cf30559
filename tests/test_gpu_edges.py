"""GPU parity at shapes the configuration tests do not reach: rectangular and non-power-of-two frames
(the direct-DFT column transform), rank 1, and the rank ranges that select the other solver variants
(Gauss-Jordan with 1 / 2 / 5 entries per thread, the 2x2-blocked LDL^H beyond R = 32) in the row-mask
engine; rank 1 and rank 40 in the entry-mask engine (its LDL^H path); patch ranks 1 and 16 on
non-square patches. Every case against the oracle: per-frame gamma and final factors within 1e-4."""

import numpy as np
import pytest

from conftest import rel
from oracle import tt_oracle as O

pytestmark = pytest.mark.gpu


def _lowrank(T, nx, ny, seed):
    g = np.random.default_rng(seed)
    u = g.standard_normal((nx, 3)) + 1j * g.standard_normal((nx, 3))
    v = g.standard_normal((ny, 3)) + 1j * g.standard_normal((ny, 3))
    out = []
    for t in range(T):
        c = np.array([1.0, 0.5 * np.cos(0.4 * t), 0.3 * np.sin(0.3 * t)])
        out.append((u * c) @ v.T / np.sqrt(nx * ny) + 0.02 * (g.standard_normal((nx, ny)) + 1j * g.standard_normal((nx, ny))))
    return np.stack(out)


@pytest.mark.parametrize("nx,ny,R", [(96, 80, 1), (100, 60, 5), (64, 48, 16), (64, 48, 33), (48, 40, 40)])
def test_row_engine_odd_shapes_and_solver_variants(nx, ny, R):
    import paper_1609_04104_b200 as tt

    T, lam = 6, 0.1
    ks = _lowrank(T, nx, ny, nx + R)
    A0, B0 = O.random_subspace(nx, ny, R, seed=R)
    g = np.random.default_rng(R)
    S = max(2, nx // 4)
    rows = [np.sort(g.choice(nx, S, replace=False)) for _ in range(T)]
    ref = O.online_run(ks, A0, B0, lam, ("fixed", 0.05), {"kind": "static", "rows": rows}, record_factors=True)
    tab = np.stack(rows)[:, None, :]
    res = tt.run_online(ks, A0[None], B0[None], lam, tt.Fixed(0.05), tt.StaticRows(tab, np.full((T, 1), S)))
    for f in range(T):
        assert rel(res.gamma[f, 0], ref["gamma"][f]) < 1e-4, f
    assert rel(res.final_A[0], ref["A"][-1]) < 1e-4
    assert rel(res.final_B[0], ref["B"][-1]) < 1e-4


@pytest.mark.parametrize("R", [1, 40])
def test_entry_engine_rank_extremes(R):
    import paper_1609_04104_b200 as tt

    n, T, lam = 32, 5, 0.1
    ks = _lowrank(T, n, n, 7 + R)
    A0, B0 = O.random_subspace(n, n, R, seed=8 + R)
    g = np.random.default_rng(R)
    lists = [g.permutation(g.choice(n * n, 300, replace=False)) for _ in range(T)]
    ref = O.online_run_entries(ks, O.fft_cols(A0), O.fft_cols(B0), lam, ("fixed", 0.05),
                               {"kind": "static", "entries": lists}, record_factors=True)
    tab = np.stack(lists)
    res = tt.run_online(ks, A0[None], B0[None], lam, tt.Fixed(0.05), tt.StaticEntries(tab, np.full(T, 300)))
    for f in range(T):
        assert rel(res.gamma[f, 0], ref["gamma"][f]) < 1e-4, f
    assert rel(res.final_A[0], O.fft_cols(ref["A"][-1], inverse=True)) < 1e-4


@pytest.mark.parametrize("rho,n1,n2", [(1, 8, 4), (16, 16, 8)])
def test_patch_ranks_on_non_square_patches(rho, n1, n2):
    import paper_1609_04104_b200 as tt

    N1, N2, T, warm = 32, 16, 6, 2
    grid = tt.PatchGrid((N1, N2), n1, n2, rho)
    rng = np.random.Generator(np.random.Philox(rho))
    A0s, B0s = tt.init_patch_factors(grid, rng)
    masks = [tt.full_entries((N1, N2))] * warm + [tt.draw_frame_entries("uniform", (N1, N2), rng, 0.4)
                                                   for _ in range(T - warm)]
    frames = _lowrank(T, N1, N2, 3 + rho)
    res = tt.run_tracking_patched(frames, grid, 0.1, tt.HessianBound(1e-3, 1e9), masks, warm_n=warm, warm_epochs=2,
                                  A0s=A0s, B0s=B0s)
    ref = O.patched_run(frames, A0s, B0s, 0.1, ("hessian", 1e-3, 1e9), n1, n2, masks, warm, 2, 1, power=False)
    for k, st in enumerate(ref["trace"]):
        assert rel(res.step_gamma[k], st["gamma"]) < 1e-4, k
        assert rel(res.step_mu[k], st["mu"]) < 1e-4, k
    assert rel(res.recon, ref["recon"]) < 1e-4


@pytest.mark.parametrize("nx,ny,R", [(64, 48, 33), (48, 40, 40), (40, 36, 64)])
def test_row_engine_tight_plan(nx, ny, R, monkeypatch):
    """The tight shared-memory plan (no fp32 GA/GB copies, no fp64 Bh staging, the two update GEMMs in
    sequence with a gamma-scaled R x R operand; rows_make_plan_cap) forced at small shapes."""
    import paper_1609_04104_b200 as tt

    monkeypatch.setenv("TT_ROWS_FORCE_TIGHT", "1")
    T, lam = 6, 0.1
    ks = _lowrank(T, nx, ny, nx + R + 1)
    A0, B0 = O.random_subspace(nx, ny, R, seed=R + 1)
    g = np.random.default_rng(R + 1)
    S = max(2, nx // 3)
    rows = [np.sort(g.choice(nx, S, replace=False)) for _ in range(T)]
    ref = O.online_run(ks, A0, B0, lam, ("fixed", 0.05), {"kind": "static", "rows": rows}, record_factors=True)
    tab = np.stack(rows)[:, None, :]
    res = tt.run_online(ks, A0[None], B0[None], lam, tt.Fixed(0.05), tt.StaticRows(tab, np.full((T, 1), S)))
    for f in range(T):
        assert rel(res.gamma[f, 0], ref["gamma"][f]) < 1e-4, f
    assert rel(res.final_A[0], ref["A"][-1]) < 1e-4
    assert rel(res.final_B[0], ref["B"][-1]) < 1e-4


@pytest.mark.parametrize("kind", ["static", "informative"])
def test_row_engine_1024_rank64(kind):
    """1024^2 at R = 64 (BASELINE C5's largest point): only the tight plan fits; several k tiles per
    frame (KT < S). Three frames against the oracle."""
    import paper_1609_04104_b200 as tt

    n, R, T, lam = 1024, 64, 3, 0.05
    ks = _lowrank(T, n, n, 11)
    A0, B0 = O.random_subspace(n, n, R, seed=12)
    if kind == "static":
        gen = np.random.Generator(np.random.Philox(key=5))
        rows = [O.vd_rows(n, -1.0, 0.1, gen.random) for _ in range(T)]
        S = len(rows[0])
        ref = O.online_run(ks, A0, B0, lam, ("fixed", 0.01), {"kind": "static", "rows": rows}, record_factors=True)
        res = tt.run_online(ks, A0[None], B0[None], lam, tt.Fixed(0.01),
                            tt.StaticRows(np.stack(rows)[:, None, :], np.full((T, 1), S)))
    else:
        ref = O.online_run(ks, A0, B0, lam, ("fixed", 0.01),
                           {"kind": "informative", "k": 103, "forced": [0], "beta": 0.1, "key": (9, 0)},
                           record_factors=True)
        res = tt.run_online(ks, A0[None], B0[None], lam, tt.Fixed(0.01),
                            tt.Informative(k=103, forced=(0,), beta=0.1, key0=9))
        for f in range(T):
            assert np.array_equal(res.rows[f][0], ref["rows"][f]), f
    for f in range(T):
        assert rel(res.gamma[f, 0], ref["gamma"][f]) < 1e-4, f
    assert rel(res.final_A[0], ref["A"][-1]) < 1e-4
    assert rel(res.final_B[0], ref["B"][-1]) < 1e-4
