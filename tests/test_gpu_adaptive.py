"""GPU: run_adaptive's schedule on the device loop against the reference's own run_adaptive
(tests/golden/adaptive_*.npz): warm-up, variable-density rows until the switch frame (drawn on the device
from the Philox stream the reference's generator uses), then informative draws with and without replacement
inside the fused rows kernel. Masks bit-exact, gamma 1e-4 per frame, NRMSE 1e-3 over the sequence, final
factors 1e-4. Plus the norm_cap flags (tracker.py:406-408) against the oracle's post-update norms."""

import numpy as np
import pytest

from conftest import load_golden, rel
from oracle import tt_oracle as O

pytestmark = pytest.mark.gpu

NAMES = ["switch_wr", "switch_wor", "wor_nowarm"]


@pytest.mark.parametrize("name", NAMES)
@pytest.mark.parametrize("cluster", [0, 2])
def test_device_schedule_matches_reference_run_adaptive(name, cluster):
    import paper_1609_04104_b200 as tt

    g = load_golden("adaptive_" + name)
    n, R, T, W, E, switch, k, repl, seed, pos0, nvd = (int(v) for v in g["meta"])
    ks = g["kspace"]
    A0 = O.fft_cols(g["Ah0"], inverse=True)
    B0 = O.fft_cols(g["Bh0"], inverse=True)
    clean = np.stack([O.dft2(ks[t].astype(np.complex128), inverse=True) for t in range(T)])
    inf = tt.Informative(k=k, forced=(0,), beta=0.1, key0=seed, replacement=bool(repl), pos0=pos0)
    pol = tt.AdaptiveSchedule(inf, switch_frame=switch, alpha=-1.0, fraction=float(g["fraction"]))
    res = tt.run_online(ks, A0[None], B0[None], float(g["lam"]), tt.Fixed(float(g["mu"])), pol, clean=clean,
                        warm_frames=W, warm_epochs=E, cluster=cluster, chunk=5)
    for f in range(T - W):
        want = g["rows"][f, :g["counts"][f]]
        np.testing.assert_array_equal(np.sort(res.rows[f][0]), want, err_msg=f"frame {f}")
        assert rel(res.gamma[f, 0], g["gamma"][f]) < 1e-4, f
    assert np.max(np.abs(np.sqrt(res.nmse[:, 0]) - np.sqrt(g["nmse"]))) < 1e-3
    assert rel(O.fft_cols(res.final_A[0]), g["Af"]) < 1e-4
    assert rel(O.fft_cols(res.final_B[0]), g["Bf"]) < 1e-4
    np.testing.assert_allclose(res.cost[:, 0], g["cost"], rtol=1e-4)


def test_wor_draws_without_forced_and_large_k():
    """Without replacement at k close to nx (most rows drawn) and no forced rows: every frame has
    exactly k distinct rows and equals the oracle's draw over the oracle's own probabilities."""
    import paper_1609_04104_b200 as tt
    from paper_1609_04104_b200.phantom import cine_phantom

    n, R, T, k = 64, 6, 6, 60
    ph = cine_phantom(n, n, T, period=8.0, seed=41)
    A0, B0 = O.random_subspace(n, n, R, seed=42)
    pol = tt.Informative(k=k, forced=(), beta=0.1, key0=21, replacement=False)
    res = tt.run_online(ph.kspace, A0[None], B0[None], 0.1, tt.Fixed(0.01), pol, clean=ph.clean)
    ref = O.online_run(ph.kspace, A0, B0, 0.1, ("fixed", 0.01),
                       {"kind": "informative", "k": k, "forced": [], "beta": 0.1, "key": (21, 0),
                        "replacement": False}, clean=ph.clean)
    for f in range(T):
        assert len(res.rows[f][0]) == k
        np.testing.assert_array_equal(res.rows[f][0], ref["rows"][f])
        assert rel(res.gamma[f, 0], ref["gamma"][f]) < 1e-4


@pytest.mark.parametrize("nslices,chunk", [(1, 3), (3, 100)])
def test_norm_cap_flags_match_oracle_norms(nslices, chunk):
    import paper_1609_04104_b200 as tt
    from paper_1609_04104_b200.phantom import cine_phantom

    n, R, T = 64, 6, 9
    ph = cine_phantom(n, n, T, period=8.0, seed=51)
    A0, B0 = O.random_subspace(n, n, R, seed=52)
    rows = [O.vd_rows(n, -1.0, 0.25, np.random.default_rng(f).random) for f in range(T)]
    rows[4] = np.empty(0, np.int64)  # an empty frame: no update, never flagged
    ref = O.online_run(ph.kspace, A0, B0, 0.1, ("fixed", 0.5), {"kind": "static", "rows": rows}, record_factors=True)
    na = np.array([np.linalg.norm(a) for a in ref["A"]])
    nb = np.array([np.linalg.norm(b) for b in ref["B"]])
    top = np.maximum(na, nb)
    u = np.unique(np.round(top, 6))
    cap = float(0.5 * (u[len(u) // 2 - 1] + u[len(u) // 2]))  # well between two distinct norms
    want = top > cap
    want[4] = False
    S = max(len(r) for r in rows)
    tab = np.full((T, nslices, S), -1, np.int64)
    cnt = np.zeros((T, nslices), np.int64)
    for f, r in enumerate(rows):
        tab[f, :, :len(r)] = r
        cnt[f] = len(r)
    ks = np.repeat(ph.kspace[:, None], nslices, axis=1)
    res = tt.run_online(ks, np.repeat(A0[None], nslices, 0), np.repeat(B0[None], nslices, 0), 0.1, tt.Fixed(0.5),
                        tt.StaticRows(tab, cnt), norm_cap=cap, chunk=chunk)
    assert res.norm_exceeded.shape == (T, nslices)
    assert 0 < want.sum() < T
    for s in range(nslices):
        np.testing.assert_array_equal(res.norm_exceeded[:, s], want)


def test_norm_cap_flags_entries_and_batch():
    """norm_cap on the entry-mask engine (flags from the factor history) against the oracle's post-update
    norms, and on batch mode (epochs = 1 equals the online run's flags)."""
    import paper_1609_04104_b200 as tt
    from paper_1609_04104_b200.phantom import cine_phantom

    n, R, T = 32, 4, 7
    ph = cine_phantom(n, n, T, period=8.0, seed=61)
    A0, B0 = O.random_subspace(n, n, R, seed=62)
    rng = np.random.default_rng(63)
    lists = [rng.permutation(rng.choice(n * n, int(0.3 * n * n), replace=False)) for _ in range(T)]
    lists[3] = np.empty(0, np.int64)
    ref = O.online_run_entries(ph.kspace, O.fft_cols(A0), O.fft_cols(B0), 0.1, ("fixed", 0.5),
                               {"kind": "static", "entries": lists}, record_factors=True)
    top = np.array([max(np.linalg.norm(a), np.linalg.norm(b)) for a, b in zip(ref["A"], ref["B"])])
    u = np.unique(np.round(top, 6))
    cap = float(0.5 * (u[len(u) // 2 - 1] + u[len(u) // 2]))
    want = top > cap
    want[3] = False
    S = max(len(x) for x in lists)
    tab = np.full((T, S), -1, np.int64)
    for f, x in enumerate(lists):
        tab[f, :len(x)] = x
    res = tt.run_online(ph.kspace, A0[None], B0[None], 0.1, tt.Fixed(0.5),
                        tt.StaticEntries(tab, np.array([len(x) for x in lists])), norm_cap=cap)
    assert 0 < want.sum() < T
    np.testing.assert_array_equal(res.norm_exceeded[:, 0], want)
    # batch mode, one epoch: the same flags as the online run
    rows = [O.vd_rows(n, -1.0, 0.25, np.random.default_rng(f).random) for f in range(T)]
    rt = np.stack(rows)
    on = tt.run_online(ph.kspace, A0[None], B0[None], 0.1, tt.Fixed(0.5), tt.StaticRows(rt[:, None, :],
                       np.full((T, 1), rt.shape[1])), norm_cap=cap)
    bt = tt.run_batch(ph.kspace, A0, B0, 0.1, tt.Fixed(0.5), rt, np.full(T, rt.shape[1]), norm_cap=cap)
    np.testing.assert_array_equal(bt.step_norm_exceeded, on.norm_exceeded[:, 0])
