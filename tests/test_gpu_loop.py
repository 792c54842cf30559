"""GPU parity of the device-resident online loop (engine / run_online)
against the reference-built golden loop and the oracle at BASELINE sizes:
per-frame gamma and factors within 1e-4 relative (teacher-forced state),
free-running NRMSE trajectory within 1e-3 absolute with oracle masks fed in,
and bit-exact informative masks when the probabilities agree."""

import numpy as np
import pytest

from conftest import load_golden, rel
from oracle import tt_oracle as O

pytestmark = pytest.mark.gpu


def test_informative_loop_matches_reference_golden():
    import paper_1609_04104_b200 as tt

    g = load_golden("loop_case")
    n, R, T, K, k0, k1 = (int(v) for v in g["meta"])
    pol = tt.Informative(k=K, forced=tuple(int(v) for v in g["forced"]), beta=0.1, key0=k0, key1=k1)
    res = tt.run_online(g["kspace"], g["A0"][None], g["B0"][None], float(g["lam"]), tt.Fixed(0.01), pol,
                        clean=g["clean"])
    for f in range(T):
        rows = g["rows"][f]
        np.testing.assert_array_equal(res.rows[f][0], rows[rows >= 0])
        assert rel(res.gamma[f, 0], g["gamma"][f]) < 1e-4
    assert np.max(np.abs(np.sqrt(res.nmse[:, 0]) - np.sqrt(g["nmse"]))) < 1e-3
    assert rel(res.final_A[0], g["A_final"]) < 1e-4


@pytest.mark.parametrize("cfg", [
    dict(n=128, R=10, lam=0.1, T=16, period=16.0, kind="vd", frac=0.25),      # config 1 shape
    dict(n=256, R=20, lam=0.05, T=12, period=20.0, kind="inf", K=64),         # config 2 shape
])
def test_trajectory_matches_oracle(cfg):
    import paper_1609_04104_b200 as tt
    from paper_1609_04104_b200.phantom import cine_phantom

    n, R, T, lam = cfg["n"], cfg["R"], cfg["T"], cfg["lam"]
    ph = cine_phantom(n, n, T, period=cfg["period"], seed=3)
    A0, B0 = O.random_subspace(n, n, R, seed=4)
    if cfg["kind"] == "vd":
        gen = np.random.Generator(np.random.Philox(key=11))
        rows = [O.vd_rows(n, -1.0, cfg["frac"], gen.random) for _ in range(T)]
        pol_o = {"kind": "static", "rows": rows}
    else:
        forced = list(range(8)) + list(range(n - 8, n))
        pol_o = {"kind": "informative", "k": cfg["K"], "forced": forced, "beta": 0.1, "key": (2024, 0)}
    ref = O.online_run(ph.kspace, A0, B0, lam, ("fixed", 0.01), pol_o, clean=ph.clean, record_factors=True)
    # feed the oracle's masks (BASELINE: "otherwise oracle masks are fed in")
    S = max(len(r) for r in ref["rows"])
    tab = np.full((T, 1, S), -1, np.int64)
    cnt = np.zeros((T, 1), np.int64)
    for f, r in enumerate(ref["rows"]):
        tab[f, 0, :len(r)] = r
        cnt[f, 0] = len(r)
    res = tt.run_online(ph.kspace, A0[None], B0[None], lam, tt.Fixed(0.01), tt.StaticRows(tab, cnt), clean=ph.clean)
    for f in range(T):
        assert rel(res.gamma[f, 0], ref["gamma"][f]) < 1e-4, f
    assert rel(res.final_A[0], ref["A"][-1]) < 1e-4
    assert np.max(np.abs(np.sqrt(res.nmse[:, 0]) - np.sqrt(np.array(ref["nmse"])))) < 1e-3
    # reconstructions themselves
    assert rel(res.recon[-1, 0], ref["recon"][-1]) < 1e-4


def test_teacher_forced_state_per_frame():
    """Each frame restarted from the oracle's state: gamma/A/B per frame."""
    import paper_1609_04104_b200 as tt
    from paper_1609_04104_b200.phantom import cine_phantom

    n, R, T, lam = 256, 20, 6, 0.05
    ph = cine_phantom(n, n, T, period=20.0, seed=8)
    A0, B0 = O.random_subspace(n, n, R, seed=9)
    forced = list(range(8)) + list(range(n - 8, n))
    ref = O.online_run(ph.kspace, A0, B0, lam, ("fixed", 0.01),
                       {"kind": "informative", "k": 64, "forced": forced, "beta": 0.1, "key": (5, 0)},
                       clean=ph.clean, record_factors=True)
    A, B = A0, B0
    for f in range(T):
        rows = ref["rows"][f]
        st = tt.TrackerState(tt.TensorSubspace((A, B)), tt.StepConfig(lam, R, tt.Fixed(0.01)), t=1 + f)
        idx = tt.rows_to_entries(rows, n)
        new, rep = tt.track_step(st, tt.MeasurementBatch(ph.kspace[f][rows, :].ravel(), tt.FourierMask((n, n), idx)))
        assert rel(rep.gamma, ref["gamma"][f]) < 1e-4
        assert rel(new.subspace.factors[0], ref["A"][f]) < 1e-4
        assert rel(new.subspace.factors[1], ref["B"][f]) < 1e-4
        A, B = ref["A"][f], ref["B"][f]


def test_batched_slices_equal_single_slice_runs():
    """C3-style batch: every slice of a batched launch equals its own run."""
    import paper_1609_04104_b200 as tt
    from paper_1609_04104_b200.phantom import cine_phantom

    n, R, T, ns = 64, 6, 5, 3
    ks = np.stack([cine_phantom(n, n, T, 8.0, seed=1, slice_index=s).kspace for s in range(ns)], axis=1)
    A0 = np.stack([O.random_subspace(n, n, R, seed=20 + s)[0] for s in range(ns)])
    B0 = np.stack([O.random_subspace(n, n, R, seed=20 + s)[1] for s in range(ns)])
    pol = tt.Informative(k=13, forced=(0,), beta=0.1, key0=9)
    batched = tt.run_online(ks, A0, B0, 0.05, tt.Fixed(0.01), pol)
    for s in range(ns):
        pol_s = tt.Informative(k=13, forced=(0,), beta=0.1, key0=9, key1=s)
        single = tt.run_online(ks[:, s], A0[s:s + 1], B0[s:s + 1], 0.05, tt.Fixed(0.01), pol_s)
        np.testing.assert_array_equal(batched.gamma[:, s], single.gamma[:, 0])
        for f in range(T):
            np.testing.assert_array_equal(batched.rows[f][s], single.rows[f][0])


def test_warm_up_protocol_then_informative_stream():
    """experiment.run_adaptive order: 5 full frames x 20 epochs with rebalance, t -> 101,
    then informative streaming frames; vs the oracle restatement of _warm_up."""
    import paper_1609_04104_b200 as tt
    from paper_1609_04104_b200.phantom import cine_phantom

    n, R, T, W, E, lam = 64, 6, 9, 5, 20, 0.1
    ph = cine_phantom(n, n, T, period=8.0, seed=21)
    A0, B0 = O.random_subspace(n, n, R, seed=22)
    Aw, Bw, t, ab = O.warm_up(ph.kspace[:W], A0, B0, lam, ("fixed", 0.01), E)
    assert t == 1 + W * E
    forced = [0, 1, n - 1]
    ref = O.online_run(ph.kspace[W:], Aw, Bw, lam, ("fixed", 0.01),
                       {"kind": "informative", "k": 16, "forced": forced, "beta": 0.1, "key": (3, 0)},
                       clean=ph.clean[W:], t0=t)
    res = tt.run_online(ph.kspace, A0[None], B0[None], lam, tt.Fixed(0.01),
                        tt.Informative(k=16, forced=tuple(forced), beta=0.1, key0=3), clean=ph.clean,
                        warm_frames=W, warm_epochs=E)
    for f in range(T - W):
        np.testing.assert_array_equal(res.rows[f][0], ref["rows"][f])
        assert rel(res.gamma[f, 0], ref["gamma"][f]) < 1e-4
    assert np.max(np.abs(np.sqrt(res.nmse[:, 0]) - np.sqrt(ref["nmse"]))) < 1e-3


@pytest.mark.parametrize("chunk", [1, 7, 1000])
def test_pipelined_run_online_is_chunk_invariant(chunk):
    """run_online's block pipelining (uploads / tracking / downloads overlapped) gives the
    same bits for any block size, from pinned, pageable and device inputs."""
    import torch
    import paper_1609_04104_b200 as tt
    from paper_1609_04104_b200.phantom import cine_phantom

    n, R, T = 64, 6, 23
    ph = cine_phantom(n, n, T, period=8.0, seed=31)
    A0, B0 = O.random_subspace(n, n, R, seed=32)
    pol = tt.Informative(k=16, forced=(0, 1, n - 1), beta=0.1, key0=5)
    ref = tt.run_online(ph.kspace, A0[None], B0[None], 0.1, tt.Fixed(0.01), pol, chunk=T)
    for src in (torch.from_numpy(ph.kspace.astype(np.complex64)).pin_memory(), ph.kspace,
                torch.from_numpy(ph.kspace.astype(np.complex64)).cuda()):
        got = tt.run_online(src, A0[None], B0[None], 0.1, tt.Fixed(0.01), pol, chunk=chunk)
        np.testing.assert_array_equal(got.gamma, ref.gamma)
        np.testing.assert_array_equal(got.recon, ref.recon)
        np.testing.assert_array_equal(got.final_A, ref.final_A)
        for f in range(T):
            np.testing.assert_array_equal(got.rows[f][0], ref.rows[f][0])


def test_online_mask_and_budget_rows():
    """run_adaptive's mask/budget rows (experiment.py:495-510) from a device run: the budget's
    expected count equals sum_i 1 - (1 - p_i)^K under each frame's (oracle) row scores."""
    import paper_1609_04104_b200 as tt
    from paper_1609_04104_b200 import reports
    from paper_1609_04104_b200.phantom import cine_phantom

    n, R, T, K = 64, 6, 6, 16
    ph = cine_phantom(n, n, T, period=8.0, seed=61)
    A0, B0 = O.random_subspace(n, n, R, seed=62)
    pol = tt.Informative(k=K, forced=(0,), beta=0.1, key0=4)
    res = tt.run_online(ph.kspace, A0[None], B0[None], 0.1, tt.Fixed(0.01), pol, keep_history=True)
    ref = O.online_run(ph.kspace, A0, B0, 0.1, ("fixed", 0.01),
                       {"kind": "informative", "k": K, "forced": [0], "beta": 0.1, "key": (4, 0)})
    mrows = reports.online_mask_rows(res, t0=5)
    assert mrows[0][0] == 5 and len(mrows) == sum(len(r[0]) for r in res.rows)
    brows = reports.online_budget_rows(res, A0, B0, K, beta=0.1, t0=5)
    for f, (t, k, size, expected) in enumerate(brows):
        p = ref["probs"][f]
        assert t == 5 + f and k == K and size == len(ref["rows"][f])
        assert expected == pytest.approx(float(np.sum(1.0 - (1.0 - p) ** K)), rel=1e-5)


@pytest.mark.parametrize("epochs,reshuffle", [(1, False), (3, True), (2, False)])
def test_batch_mode_matches_oracle(epochs, reshuffle):
    """tracker.run / run_tracking batch mode: epochs over the same row-mask data, rebalance between
    epochs, rng.permutation reshuffles (the caller's generator, stepped as the reference does), then
    the re-projection onto the final subspace; per-step gammas and final images vs the oracle."""
    import paper_1609_04104_b200 as tt
    from paper_1609_04104_b200.phantom import cine_phantom

    n, R, T, lam = 64, 6, 8, 0.1
    ph = cine_phantom(n, n, T, period=8.0, seed=71)
    A0, B0 = O.random_subspace(n, n, R, seed=72)
    rng = np.random.default_rng(73)
    rows = [np.sort(rng.choice(n, 16, replace=False)) for _ in range(T)]
    tab = np.stack(rows)
    ref = O.batch_run(ph.kspace, A0, B0, lam, ("fixed", 0.01), rows, epochs, rng=np.random.default_rng(9),
                      reshuffle=reshuffle)
    got = tt.run_batch(ph.kspace, A0, B0, lam, tt.Fixed(0.01), tab, np.full(T, 16), epochs=epochs,
                       rng=np.random.default_rng(9), reshuffle=reshuffle)
    for a, b in zip(got.orders, ref["orders"]):
        np.testing.assert_array_equal(a, b)
    for k, rep in enumerate(ref["reports"]):
        assert rel(got.step_gamma[k], rep["gamma"]) < 1e-4, k
    for f in range(T):
        assert rel(got.gamma[f], ref["gamma"][f]) < 1e-4, f
        assert rel(got.recon[f], ref["recon"][f]) < 1e-4, f
    assert got.t == ref["final"][2]


@pytest.mark.parametrize("chunk", [1000, 3])
def test_hessian_step_trajectory_matches_oracle(chunk):
    """HessianBound through the device loop: alpha_t (closed form of the power method), the running
    alpha_bar carried inside the kernel and across launches, mu_t = 1/alpha_bar, per-frame gamma and
    the NRMSE trajectory vs the oracle with oracle masks fed in."""
    import paper_1609_04104_b200 as tt
    from paper_1609_04104_b200.phantom import cine_phantom

    n, R, T, lam = 128, 10, 10, 0.1
    ph = cine_phantom(n, n, T, period=8.0, seed=81)
    A0, B0 = O.random_subspace(n, n, R, seed=82)
    forced = list(range(4)) + list(range(n - 4, n))
    ref = O.online_run(ph.kspace, A0, B0, lam, ("hessian", 1e-3, 1e6),
                       {"kind": "informative", "k": 32, "forced": forced, "beta": 0.1, "key": (6, 0)},
                       clean=ph.clean)
    S = max(len(r) for r in ref["rows"])
    tab = np.full((T, 1, S), -1, np.int64)
    cnt = np.zeros((T, 1), np.int64)
    for f, r in enumerate(ref["rows"]):
        tab[f, 0, :len(r)] = r
        cnt[f, 0] = len(r)
    res = tt.run_online(ph.kspace, A0[None], B0[None], lam, tt.HessianBound(1e-3, 1e6), tt.StaticRows(tab, cnt),
                        clean=ph.clean, chunk=chunk)
    for f in range(T):
        assert res.mu[f, 0] == pytest.approx(ref["mu"][f], rel=1e-5), f
        assert rel(res.gamma[f, 0], ref["gamma"][f]) < 1e-4, f
    assert np.max(np.abs(np.sqrt(res.nmse[:, 0]) - np.sqrt(np.array(ref["nmse"])))) < 1e-3


def test_run_online_kspace_reconstruction_domain():
    """recon_domain="kspace" returns Ah diag(gamma) Bh^T (run_adaptive's .kspace record, no inverse FFT):
    the unitary 2-D DFT of the image-domain reconstruction, with the same NMSE against the clean frames."""
    import paper_1609_04104_b200 as tt
    from paper_1609_04104_b200.phantom import cine_phantom

    n, R, T = 64, 6, 7
    ph = cine_phantom(n, n, T, period=8.0, seed=71)
    A0, B0 = O.random_subspace(n, n, R, seed=72)
    pol = tt.Informative(k=16, forced=(0,), beta=0.1, key0=73)
    im = tt.run_online(ph.kspace, A0[None], B0[None], 0.1, tt.Fixed(0.01), pol, clean=ph.clean)
    ks = tt.run_online(ph.kspace, A0[None], B0[None], 0.1, tt.Fixed(0.01), pol, clean=ph.clean,
                       recon_domain="kspace")
    np.testing.assert_array_equal(ks.gamma, im.gamma)
    for f in range(T):
        assert rel(ks.recon[f, 0], O.dft2(im.recon[f, 0].astype(np.complex128))) < 1e-5
    np.testing.assert_allclose(ks.nmse, im.nmse, rtol=1e-4)


@pytest.mark.parametrize("transfer", ["upload", "zero-copy"])
def test_run_online_truth_transfer_modes_are_bit_identical(transfer):
    """The row kernels reading a page-locked host truth in place (only the sampled rows cross the host link)
    give the same bits as the uploaded truth and the device-resident truth."""
    import torch

    import paper_1609_04104_b200 as tt
    from paper_1609_04104_b200.phantom import cine_phantom

    n, R, T, ns = 64, 6, 9, 3
    ks = np.stack([cine_phantom(n, n, T, period=8.0, seed=80 + s).kspace for s in range(ns)], axis=1)
    A0 = np.stack([O.random_subspace(n, n, R, seed=90 + s)[0] for s in range(ns)])
    B0 = np.stack([O.random_subspace(n, n, R, seed=90 + s)[1] for s in range(ns)])
    pol = tt.Informative(k=16, forced=(0,), beta=0.1, key0=5)
    ref = tt.run_online(torch.from_numpy(ks.astype(np.complex64)).cuda(), A0, B0, 0.1, tt.Fixed(0.01), pol)
    pinned = torch.from_numpy(ks.astype(np.complex64)).pin_memory()
    got = tt.run_online(pinned, A0, B0, 0.1, tt.Fixed(0.01), pol, truth_transfer=transfer, chunk=4)
    np.testing.assert_array_equal(got.gamma, ref.gamma)
    np.testing.assert_array_equal(got.recon, ref.recon)
    for f in range(T):
        for s in range(ns):
            np.testing.assert_array_equal(got.rows[f][s], ref.rows[f][s])
    # with the warm-up protocol (its full frames are made resident for the epochs)
    ref_w = tt.run_online(torch.from_numpy(ks.astype(np.complex64)).cuda(), A0, B0, 0.1, tt.Fixed(0.01), pol,
                          warm_frames=2, warm_epochs=3)
    got_w = tt.run_online(pinned, A0, B0, 0.1, tt.Fixed(0.01), pol, truth_transfer=transfer, warm_frames=2,
                          warm_epochs=3)
    np.testing.assert_array_equal(got_w.gamma, ref_w.gamma)
    np.testing.assert_array_equal(got_w.recon, ref_w.recon)
    with pytest.raises(ValueError):
        tt.run_online(ks, A0, B0, 0.1, tt.Fixed(0.01), pol, truth_transfer="zero-copy")  # pageable
