"""GPU parity: one online step through the drop-in API (track_step -> C ABI
-> fused row kernel / generic index kernels) against the reference's golden
outputs and the oracle on seeded inputs. fp32 data; tolerance 1e-4 relative
(norm-wise) for gamma, A, B (BASELINE north_star)."""

import numpy as np
import pytest

from conftest import load_golden, rel
from oracle import tt_oracle as O

pytestmark = pytest.mark.gpu
TOL = 1e-4

STEP = load_golden("step_cases")
NAMES = [str(n) for n in STEP["names"]]


def _case(name):
    from test_oracle import step_case

    return step_case(STEP, name)


def _run_api(c):
    import paper_1609_04104_b200 as tt

    step = tt.Fixed(c["step"][1]) if c["step"][0] == "fixed" else tt.HessianBound(c["step"][1], c["step"][2])
    cfg = tt.StepConfig(lam=c["lam"], rank=c["A"].shape[1], step=step)
    st = tt.TrackerState(tt.TensorSubspace((c["A"], c["B"])), cfg, t=c["t"], alpha_bar=c["alpha_bar"])
    n1, n2 = c["A"].shape[0], c["B"].shape[0]
    Desc = tt.FourierMask if c["kind"] == "fourier" else tt.EntryMask
    desc = Desc((n1, n2), c["idx"])
    return tt.track_step(st, tt.MeasurementBatch(c["y"], desc)), desc


@pytest.mark.parametrize("name", NAMES)
def test_track_step_matches_reference_golden(name):
    c = _case(name)
    (new, rep), desc = _run_api(c)
    if c["mask"] == 0:
        assert desc.row_lines is not None  # routed to the fused row-mask kernel
    A2, B2 = new.subspace.factors
    assert rel(A2, c["A_out"]) < TOL
    assert rel(B2, c["B_out"]) < TOL
    assert rel(rep.gamma, c["gamma"]) < TOL
    if c["residual"].size:
        assert rel(rep.residual, c["residual"]) < TOL
    assert rep.instantaneous_cost == pytest.approx(c["cost"], rel=TOL)
    assert rep.step_size == pytest.approx(c["mu"], rel=TOL)
    assert new.t == c["t_out"] and rep.t == c["t"]
    assert new.alpha_bar == pytest.approx(c["alpha_bar_out"], rel=TOL)


def _random_case(seed, n1, n2, R, S, lam, t, noise=0.05):
    rng = np.random.default_rng(seed)
    A = (rng.standard_normal((n1, R)) + 1j * rng.standard_normal((n1, R))) / np.sqrt(2 * n1)
    B = (rng.standard_normal((n2, R)) + 1j * rng.standard_normal((n2, R))) / np.sqrt(2 * n2)
    rows = rng.choice(n1, size=S, replace=False)
    idx = O.rows_to_entries(rows, n2)
    Ah, Bh = O.measurement_factors(A, B, "fourier")
    g = rng.standard_normal(R) + 1j * rng.standard_normal(R)
    y = (Ah[idx[:, 0]] * Bh[idx[:, 1]]) @ g + noise * (rng.standard_normal(len(idx)) + 1j * rng.standard_normal(len(idx)))
    return A, B, rows, idx, y


@pytest.mark.parametrize("shape", [(128, 128, 10, 32, 0.1), (256, 256, 20, 64, 0.05), (256, 256, 16, 52, 0.05),
                                   (64, 96, 4, 7, 0.3), (1024, 1024, 32, 128, 0.1), (200, 256, 12, 50, 0.2),
                                   (512, 512, 64, 64, 0.1)])
@pytest.mark.parametrize("hess", [False, True])
def test_row_step_matches_oracle_at_config_sizes(shape, hess):
    import paper_1609_04104_b200 as tt

    n1, n2, R, S, lam = shape
    A, B, rows, idx, y = _random_case(n1 * 7 + R, n1, n2, R, S, lam, 9)
    step = ("hessian", 1e-3, 1e9) if hess else ("fixed", 0.01)
    want = O.track_step(A, B, 9, 2.0 if hess else 0.0, y, idx, "fourier", lam, step, power=False)
    st = tt.TrackerState(tt.TensorSubspace((A, B)),
                         tt.StepConfig(lam, R, tt.HessianBound(1e-3, 1e9) if hess else tt.Fixed(0.01)),
                         t=9, alpha_bar=2.0 if hess else 0.0)
    new, rep = tt.track_step(st, tt.MeasurementBatch(y, tt.FourierMask((n1, n2), idx)))
    assert rel(rep.gamma, want["gamma"]) < TOL
    A2, B2 = new.subspace.factors
    assert rel(A2, want["A"]) < TOL and rel(B2, want["B"]) < TOL
    assert rep.instantaneous_cost == pytest.approx(want["cost"], rel=TOL)
    assert rep.step_size == pytest.approx(want["mu"], rel=TOL)
    assert rel(rep.residual, want["residual"]) < 1e-3


def test_entry_mask_equals_fourier_mask_on_transformed_factors():
    """test_mri.py:258-286 analogue: EntryMask on (F A, F B) == FourierMask on (A, B)."""
    import paper_1609_04104_b200 as tt

    A, B, rows, idx, y = _random_case(3, 32, 24, 3, 8, 0.3, 2)
    cfg = tt.StepConfig(0.3, 3, tt.Fixed(0.02))
    sf, rf = tt.track_step(tt.TrackerState(tt.TensorSubspace((A, B)), cfg), tt.MeasurementBatch(y, tt.FourierMask((32, 24), idx)))
    Ah, Bh = O.measurement_factors(A, B, "fourier")
    se, re_ = tt.track_step(tt.TrackerState(tt.TensorSubspace((Ah, Bh)), cfg), tt.MeasurementBatch(y, tt.EntryMask((32, 24), idx)))
    assert rel(rf.gamma, re_.gamma) < 1e-5
    assert rel(O.fft_cols(sf.subspace.factors[0]), se.subspace.factors[0]) < 1e-5


def test_empty_batch_advances_time_only():
    import paper_1609_04104_b200 as tt

    rng = np.random.default_rng(14)
    st = tt.init_state(tt.StepConfig(0.5, 2, tt.Fixed(0.05)), (4, 4), rng)
    new, rep = tt.track_step(st, tt.MeasurementBatch(np.zeros(0, complex), tt.EntryMask((4, 4), np.empty((0, 2), int))))
    assert new.t == st.t + 1
    for f, g in zip(st.subspace.factors, new.subspace.factors):
        np.testing.assert_array_equal(f, g)
    assert rep.gamma.shape == (2,) and rep.residual.size == 0 and rep.step_size == 0.0
    A, B = st.subspace.factors
    assert rep.instantaneous_cost == pytest.approx(0.5 * 0.5 * (np.linalg.norm(A) ** 2 + np.linalg.norm(B) ** 2), rel=1e-6)


def test_descriptor_shape_mismatch_raises():
    import paper_1609_04104_b200 as tt

    st = tt.init_state(tt.StepConfig(0.5, 2, tt.Fixed(0.05)), (4, 4), np.random.default_rng(17))
    with pytest.raises(ValueError):
        tt.track_step(st, tt.MeasurementBatch(np.zeros(1, complex), tt.EntryMask((5, 5), [[0, 0]])))


def test_bit_identical_repeat_runs():
    import paper_1609_04104_b200 as tt

    def traj():
        rng = np.random.default_rng(99)
        st = tt.init_state(tt.StepConfig(0.3, 4, tt.Fixed(0.02)), (64, 48), rng)
        for t in range(6):
            rows = rng.choice(64, 12, replace=False)
            idx = tt.rows_to_entries(rows, 48)
            y = rng.standard_normal(len(idx)) + 1j * rng.standard_normal(len(idx))
            st, _ = tt.track_step(st, tt.MeasurementBatch(y, tt.FourierMask((64, 48), idx)))
        for t in range(3):
            idx = np.argwhere(rng.random((64, 48)) < 0.3)
            y = rng.standard_normal(len(idx)) + 1j * rng.standard_normal(len(idx))
            st, _ = tt.track_step(st, tt.MeasurementBatch(y, tt.FourierMask((64, 48), idx)))
        return st.subspace.factors

    a, b = traj(), traj()
    for f, g in zip(a, b):
        np.testing.assert_array_equal(f, g)


def test_hessian_step_size_bound():
    """test_tracker.py:264-273: mu <= 1/(c_floor t)."""
    import paper_1609_04104_b200 as tt

    rng = np.random.default_rng(16)
    st = tt.init_state(tt.StepConfig(0.5, 2, tt.HessianBound(0.5, 1e6)), (5, 5), rng)
    idx = np.argwhere(rng.random((5, 5)) < 0.6)
    y = rng.standard_normal(len(idx)) + 1j * rng.standard_normal(len(idx))
    for _ in range(4):
        st, rep = tt.track_step(st, tt.MeasurementBatch(y, tt.EntryMask((5, 5), idx)))
        assert rep.step_size <= 1.0 / (0.5 * rep.t) + 1e-12


def test_solve_gamma_matches_reference_golden():
    import paper_1609_04104_b200 as tt

    g = load_golden("solve_cases")
    for c in range(int(g["count"])):
        got = tt.solve_gamma(g[f"c{c}__phi"], g[f"c{c}__y"], float(g[f"c{c}__lam"]))
        assert rel(got, g[f"c{c}__gamma"]) < 1e-9
    assert np.array_equal(tt.solve_gamma(np.zeros((0, 4)), np.zeros(0), 1.0), np.zeros(4))


@pytest.mark.parametrize("name", [n for n in NAMES if n != "empty"])
def test_standalone_gradient_cost_and_curvature(name):
    """factor_gradient / instantaneous_cost / hessian_bound as standalone calls vs the oracle
    (and the reference's power-method alpha from the golden case, within its tolerance)."""
    import paper_1609_04104_b200 as tt

    c = _case(name)
    A, B = c["A"], c["B"]
    n1, n2 = A.shape[0], B.shape[0]
    Desc = tt.FourierMask if c["kind"] == "fourier" else tt.EntryMask
    desc = Desc((n1, n2), c["idx"])
    sub = tt.TensorSubspace((A, B))
    gam, res = c["gamma"], c["residual"]
    got = tt.factor_gradient(sub, gam, desc, res, c["lam"], c["t"])
    dA, dB = O.data_terms(A, B, gam, c["idx"], res, c["kind"])
    want = [(c["lam"] / c["t"]) * A - dA, (c["lam"] / c["t"]) * B - dB]
    for gg, ww in zip(got, want):
        assert rel(gg, ww) < 1e-5
    cost = tt.instantaneous_cost(sub, tt.MeasurementBatch(c["y"], desc), c["lam"], c["t"], gam)
    assert cost == pytest.approx(c["cost"], rel=1e-5)
    alpha = tt.hessian_bound(sub, gam, desc, c["lam"], c["t"])
    assert alpha == pytest.approx(O.alpha_closed(A, B, gam, c["idx"], c["kind"], c["lam"], c["t"]), rel=1e-5)
    assert alpha == pytest.approx(O.alpha_power(A, B, gam, c["idx"], c["kind"], c["lam"], c["t"]), rel=1e-5)
    assert tt.hessian_bound(sub, np.zeros_like(gam), desc, 0.6, 3) == pytest.approx(0.2)
    assert tt.hessian_bound(sub, gam, desc, c["lam"], c["t"], c_floor=1e6, c_cap=1e7) == 1e6


def test_empirical_cost_and_gradient():
    """empirical_cost / empirical_cost_gradient (tracker.py:414-453): per batch the ridge re-solve, the
    cost at tau = 1..T, and the partial factor gradient, averaged; against the same sums from the
    oracle (ridge by SVD, explicit residual and data terms)."""
    import paper_1609_04104_b200 as tt

    rng = np.random.default_rng(3)
    n1, n2, R, lam = 16, 12, 3, 0.2
    A, B = O.random_subspace(n1, n2, R, seed=5)
    batches, ref_cost = [], 0.0
    ref_g = [np.zeros_like(A), np.zeros_like(B)]
    for tau in range(1, 5):
        kind = "fourier" if tau % 2 else "entry"
        rows = np.sort(rng.choice(n1, 5, replace=False))
        idx = O.rows_to_entries(rows, n2) if kind == "fourier" else np.stack(
            [rng.choice(n1, 40), rng.choice(n2, 40)], axis=1)
        idx = np.unique(idx, axis=0) if kind == "entry" else idx
        y = rng.standard_normal(len(idx)) + 1j * rng.standard_normal(len(idx))
        Desc = tt.FourierMask if kind == "fourier" else tt.EntryMask
        batches.append(tt.MeasurementBatch(y, Desc((n1, n2), idx)))
        phi = O.phi_matrix(A, B, idx, kind)
        g = O.ridge_svd(phi, y, lam)
        e = y - phi @ g
        ref_cost += 0.5 * np.linalg.norm(e) ** 2 + 0.5 * (lam / tau) * (np.linalg.norm(A) ** 2 + np.linalg.norm(B) ** 2)
        dA, dB = O.data_terms(A, B, g, idx, e, kind)
        ref_g[0] += (lam / tau) * A - dA
        ref_g[1] += (lam / tau) * B - dB
    st = tt.TrackerState(tt.TensorSubspace((A, B)), tt.StepConfig(lam=lam, rank=R))
    assert tt.empirical_cost(st, batches) == pytest.approx(ref_cost / 4, rel=1e-5)
    for got, want in zip(tt.empirical_cost_gradient(st, batches), ref_g):
        assert rel(got, want / 4) < 1e-4
    with pytest.raises(ValueError):
        tt.empirical_cost(st, [])
