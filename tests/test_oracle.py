"""CPU: the oracle restatement against the reference's own outputs
(tests/golden, written by oracle/make_golden.py) and against numpy's RNG.
No GPU, no /root/reference needed."""

import numpy as np
import pytest

from conftest import load_golden, rel
from oracle import tt_oracle as O


def step_case(g, name):
    p = f"{name}__"
    n1, n2, R, t, fourier, mask, hess = (int(v) for v in g[p + "meta"])
    lam, s1, s2, ab = (float(v) for v in g[p + "fparams"])
    step = ("hessian", s1, s2) if hess else ("fixed", s1)
    return dict(A=g[p + "A"], B=g[p + "B"], idx=g[p + "idx"], rows=g[p + "rows"], y=g[p + "y"], t=t,
                kind="fourier" if fourier else "entry", mask=mask, step=step, lam=lam, alpha_bar=ab,
                A_out=g[p + "A_out"], B_out=g[p + "B_out"], gamma=g[p + "gamma"], residual=g[p + "residual"],
                cost=float(g[p + "cost"]), mu=float(g[p + "mu"]), alpha_bar_out=float(g[p + "alpha_bar_out"]),
                t_out=int(g[p + "t_out"]))


STEP = load_golden("step_cases")
NAMES = [str(n) for n in STEP["names"]]


@pytest.mark.parametrize("name", NAMES)
def test_track_step_matches_reference_golden(name):
    c = step_case(STEP, name)
    out = O.track_step(c["A"], c["B"], c["t"], c["alpha_bar"], c["y"], c["idx"], c["kind"], c["lam"], c["step"],
                       power=True)
    assert rel(out["A"], c["A_out"]) < 1e-10
    assert rel(out["B"], c["B_out"]) < 1e-10
    assert rel(out["gamma"], c["gamma"]) < 1e-10
    assert rel(out["residual"], c["residual"]) < 1e-9
    assert out["cost"] == pytest.approx(c["cost"], rel=1e-10)
    assert out["mu"] == pytest.approx(c["mu"], rel=1e-12)
    assert out["t"] == c["t_out"]
    assert out["alpha_bar"] == pytest.approx(c["alpha_bar_out"], rel=1e-12)


@pytest.mark.parametrize("name", [n for n in NAMES if "hess" in n])
def test_closed_form_curvature_matches_power_method(name):
    c = step_case(STEP, name)
    A, B = c["A"], c["B"]
    a_pow = O.alpha_power(A, B, c["gamma"], c["idx"], c["kind"], c["lam"], c["t"])
    a_cf = O.alpha_closed(A, B, c["gamma"], c["idx"], c["kind"], c["lam"], c["t"])
    assert a_cf == pytest.approx(a_pow, rel=1e-6)
    assert a_cf >= a_pow * (1 - 1e-12)  # power iteration approaches from below


def test_ridge_matches_reference_golden():
    g = load_golden("solve_cases")
    for c in range(int(g["count"])):
        phi, y, lam = g[f"c{c}__phi"], g[f"c{c}__y"], float(g[f"c{c}__lam"])
        assert rel(O.ridge_svd(phi, y, lam), g[f"c{c}__gamma"]) < 1e-10
        assert rel(O.ridge_normal(phi, y, lam), g[f"c{c}__gamma"]) < 1e-9


def test_scores_match_reference_golden():
    g = load_golden("sampling_cases")
    for c in range(int(g["nscores"])):
        A, B, beta = g[f"s{c}__A"], g[f"s{c}__B"], float(g[f"s{c}__beta"])
        assert rel(O.row_probs(A, B.shape[0], beta), g[f"s{c}__rows"]) < 1e-13
        assert rel(O.entry_probs(A, B, beta), g[f"s{c}__entries"]) < 1e-13


def test_draws_match_reference_golden():
    g = load_golden("sampling_cases")
    for c in range(int(g["ndraws"])):
        p, k = g[f"d{c}__p"], int(g[f"d{c}__k"])
        forced = g[f"d{c}__forced"]
        key = tuple(int(v) for v in g[f"d{c}__key"])
        pos = 0
        for rep in range(3):
            om, used = O.draw_rows(p, k, forced, key, pos)
            pos += used
            np.testing.assert_array_equal(om, g[f"d{c}__omega{rep}"])


def test_vd_rows_match_reference_golden():
    g = load_golden("sampling_cases")
    for c in range(int(g["nvd"])):
        key = tuple(int(v) for v in g[f"v{c}__key"])
        gen = np.random.Generator(np.random.Philox(key=key[0] + (key[1] << 64)))
        rows = O.vd_rows(int(g[f"v{c}__n1"]), float(g[f"v{c}__alpha"]), float(g[f"v{c}__frac"]), gen.random)
        np.testing.assert_array_equal(rows, g[f"v{c}__rows"])


def test_values_match_reference_golden():
    g = load_golden("value_cases")
    assert rel(O.synth(g["A"], g["B"], g["gamma"]), g["synth"]) < 1e-13
    ra, rb = O.rebalance(g["A"], g["B"])
    assert rel(ra, g["rebal_A"]) < 1e-13 and rel(rb, g["rebal_B"]) < 1e-13
    assert rel(O.dft2(g["dft_in"]), g["dft_out"]) < 1e-13
    assert rel(O.dft2(g["dft_in"], inverse=True), g["idft_out"]) < 1e-13


def test_online_loop_matches_reference_golden():
    g = load_golden("loop_case")
    n, R, T, K, k0, k1 = (int(v) for v in g["meta"])
    out = O.online_run(g["kspace"], g["A0"], g["B0"], float(g["lam"]), ("fixed", 0.01),
                       {"kind": "informative", "k": K, "forced": g["forced"], "beta": 0.1, "key": (k0, k1)},
                       clean=g["clean"])
    for f in range(T):
        rows = g["rows"][f]
        np.testing.assert_array_equal(out["rows"][f], rows[rows >= 0])
        assert rel(out["gamma"][f], g["gamma"][f]) < 1e-9
    np.testing.assert_allclose(out["nmse"], g["nmse"], rtol=1e-9)
    assert rel(out["final"][0], g["A_final"]) < 1e-9


@pytest.mark.parametrize("key", [(5, 0), (3, 7), (2**64 - 1, 2**63)])
def test_philox_restatement_is_numpy_philox(key):
    gen = np.random.Generator(np.random.Philox(key=key[0] + (key[1] << 64)))
    want = gen.random(37)
    np.testing.assert_array_equal(O.philox_uniforms(key, 0, 37), want)
    # stream positions continue across calls
    want2 = gen.random(9)
    np.testing.assert_array_equal(O.philox_uniforms(key, 37, 9), want2)


def test_choice_restatement_is_numpy_choice():
    rng = np.random.default_rng(0)
    for trial in range(20):
        n = int(rng.integers(2, 300))
        p = rng.random(n) ** 4
        p /= p.sum()
        key = (int(rng.integers(1 << 62)), trial)
        gen = np.random.Generator(np.random.Philox(key=key[0] + (key[1] << 64)))
        size = int(rng.integers(1, 100))
        want = gen.choice(n, size=size, replace=True, p=p)
        got = O.choice_with_replacement(p, size, O.philox_uniforms(key, 0, size))
        np.testing.assert_array_equal(got, want)


def test_entries_loop_equals_rows_loop_on_kspace_factors():
    """online_run_entries (EntryMask on (F_x A, F_y B), run_adaptive's entries mode) equals the FourierMask
    row loop when the entry lists are whole rows (test_mri.py:258-286 at the loop level)."""
    rng = np.random.default_rng(3)
    n, R, T = 12, 3, 4
    ks = rng.standard_normal((T, n, n)) + 1j * rng.standard_normal((T, n, n))
    A, B = O.random_subspace(n, n, R, seed=4)
    rows = [np.sort(rng.choice(n, 5, replace=False)) for _ in range(T)]
    a = O.online_run(ks, A, B, 0.2, ("fixed", 0.02), {"kind": "static", "rows": rows}, record_factors=True)
    ents = [(r[:, None] * n + np.arange(n)[None, :]).ravel() for r in rows]
    b = O.online_run_entries(ks, O.fft_cols(A), O.fft_cols(B), 0.2, ("fixed", 0.02),
                             {"kind": "static", "entries": ents}, record_factors=True)
    for f in range(T):
        np.testing.assert_allclose(b["gamma"][f], a["gamma"][f], rtol=1e-10, atol=1e-12)
        np.testing.assert_allclose(b["recon"][f], a["recon"][f], rtol=1e-10, atol=1e-12)
        np.testing.assert_allclose(b["A"][f], O.fft_cols(a["A"][f]), rtol=1e-10, atol=1e-12)
