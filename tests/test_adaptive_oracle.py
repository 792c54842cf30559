"""CPU: the oracle's run_adaptive schedule (variable-density rows until the switch frame, then informative
draws with or without replacement, experiment.py:462-510, sampler.py:146-169) against the reference's own
run_adaptive outputs (tests/golden/adaptive_*.npz, written by oracle/make_golden_adaptive.py)."""

import numpy as np
import pytest

from conftest import load_golden, rel
from oracle import tt_oracle as O

NAMES = ["switch_wr", "switch_wor", "wor_nowarm"]


def case(name):
    g = load_golden("adaptive_" + name)
    n, R, T, W, E, switch, k, repl, seed, pos0, nvd = (int(v) for v in g["meta"])
    return g, dict(n=n, R=R, T=T, W=W, E=E, switch=switch, k=k, repl=bool(repl), seed=seed, pos0=pos0, nvd=nvd,
                   lam=float(g["lam"]), mu=float(g["mu"]), fraction=float(g["fraction"]))


@pytest.mark.parametrize("name", NAMES)
def test_oracle_schedule_matches_reference_run_adaptive(name):
    g, c = case(name)
    ks = g["kspace"].astype(np.complex128)
    A, B = O.fft_cols(g["Ah0"], inverse=True), O.fft_cols(g["Bh0"], inverse=True)
    W = c["W"]
    if W:
        A, B, t1, _ = O.warm_up(ks[:W], A, B, c["lam"], ("fixed", c["mu"]), c["E"])
        assert t1 == 1 + W * c["E"]
    else:
        t1 = 1
    clean = np.stack([O.dft2(ks[t], inverse=True) for t in range(W, c["T"])])
    pol = {"kind": "schedule", "vd_frames": c["nvd"], "alpha": -1.0, "fraction": c["fraction"], "k": c["k"],
           "forced": [0], "beta": 0.1, "key": (c["seed"], 0), "position": c["pos0"], "replacement": c["repl"]}
    out = O.online_run(ks[W:], A, B, c["lam"], ("fixed", c["mu"]), pol, clean=clean, t0=t1)
    for f in range(c["T"] - W):
        want = g["rows"][f, :g["counts"][f]]
        np.testing.assert_array_equal(np.sort(out["rows"][f]), want)
        if f >= c["nvd"] and not c["repl"]:
            assert len(want) == c["k"]  # without replacement: exactly k distinct rows
        assert rel(out["gamma"][f], g["gamma"][f]) < 1e-9
    np.testing.assert_allclose(out["nmse"], g["nmse"], rtol=1e-9, atol=1e-12)
    assert rel(O.fft_cols(out["final"][0]), g["Af"]) < 1e-9
    assert rel(O.fft_cols(out["final"][1]), g["Bf"]) < 1e-9


def test_wor_draw_consumes_one_uniform_per_draw():
    p = np.random.default_rng(1).random(50)
    p /= p.sum()
    rows, used = O.draw_rows_wor(p, 12, [0, 7], (5, 0), 3)
    assert used == 10 and len(rows) == 12 and len(np.unique(rows)) == 12
    gen = np.random.Generator(np.random.Philox(key=5))
    gen.random(3)
    w = p.copy()
    w[[0, 7]] = 0.0
    want = O.draw_without_replacement(w, 10, gen.random)
    np.testing.assert_array_equal(rows, np.union1d([0, 7], want))
    with pytest.raises(ValueError):
        O.draw_rows_wor(p, 51, [0], (5, 0), 0)
