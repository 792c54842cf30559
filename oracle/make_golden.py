"""Pin the oracle against the reference and write golden fixtures.

TEST INFRASTRUCTURE. Runs only in the build container, where the reference
package lives at /root/reference (read-only). It:

1. imports the reference modules ``core``, ``observation``, ``tracker``,
   ``sampler`` directly, by pre-registering a bare ``tensortrack`` package
   module so ``__init__.py`` (which pulls scikit-image through
   ``metrics.py``) never runs;
2. checks every oracle function against the reference function it restates
   on seeded inputs (raises on disagreement);
3. writes the *reference's own outputs* for seeded cases as small ``.npz``
   fixtures under ``tests/golden/``. The GPU parity tests and
   ``tests/test_oracle.py`` read those fixtures; nothing at test time needs
   /root/reference.

Usage: ``python oracle/make_golden.py``  (re-run only when cases change).
"""

from __future__ import annotations

import os
import sys
import types

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
sys.path.insert(0, REPO)
from oracle import tt_oracle as O  # noqa: E402

REF_PKG = "/root/reference/pkg/src/tensortrack"
GOLDEN = os.path.join(REPO, "tests", "golden")


def load_reference():
    if "tensortrack" not in sys.modules:
        pkg = types.ModuleType("tensortrack")
        pkg.__path__ = [REF_PKG]
        sys.modules["tensortrack"] = pkg
    import importlib

    mods = {}
    for name in ("core", "observation", "tracker", "sampler", "mri"):
        mods[name] = importlib.import_module(f"tensortrack.{name}")
    return types.SimpleNamespace(**mods)


def _rand_c(rng, *shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def _close(a, b, tol=1e-10, what=""):
    a = np.asarray(a)
    b = np.asarray(b)
    den = max(np.linalg.norm(b), 1e-300)
    err = np.linalg.norm(a - b) / den if b.size else 0.0
    if not err <= tol:
        raise AssertionError(f"oracle disagrees with reference on {what}: rel {err:.3e}")
    return err


def step_cases(ref):
    """track_step on Fourier rows / Fourier entries / entry masks, fixed and
    Hessian steps. Returns fixture arrays (reference outputs)."""
    out = {}
    cases = [
        # name, n1, n2, R, kind, mask, step, lam, t
        ("fr_fixed", 16, 12, 3, "fourier", "rows", ("fixed", 0.02), 0.3, 4),
        ("fr_hess", 16, 12, 3, "fourier", "rows", ("hessian", 0.5, 1e6), 0.3, 4),
        ("fe_fixed", 12, 10, 4, "fourier", "entries", ("fixed", 0.05), 0.2, 3),
        ("fe_hess", 12, 10, 4, "fourier", "entries", ("hessian", 1e-3, 1e9), 0.2, 3),
        ("ee_fixed", 11, 9, 3, "entry", "entries", ("fixed", 0.05), 0.4, 2),
        ("ee_hess", 11, 9, 3, "entry", "entries", ("hessian", 1e-3, 1e9), 0.4, 2),
        ("odd_fixed", 7, 5, 2, "fourier", "entries", ("fixed", 0.03), 0.1, 1),
        ("c1_fixed", 128, 128, 10, "fourier", "rows", ("fixed", 0.01), 0.1, 7),
        ("c2_fixed", 256, 256, 20, "fourier", "rows", ("fixed", 0.01), 0.05, 11),
        ("empty", 8, 8, 2, "fourier", "empty", ("fixed", 0.05), 0.5, 5),
    ]
    names = []
    for ci, (name, n1, n2, R, kind, mask, step, lam, t) in enumerate(cases):
        rng = np.random.default_rng(1000 + ci)
        A = _rand_c(rng, n1, R) / np.sqrt(2 * n1)
        B = _rand_c(rng, n2, R) / np.sqrt(2 * n2)
        if mask == "rows":
            nrows = max(1, n1 // 4)
            rows = rng.choice(n1, size=nrows, replace=False)  # draw order, unsorted
            idx = O.rows_to_entries(rows, n2)
        elif mask == "entries":
            idx = np.argwhere(rng.random((n1, n2)) < 0.45)
            rows = np.zeros(0, np.int64)
        else:
            idx = np.zeros((0, 2), np.int64)
            rows = np.zeros(0, np.int64)
        # data = a noisy rank-R frame seen through the mask
        Ah, Bh = O.measurement_factors(A, B, kind)
        g_true = _rand_c(rng, R)
        y = (Ah[idx[:, 0]] * Bh[idx[:, 1]]) @ g_true * 0.7 + 0.05 * _rand_c(rng, len(idx))
        alpha_bar = 3.0 if step[0] == "hessian" else 0.0

        Desc = ref.observation.FourierMask if kind == "fourier" else ref.observation.EntryMask
        desc = Desc((n1, n2), idx)
        stepobj = ref.tracker.Fixed(step[1]) if step[0] == "fixed" else ref.tracker.HessianBound(step[1], step[2])
        cfg = ref.tracker.StepConfig(lam=lam, rank=R, step=stepobj)
        st = ref.tracker.TrackerState(ref.core.TensorSubspace((A, B)), cfg, t=t, alpha_bar=alpha_bar)
        new, rep = ref.tracker.track_step(st, ref.observation.MeasurementBatch(y, desc))
        A2, B2 = new.subspace.factors

        mine = O.track_step(A, B, t, alpha_bar, y, idx, kind, lam, step, power=True)
        _close(mine["A"], A2, 1e-10, f"{name} A")
        _close(mine["B"], B2, 1e-10, f"{name} B")
        _close(mine["gamma"], rep.gamma, 1e-10, f"{name} gamma")
        _close(mine["residual"], rep.residual, 1e-9, f"{name} residual")
        assert abs(mine["cost"] - rep.instantaneous_cost) <= 1e-10 * max(1.0, abs(rep.instantaneous_cost))
        assert abs(mine["mu"] - rep.step_size) <= 1e-12 * max(1.0, abs(rep.step_size))
        if step[0] == "hessian" and len(idx):
            a_ref = ref.tracker.hessian_bound(st.subspace, rep.gamma, desc, lam, t, step[1], step[2])
            a_cf = O.alpha_closed(A, B, rep.gamma, idx, kind, lam, t, step[1], step[2])
            # the power method converges from below to the closed form
            assert abs(a_cf - a_ref) <= 1e-6 * a_cf, (name, a_cf, a_ref)

        names.append(name)
        p = f"{name}__"
        out.update({p + "A": A, p + "B": B, p + "idx": idx, p + "rows": rows, p + "y": y,
                    p + "meta": np.array([n1, n2, R, t, 1 if kind == "fourier" else 0,
                                          {"rows": 0, "entries": 1, "empty": 2}[mask],
                                          0 if step[0] == "fixed" else 1]),
                    p + "fparams": np.array([lam, step[1], step[2] if len(step) > 2 else 0.0, alpha_bar]),
                    p + "A_out": A2, p + "B_out": B2, p + "gamma": rep.gamma, p + "residual": rep.residual,
                    p + "cost": np.array(rep.instantaneous_cost), p + "mu": np.array(rep.step_size),
                    p + "alpha_bar_out": np.array(new.alpha_bar), p + "t_out": np.array(new.t)})
    out["names"] = np.array(names)
    return out


def solve_cases(ref):
    rng = np.random.default_rng(3)
    out = {}
    for c in range(12):
        L = int(rng.integers(5, 61))
        r = int(rng.integers(1, 21))
        lam = float(rng.choice([0.01, 2.0, 100.0]))
        phi = _rand_c(rng, L, r)
        y = _rand_c(rng, L)
        g = ref.tracker.solve_gamma(phi, y, lam)
        _close(O.ridge_svd(phi, y, lam), g, 1e-10, "solve_gamma")
        _close(O.ridge_normal(phi, y, lam), g, 1e-9, "normal equations")
        out.update({f"c{c}__phi": phi, f"c{c}__y": y, f"c{c}__lam": np.array(lam), f"c{c}__gamma": g})
    out["count"] = np.array(12)
    return out


def sampling_cases(ref):
    out = {}
    rng = np.random.default_rng(44)
    # row / entry scores (fp64 laws)
    for c, (n1, n2, R, beta) in enumerate([(16, 12, 3, 0.1), (64, 48, 5, 0.0), (128, 96, 20, 0.1), (9, 7, 2, 0.5)]):
        A = _rand_c(rng, n1, R)
        B = _rand_c(rng, n2, R)
        sub = ref.core.TensorSubspace((A, B))
        rs = ref.sampler.row_scores(sub, beta).scores
        es = ref.sampler.entry_scores(sub, beta).scores
        _close(O.row_probs(A, n2, beta), rs, 1e-13, "row_scores")
        _close(O.entry_probs(A, B, beta), es, 1e-13, "entry_scores")
        out.update({f"s{c}__A": A, f"s{c}__B": B, f"s{c}__beta": np.array(beta),
                    f"s{c}__rows": rs, f"s{c}__entries": es})
    out["nscores"] = np.array(4)
    # draws with replacement on a Philox stream, through the reference draw_samples
    draws = [(256, 64, list(range(8)) + list(range(248, 256)), (2024, 0)),
             (256, 52, [0], (7, 3)),
             (128, 32, [], (11, 1)),
             (1024, 128, [0], (5, 9)),
             (40, 17, [3, 5], (1, 1))]
    for c, (n, k, forced, key) in enumerate(draws):
        p = rng.random(n) ** 3 + 0.01
        p = p / p.sum()
        dist = ref.sampler.SamplingDistribution(p, "rows")
        g = np.random.Generator(np.random.Philox(key=key[0] + (key[1] << 64)))
        plans = []
        pos = 0
        for rep in range(3):  # consecutive frames share the stream
            plan = ref.sampler.draw_samples(dist, k, True, g, forced=forced if forced else None)
            mine, used = O.draw_rows(p, k, forced, key, pos)
            pos += used
            if not np.array_equal(mine, plan.omega):
                raise AssertionError("draw_rows disagrees with reference draw_samples")
            plans.append(plan.omega)
        out.update({f"d{c}__p": p, f"d{c}__k": np.array(k), f"d{c}__forced": np.array(forced, np.int64),
                    f"d{c}__key": np.array(key, np.uint64),
                    f"d{c}__omega0": plans[0], f"d{c}__omega1": plans[1], f"d{c}__omega2": plans[2]})
    out["ndraws"] = np.array(len(draws))
    # variable-density rows (sequential without replacement) on Philox
    for c, (n1, alpha, frac, key) in enumerate([(128, -1.0, 0.25, (9, 0)), (1024, -1.0, 0.125, (9, 1)),
                                                 (40, -0.5, 0.33, (2, 2))]):
        g = np.random.Generator(np.random.Philox(key=key[0] + (key[1] << 64)))
        rows = ref.observation.variable_density_rows(n1, alpha, frac, g)
        g2 = np.random.Generator(np.random.Philox(key=key[0] + (key[1] << 64)))
        mine = O.vd_rows(n1, alpha, frac, g2.random)
        if not np.array_equal(rows, mine):
            raise AssertionError("vd_rows disagrees with reference")
        out.update({f"v{c}__n1": np.array(n1), f"v{c}__alpha": np.array(alpha),
                    f"v{c}__frac": np.array(frac), f"v{c}__key": np.array(key, np.uint64),
                    f"v{c}__rows": rows})
    out["nvd"] = np.array(3)
    return out


def value_cases(ref):
    out = {}
    rng = np.random.default_rng(55)
    A = _rand_c(rng, 20, 4)
    B = _rand_c(rng, 14, 4)
    g = _rand_c(rng, 4)
    sub = ref.core.TensorSubspace((A, B))
    X = ref.core.synthesize_slice(sub, g)
    _close(O.synth(A, B, g), X, 1e-13, "synthesize_slice")
    est = ref.mri.reconstruct_frame(sub, g)
    _close(O.synth(A, B, g), est.kspace, 1e-13, "reconstruct_frame")
    A[:, 2] *= 40.0
    B[:, 1] *= 1e-3
    rb = ref.core.rebalance(ref.core.TensorSubspace((A, B))).factors
    ra, rb2 = O.rebalance(A, B)
    _close(ra, rb[0], 1e-13, "rebalance A")
    _close(rb2, rb[1], 1e-13, "rebalance B")
    out.update(A=A, B=B, gamma=g, synth=ref.core.synthesize_slice(ref.core.TensorSubspace((A, B)), g),
               image=ref.mri.reconstruct_frame(ref.core.TensorSubspace((A, B)), g).image,
               rebal_A=rb[0], rebal_B=rb[1])
    x = _rand_c(rng, 16, 12)
    out["dft_in"] = x
    out["dft_out"] = ref.observation.unitary_dft2(x)
    out["idft_out"] = ref.observation.unitary_dft2(x, inverse=True)
    return out


def loop_case(ref):
    """Short free-running online loop built only from reference public
    functions in run_adaptive order: informative rows with a
    dedicated Philox mask stream and pre-noised truth."""
    from paper_1609_04104_b200.phantom import cine_phantom

    n, R, T, lam = 64, 6, 10, 0.1
    ph = cine_phantom(n, n, T, period=8.0, seed=17)
    kspace = ph.kspace.astype(np.complex128)
    A0, B0 = O.random_subspace(n, n, R, seed=5)
    key = (77, 0)
    K = 16
    forced = list(range(4)) + list(range(n - 4, n))
    g = np.random.Generator(np.random.Philox(key=key[0] + (key[1] << 64)))
    cfg = ref.tracker.StepConfig(lam=lam, rank=R, step=ref.tracker.Fixed(0.01))
    st = ref.tracker.TrackerState(ref.core.TensorSubspace((A0, B0)), cfg)
    gam, costs, rows_all, nm = [], [], [], []
    for f in range(T):
        A, B = st.subspace.factors
        khat = ref.core.TensorSubspace((np.fft.fft(A, axis=0, norm="ortho"), np.fft.fft(B, axis=0, norm="ortho")))
        dist = ref.sampler.row_scores(khat, 0.1)
        plan = ref.sampler.draw_samples(dist, K, True, g, forced=forced)
        idx = ref.observation.rows_to_entries(plan.omega, n)
        y = kspace[f][plan.omega, :].ravel()
        st, rep = ref.tracker.track_step(st, ref.observation.MeasurementBatch(y, ref.observation.FourierMask((n, n), idx)))
        X = ref.core.synthesize_slice(st.subspace, rep.gamma)
        gam.append(rep.gamma)
        costs.append(rep.instantaneous_cost)
        rows_all.append(plan.omega)
        cf = ph.clean[f].astype(np.complex128)
        nm.append(float(np.linalg.norm(cf - X) ** 2 / np.linalg.norm(cf) ** 2))
    mine = O.online_run(kspace, A0, B0, lam, ("fixed", 0.01),
                        {"kind": "informative", "k": K, "forced": forced, "beta": 0.1, "key": key},
                        clean=ph.clean)
    for f in range(T):
        if not np.array_equal(mine["rows"][f], rows_all[f]):
            raise AssertionError(f"oracle loop mask differs at frame {f}")
        _close(mine["gamma"][f], gam[f], 1e-9, "loop gamma")
    _close(mine["final"][0], st.subspace.factors[0], 1e-9, "loop A")
    _close(np.array(mine["nmse"]), np.array(nm), 1e-9, "loop nmse")
    rows_pad = np.full((T, K), -1, np.int64)
    for f, r in enumerate(rows_all):
        rows_pad[f, :len(r)] = r
    return dict(kspace=ph.kspace, clean=ph.clean, A0=A0, B0=B0, gamma=np.array(gam), cost=np.array(costs),
                rows=rows_pad, nmse=np.array(nm), A_final=st.subspace.factors[0], B_final=st.subspace.factors[1],
                meta=np.array([n, R, T, K, key[0], key[1]]), lam=np.array(lam), forced=np.array(forced))


def main():
    ref = load_reference()
    os.makedirs(GOLDEN, exist_ok=True)
    for fname, fn in [("step_cases", step_cases), ("solve_cases", solve_cases),
                      ("sampling_cases", sampling_cases), ("value_cases", value_cases),
                      ("loop_case", loop_case)]:
        data = fn(ref)
        path = os.path.join(GOLDEN, fname + ".npz")
        np.savez_compressed(path, **data)
        print(f"wrote {path} ({os.path.getsize(path) / 1024:.1f} KiB)")
    print("oracle pinned against the reference: all checks passed")


if __name__ == "__main__":
    main()
