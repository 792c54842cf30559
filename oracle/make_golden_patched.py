"""Golden vectors for the per-patch trackers (experiment._run_tracking_patched, experiment.py:332-441),
produced by the reference itself. Test infrastructure only: run in the build container; the fixtures
are committed under tests/golden/patched_*.npz.

The reference's run_tracking is run with a PatchConfig and noise_sigma = 0 (noise is
pre-baked into the truth). Its generator is then replayed to recover the inputs it drew (per-patch
random_subspace inits, then the per-frame masks of _draw_frame_entries, then the reshuffle
permutations), the oracle's patched_run is driven with them and asserted equal to the reference at
1e-10, and inputs plus the reference's outputs are written. scikit-image is absent, so a stub
`skimage.metrics` is registered before importing experiment (the SSIM column is not compared).
"""

from __future__ import annotations

import importlib
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

CASES = {
    # name: frame (N1, N2), patch (n1, n2, rho), T, warm_n, warm_epochs, epochs, reshuffle, sampling, step
    "patched_vd": dict(shape=(32, 32), patch=(8, 8, 2), T=9, warm_n=2, warm_epochs=2, epochs=2, reshuffle=True,
                       sampling=dict(mode="variable_density", fraction=0.3), step=("fixed", 0.3), seed=11),
    "patched_uniform": dict(shape=(32, 16), patch=(8, 4, 3), T=7, warm_n=1, warm_epochs=1, epochs=1,
                            reshuffle=False, sampling=dict(mode="uniform", fraction=0.35),
                            step=("hessian", 1e-3, 1e9), seed=12),
}


def load():
    if "tensortrack" not in sys.modules:
        pkg = types.ModuleType("tensortrack")
        pkg.__path__ = [REF_PKG]
        sys.modules["tensortrack"] = pkg
    sk = types.ModuleType("skimage")
    skm = types.ModuleType("skimage.metrics")
    skm.structural_similarity = lambda *a, **k: 0.0
    sk.metrics = skm
    sys.modules.setdefault("skimage", sk)
    sys.modules.setdefault("skimage.metrics", skm)
    return (importlib.import_module("tensortrack.experiment"), importlib.import_module("tensortrack.config"),
            importlib.import_module("tensortrack.tracker"))


def truth_tensor(shape, T, seed):
    """Smooth low-rank k-space-like data plus a small perturbation, frames last (the reference's layout)."""
    g = np.random.default_rng(1000 + seed)
    N1, N2 = shape
    u = g.standard_normal((N1, 3)) + 1j * g.standard_normal((N1, 3))
    v = g.standard_normal((N2, 3)) + 1j * g.standard_normal((N2, 3))
    x = np.empty((N1, N2, T), np.complex128)
    for t in range(T):
        c = np.array([1.0, 0.5 * np.cos(0.4 * t), 0.3 * np.sin(0.3 * t)])
        x[..., t] = (u * c) @ v.T / np.sqrt(N1 * N2) + 0.01 * (g.standard_normal((N1, N2)) + 1j * g.standard_normal((N1, N2)))
    return x


def close(a, b, what, tol=1e-10):
    a, b = np.asarray(a), np.asarray(b)
    den = max(np.linalg.norm(b), 1e-300)
    err = np.linalg.norm(a - b) / den if b.size else 0.0
    if not err <= tol:
        raise AssertionError(f"oracle disagrees with the reference on {what}: rel {err:.3e}")


def main():
    ex, cf, tr = load()
    for name, c in CASES.items():
        N1, N2 = c["shape"]
        n1, n2, rho = c["patch"]
        T = c["T"]
        lam = 0.1
        step = c["step"]
        kw = dict(step_mode=step[0])
        if step[0] == "fixed":
            kw["mu"] = step[1]
        else:
            kw["c_floor"], kw["c_cap"] = step[1], step[2]
        cfg = cf.ExperimentConfig(seed=c["seed"], rank=rho, lam=lam, epochs=c["epochs"], reshuffle=c["reshuffle"],
                                  sampling=cf.SamplingConfig(**c["sampling"]), patch=cf.PatchConfig(n1, n2, rho),
                                  noise_sigma=0.0, warm_start_frames=c["warm_n"], warm_epochs=c["warm_epochs"], **kw)
        truth = truth_tensor((N1, N2), T, c["seed"])
        ref = ex.run_tracking(truth, cfg)
        # replay the generator: inits, masks, then (inside patched_run) the permutations
        rng = np.random.default_rng(c["seed"])
        npatch = (N1 // n1) * (N2 // n2)
        A0s, B0s = [], []
        for _ in range(npatch):
            sub = tr.random_subspace((n1, n2), rho, rng, 1.0)
            A0s.append(sub.factors[0])
            B0s.append(sub.factors[1])
        entries = [O.full_entries((N1, N2)) for _ in range(c["warm_n"])]
        for t in range(c["warm_n"], T):
            e, _ = ex._draw_frame_entries(cfg, (N1, N2), rng)
            entries.append(np.asarray(e, np.int64))
        frames = np.moveaxis(truth, -1, 0)
        step_o = ("fixed", step[1]) if step[0] == "fixed" else ("hessian", step[1], step[2])
        out = O.patched_run(frames, A0s, B0s, lam, step_o, n1, n2, entries, c["warm_n"], c["warm_epochs"],
                            c["epochs"], rng=rng, reshuffle=c["reshuffle"])
        assert len(out["trace"]) == len(ref.trace)
        for k, (a, b) in enumerate(zip(out["trace"], ref.trace)):
            close(a["gamma"], b.gamma, f"{name} step {k} gamma")
            close(a["residual"], b.residual, f"{name} step {k} residual")
            close(a["cost"], b.instantaneous_cost, f"{name} step {k} cost")
            close(a["mu"], b.step_size, f"{name} step {k} mu")
            assert a["t"] == b.t
        close(out["recon"], np.moveaxis(ref.recon, -1, 0), f"{name} recon")
        for t, m in enumerate(ref.metrics):
            close(O.nmse(frames[t], out["recon"][t]), m.nmse, f"{name} nmse {t}", 1e-9)
        L = max(len(e) for e in entries)
        etab = np.full((T, L, 2), -1, np.int32)
        for t, e in enumerate(entries):
            etab[t, :len(e)] = e
        res = [b.residual for b in ref.trace]
        R = max(len(r) for r in res)
        rtab = np.zeros((len(res), R), np.complex128)
        for k, r in enumerate(res):
            rtab[k, :len(r)] = r
        np.savez_compressed(
            os.path.join(GOLDEN, f"{name}.npz"),
            frames=frames, A0s=np.stack(A0s), B0s=np.stack(B0s), entries=etab,
            counts=np.array([len(e) for e in entries], np.int32),
            shape=np.array([N1, N2]), patch=np.array([n1, n2, rho]), lam=lam,
            step_kind=step[0], step_par=np.array(step[1:], np.float64),
            T=T, warm_n=c["warm_n"], warm_epochs=c["warm_epochs"], epochs=c["epochs"], reshuffle=c["reshuffle"],
            seed=c["seed"], orders=np.array([o for o in out["orders"]], dtype=object) if False else np.concatenate(out["orders"]),
            trace_gamma=np.stack([b.gamma for b in ref.trace]), trace_cost=np.array([b.instantaneous_cost for b in ref.trace]),
            trace_mu=np.array([b.step_size for b in ref.trace]), trace_t=np.array([b.t for b in ref.trace]),
            trace_resid=rtab, trace_resid_len=np.array([len(r) for r in res]),
            recon=np.moveaxis(ref.recon, -1, 0), nmse=np.array([m.nmse for m in ref.metrics]),
            samples=np.array([m.samples for m in ref.metrics]))
        print(name, "ok:", len(ref.trace), "steps,", npatch, "patches; recon nmse", float(np.mean([m.nmse for m in ref.metrics])))


if __name__ == "__main__":
    main()
