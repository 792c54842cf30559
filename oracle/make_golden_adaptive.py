"""run_adaptive golden runs from the REFERENCE itself: the switch-frame schedule and informative draws
with and without replacement.

TEST INFRASTRUCTURE (build container only; /root/reference is read-only and absent on the GPU box).
The reference's own ``experiment.run_adaptive`` (experiment.py:444-556) is run on a small seeded cine
phantom's k-space with its complete protocol: ``init_state`` from the run's generator, the warm-up
(``warm_start_frames`` full frames x ``warm_epochs`` with rebalancing, experiment.py:219-239), then
variable-density rows until ``switch_frame`` (experiment.py:484-497) and ``row_scores`` +
``draw_samples`` after it (experiment.py:498-510, forced DC line), EntryMask steps on the k-space
state, the reconstruction with the post-update factors (experiment.py:525). The run's generator is
``np.random.Generator(np.random.Philox(key=seed))`` (``np.random.default_rng`` is patched for the
run: the device indexes the Philox stream directly), so the device engine replays it with
``Informative(key0=seed, pos0=<words init_state consumed>)``.

Written per case to ``tests/golden/adaptive_<name>.npz``: the initial k-space factors, the Philox
position after ``init_state``, the truth, every streaming frame's rows (sorted, as the reference
records its masks, experiment.py:495,507; -1 padded), gamma, cost and step, the per-frame NMSE, and the
final factors. Then the
oracle restatement (``tt_oracle.warm_up`` + ``online_run`` with the "schedule" policy) is checked
against it, so the oracle is pinned to the reference on this path.

Usage: ``python oracle/make_golden_adaptive.py``
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
REF_PKG = "/root/reference/pkg/src/tensortrack"
GOLD = os.path.join(REPO, "tests", "golden")

CASES = {
    # name: (n, R, T, warm, epochs, switch, k, replacement, lam, mu, fraction, seed)
    "switch_wr": (48, 5, 22, 2, 3, 8, 14, True, 0.1, 0.01, 0.25, 11),
    "switch_wor": (48, 5, 22, 2, 3, 8, 14, False, 0.1, 0.01, 0.25, 12),
    "wor_nowarm": (40, 4, 14, 0, 1, 0, 12, False, 0.05, 0.02, 0.25, 13),
}


def load_reference():
    if "tensortrack" not in sys.modules:
        pkg = types.ModuleType("tensortrack")
        pkg.__path__ = [REF_PKG]
        sys.modules["tensortrack"] = pkg
    if "skimage.metrics" not in sys.modules:  # SSIM: evaluation only, absent from this image
        sk = types.ModuleType("skimage")
        skm = types.ModuleType("skimage.metrics")
        skm.structural_similarity = lambda *a, **k: 0.0
        sk.metrics = skm
        sys.modules["skimage"] = sk
        sys.modules["skimage.metrics"] = skm
    return types.SimpleNamespace(**{m: importlib.import_module(f"tensortrack.{m}")
                                    for m in ("experiment", "config", "tracker", "observation", "core")})


def run_case(ref, name, n, R, T, W, E, switch, k, repl, lam, mu, frac, seed):
    from oracle import tt_oracle as O
    from paper_1609_04104_b200.phantom import cine_phantom

    Cf = ref.config
    ph = cine_phantom(n, n, T, period=8.0, seed=seed)
    truth = np.moveaxis(ph.kspace.astype(np.complex128), 0, -1)  # frames last, as run_adaptive reads them
    samp = Cf.SamplingConfig(mode="adaptive", fraction=frac, k=k, replacement=repl, beta=0.1, switch_frame=switch,
                             domain="rows")
    cfg = Cf.ExperimentConfig(seed=seed, rank=R, lam=lam, mu=mu, warm_start_frames=W, warm_epochs=E, sampling=samp)
    mk = lambda s: np.random.Generator(np.random.Philox(key=s))  # noqa: E731
    real = np.random.default_rng
    np.random.default_rng = mk
    try:
        g0 = mk(seed)
        st0 = ref.tracker.init_state(ref.experiment._step_config(cfg), (n, n), g0)
        bg = g0.bit_generator.state
        pos0 = (int(bg["state"]["counter"][0]) - 1) * 4 + int(bg["buffer_pos"])
        assert not any(int(v) for v in bg["state"]["counter"][1:]) and not bg["has_uint32"]
        res = ref.experiment.run_adaptive(truth, cfg)
    finally:
        np.random.default_rng = real
    Ah0, Bh0 = st0.subspace.factors
    nstream = T - W
    rows = [[] for _ in range(nstream)]
    for rec in res.mask_rows:
        t, i = rec[0], rec[1]
        if t >= W:
            rows[t - W].append(i)
    tr = res.trace[W * E:]
    assert len(tr) == nstream
    gamma = np.stack([r.gamma for r in tr])
    cost = np.array([r.instantaneous_cost for r in tr])
    mus = np.array([r.step_size for r in tr])
    nm = np.array([m.nmse for m in res.metrics[W:]])
    Af, Bf = res.final_subspace.factors
    nvd = min(max(switch - W, 0), nstream)
    # oracle restatement from the same start: warm-up, then the schedule
    A_img, B_img = O.fft_cols(Ah0, inverse=True), O.fft_cols(Bh0, inverse=True)
    Aw, Bw, t1, ab = O.warm_up(ph.kspace[:W], A_img, B_img, lam, ("fixed", mu), E) if W else (A_img, B_img, 1, 0.0)
    clean = np.stack([O.dft2(truth[..., t], inverse=True) for t in range(W, T)])
    orc = O.online_run(ph.kspace[W:], Aw, Bw, lam, ("fixed", mu),
                       {"kind": "schedule", "vd_frames": nvd, "alpha": -1.0, "fraction": frac, "k": k, "forced": [0],
                        "beta": 0.1, "key": (seed, 0), "position": pos0, "replacement": repl},
                       clean=clean, t0=t1)
    for f in range(nstream):
        want = np.asarray(rows[f], np.int64)
        got = np.sort(orc["rows"][f])  # the mask rows are recorded sorted (experiment.py:495)
        assert np.array_equal(got, want), (name, f, got, want)
        rg = np.linalg.norm(orc["gamma"][f] - gamma[f]) / np.linalg.norm(gamma[f])
        assert rg < 1e-9, (name, f, rg)
    assert np.max(np.abs(np.array(orc["nmse"]) - nm)) < 1e-10
    fa = np.linalg.norm(O.fft_cols(orc["final"][0]) - Af) / np.linalg.norm(Af)
    assert fa < 1e-9, fa
    out = os.path.join(GOLD, f"adaptive_{name}.npz")
    np.savez_compressed(out, meta=np.array([n, R, T, W, E, switch, k, int(repl), seed, pos0, nvd], np.int64),
                        lam=lam, mu=mu, fraction=frac, Ah0=Ah0, Bh0=Bh0, kspace=ph.kspace.astype(np.complex64),
                        rows=np.array([list(r) + [-1] * (n - len(r)) for r in rows], np.int64),
                        counts=np.array([len(r) for r in rows], np.int64), gamma=gamma, cost=cost,
                        step=mus, nmse=nm, Af=Af, Bf=Bf)
    print(f"{name}: {nvd} VD frames then {nstream - nvd} informative (replacement={repl}), pos0 {pos0}; "
          f"oracle == reference; wrote {out}")


def main():
    ref = load_reference()
    for name, c in CASES.items():
        run_case(ref, name, *c)


if __name__ == "__main__":
    main()
