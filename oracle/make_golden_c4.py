"""Config-4 full-sequence golden trajectory from the REFERENCE itself.

TEST INFRASTRUCTURE (build container only; /root/reference is read-only and
absent on the GPU box). BASELINE config 4 (1024x1024 complex64 cine phantom,
T=256, R=32, lambda=0.1, Fixed mu=0.01, variable-density rows 12.5% = 128 rows
per frame from Generator(Philox(2024))) is run cold-started through the
reference's own per-frame API — ``tracker.track_step`` on a ``FourierMask``
(tracker.py:367-411, observation.py:74-90) with image-domain factors, the
north-star call — and ``mri.reconstruct_frame`` (mri.py:107-121) for every
frame's estimate. About 0.8 s per frame (numpy SVD of the 131072 x 32 Phi),
~4 minutes in all; too slow for a test, so the trajectory is committed:

* ``rows``     (T, 128) int16: each frame's VD rows in draw order (the reference's
                own ``variable_density_rows`` on the Philox generator);
* ``gamma``    (T, R) complex128, ``cost`` (T,), ``mu`` (T,);
* ``nrmse``    (T,): sqrt(nmse(clean_t, estimate_t)) (metrics.py:53-62);
* ``A_ck``/``B_ck`` complex64 factors after the frames in ``ck`` (0, 127, 255).

The initial factors are ``bench.init_factors``'s (default_rng([7, 0]) complex
Gaussian / sqrt(2N)) rounded to complex64, and the data is
``phantom.cine_phantom(1024, 1024, 256, period=16, seed=2024, slice_index=0)``
(complex64), so the device engine starts from bit-identical inputs.
``tests/test_gpu_fullparity.py::test_c4_full_sequence`` replays it.

Usage: ``python oracle/make_golden_c4.py [T]``
"""

from __future__ import annotations

import importlib
import os
import sys
import time
import types

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
sys.path.insert(0, REPO)
REF_PKG = "/root/reference/pkg/src/tensortrack"
OUT = os.path.join(REPO, "tests", "golden", "c4_trajectory.npz")

N, R, LAM, MU, PERIOD, VD, KEY = 1024, 32, 0.1, 0.01, 16.0, 0.125, 2024
CK = (0, 127, 255)


def load_reference():
    if "tensortrack" not in sys.modules:
        pkg = types.ModuleType("tensortrack")
        pkg.__path__ = [REF_PKG]
        sys.modules["tensortrack"] = pkg
    return types.SimpleNamespace(**{m: importlib.import_module(f"tensortrack.{m}")
                                    for m in ("core", "observation", "tracker", "mri")})


def init_factors(n, r, seed=7, s=0):
    """bench.init_factors for one slice, rounded to the complex64 the device starts from."""
    rng = np.random.default_rng([seed, s])
    a = (rng.standard_normal((n, r)) + 1j * rng.standard_normal((n, r))) / np.sqrt(2 * n)
    b = (rng.standard_normal((n, r)) + 1j * rng.standard_normal((n, r))) / np.sqrt(2 * n)
    return a.astype(np.complex64).astype(np.complex128), b.astype(np.complex64).astype(np.complex128)


def main():
    from paper_1609_04104_b200.phantom import cine_phantom

    T = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    ref = load_reference()
    Tr, Ob, Co, Mr = ref.tracker, ref.observation, ref.core, ref.mri
    ph = cine_phantom(N, N, T, period=PERIOD, seed=2024, slice_index=0)
    A0, B0 = init_factors(N, R)
    gen = np.random.Generator(np.random.Philox(key=KEY))
    state = Tr.TrackerState(Co.TensorSubspace((A0, B0)), Tr.StepConfig(LAM, R, Tr.Fixed(MU)))
    rows_all, gam, cost, mu, nrm = [], [], [], [], []
    a_ck, b_ck = [], []
    t0 = time.perf_counter()
    for f in range(T):
        rows = Ob.variable_density_rows(N, -1.0, VD, gen)
        ent = Ob.rows_to_entries(rows, N)
        y = ph.kspace[f].astype(np.complex128)[rows, :].ravel()
        batch = Ob.MeasurementBatch(y, Ob.FourierMask((N, N), ent), t=f)
        state, rep = Tr.track_step(state, batch)
        est = Mr.reconstruct_frame(state.subspace, rep.gamma).kspace  # post-update factors (experiment.py:525)
        clean = ph.clean[f].astype(np.complex128)
        nrm.append(np.sqrt(np.linalg.norm(clean - est) ** 2 / np.linalg.norm(clean) ** 2))
        rows_all.append(np.asarray(rows, np.int16))
        gam.append(rep.gamma)
        cost.append(rep.instantaneous_cost)
        mu.append(rep.step_size)
        if f in CK:
            a_ck.append(state.subspace.factors[0].astype(np.complex64))
            b_ck.append(state.subspace.factors[1].astype(np.complex64))
        if f % 16 == 0:
            print(f"frame {f}: nrmse {nrm[-1]:.4f} ({time.perf_counter() - t0:.0f} s)", flush=True)
    np.savez_compressed(
        OUT, meta=np.array([N, R, T, KEY], np.int64), lam=LAM, mu_fixed=MU, period=PERIOD, vd=VD,
        rows=np.stack(rows_all), gamma=np.stack(gam), cost=np.array(cost), mu=np.array(mu), nrmse=np.array(nrm),
        ck=np.array([c for c in CK if c < T], np.int64), A_ck=np.stack(a_ck), B_ck=np.stack(b_ck))
    print("wrote", OUT, f"{time.perf_counter() - t0:.0f} s")


if __name__ == "__main__":
    main()
