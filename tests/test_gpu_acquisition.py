"""Acquisition on the device: StreamingProvider's frame-order tripwire
(experiment.py:70-111), entry reads, and project / measure (observation.py:186-204, :335-353)."""

import numpy as np
import pytest

from conftest import rel
from oracle import tt_oracle as O

pytestmark = pytest.mark.gpu


def _truth(n1=24, n2=20, T=5, seed=3):
    rng = np.random.default_rng(seed)
    return rng.standard_normal((n1, n2, T)) + 1j * rng.standard_normal((n1, n2, T))  # frames last, as the reference


def test_frame_order_tripwire():
    import paper_1609_04104_b200 as tt

    p = tt.StreamingProvider(_truth())
    assert p.frames == 5 and p.frame_shape == (24, 20)
    p.full_frame(0)
    p.full_frame(0)  # re-reading a served frame is allowed
    with pytest.raises(RuntimeError):
        p.entries(2, [[0, 0]])  # frame 1 not processed yet
    p.entries(1, [[0, 0]])
    with pytest.raises(IndexError):
        p.full_frame(5)
    with pytest.raises(IndexError):
        p.full_frame(-1)


def test_entries_and_sketches_match_numpy():
    import paper_1609_04104_b200 as tt

    X = _truth()
    p = tt.StreamingProvider(X)
    rng = np.random.default_rng(8)
    idx = np.argwhere(rng.random((24, 20)) < 0.3)
    got = p.entries(0, idx)
    np.testing.assert_array_equal(got, X[..., 0].astype(np.complex64)[tuple(idx.T)].astype(np.complex128))
    # FourierMask sketch = unitary_dft2(frame)[idx]; noise from the caller's rng, drawn like the reference
    desc = tt.FourierMask((24, 20), idx)
    r1, r2 = np.random.default_rng(5), np.random.default_rng(5)
    b = p.sketch(1, desc, 0.01, r1)
    clean = O.dft2(X[..., 1].astype(np.complex64))[tuple(idx.T)]
    noise = r2.standard_normal(len(idx)) + 1j * r2.standard_normal(len(idx))
    assert rel(np.asarray(b.y), clean + 0.01 * noise) < 1e-5
    assert r1.random() == r2.random()  # generator streams stay in step
    e = tt.measure(X[..., 2], tt.EntryMask((24, 20), idx), 0.0, None)
    np.testing.assert_allclose(np.asarray(e.y), X[..., 2][tuple(idx.T)], rtol=1e-6)
    with pytest.raises(ValueError):
        tt.project(X[..., 0], tt.EntryMask((20, 24), [[0, 0]]))
    with pytest.raises(ValueError):
        tt.measure(X[..., 0], desc, -1.0, None)


def test_provider_truth_feeds_the_engine():
    """The provider's device truth is the engines' resident k-space (frames leading)."""
    import paper_1609_04104_b200 as tt
    from paper_1609_04104_b200.phantom import cine_phantom

    n, R, T = 32, 4, 4
    ph = cine_phantom(n, n, T, 8.0, seed=2)
    prov = tt.StreamingProvider(np.moveaxis(ph.kspace, 0, -1))
    A0, B0 = O.random_subspace(n, n, R, seed=3)
    pol = tt.Informative(k=8, forced=(0,), key0=1)
    a = tt.run_online(prov.truth_device, A0[None], B0[None], 0.1, tt.Fixed(0.01), pol)
    b = tt.run_online(ph.kspace, A0[None], B0[None], 0.1, tt.Fixed(0.01), pol)
    np.testing.assert_array_equal(a.gamma, b.gamma)
