"""GPU: the default cluster of a row-mask launch is the widest one whose resident-cluster count (the occupancy
calculator's, tt_rows_max_clusters) covers the slices, so no batched launch runs in waves; a batched launch at
the chosen cluster equals the single-slice runs at that cluster bit for bit (the slices of
experiment.py:332-441 are independent)."""

import ctypes as C

import numpy as np
import pytest

from oracle import tt_oracle as O

pytestmark = pytest.mark.gpu


def _max_clusters(L, n, R, S, c):
    m = C.c_int(0)
    L.check(L.lib().tt_rows_max_clusters(n, n, R, S, c, C.byref(m)), "occupancy")
    return m.value


def test_default_cluster_keeps_every_slice_resident():
    from paper_1609_04104_b200 import _lib as L
    from paper_1609_04104_b200 import _ops as K

    L.load()
    n, R, S = 256, 16, 52
    occ = {c: _max_clusters(L, n, R, S, c) for c in (2, 4, 8, 16)}
    assert occ[2] >= occ[4] >= occ[8] >= occ[16] >= 1
    assert all(occ[c] * c <= 148 for c in occ)
    last = 32
    for ns in (1, occ[16], occ[16] + 1, occ[8], occ[8] + 1, occ[4], occ[4] + 1, 64, occ[2], occ[2] + 1):
        cl = K.RowsScratch(ns, n, n, R, S).cluster
        assert cl <= last  # more slices never widen the cluster
        last = cl
        if cl > 1:
            assert ns <= occ[cl], (ns, cl, occ)
        wider = [c for c in occ if c > cl and ns <= occ[c]]
        assert not wider, (ns, cl, wider)
    m = C.c_int(0)
    assert L.lib().tt_rows_max_clusters(n, n, R, S, 0, C.byref(m)) != 0  # bad cluster: an error code, no launch


def test_batched_launch_at_the_chosen_cluster_equals_single_slices():
    import paper_1609_04104_b200 as tt
    from paper_1609_04104_b200 import _lib as L
    from paper_1609_04104_b200 import _ops as K
    from paper_1609_04104_b200.phantom import cine_phantom

    L.load()
    n, R, T, k = 64, 6, 4, 13
    ns = _max_clusters(L, n, R, k, 16) + 1  # one slice more than the clusters of 16 the device holds
    cl = K.RowsScratch(ns, n, n, R, k).cluster
    assert cl < 16
    ks = np.stack([cine_phantom(n, n, T, 8.0, seed=3, slice_index=s).kspace for s in range(ns)], axis=1)
    AB = [O.random_subspace(n, n, R, seed=40 + s) for s in range(ns)]
    A0, B0 = np.stack([a for a, _ in AB]), np.stack([b for _, b in AB])
    pol = tt.Informative(k=k, forced=(0,), beta=0.1, key0=5)
    batched = tt.run_online(ks, A0, B0, 0.05, tt.Fixed(0.01), pol)
    for s in (0, ns - 1):
        pol_s = tt.Informative(k=k, forced=(0,), beta=0.1, key0=5, key1=s)
        single = tt.run_online(ks[:, s], A0[s:s + 1], B0[s:s + 1], 0.05, tt.Fixed(0.01), pol_s, cluster=cl)
        np.testing.assert_array_equal(batched.gamma[:, s], single.gamma[:, 0])
        for f in range(T):
            np.testing.assert_array_equal(batched.rows[f][s], single.rows[f][0])
