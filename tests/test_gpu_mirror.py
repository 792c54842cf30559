"""GPU: the mirrored-state rows kernel (tt_rows2.cu, opt-in with TT_ROWS_MIRROR=1: every CTA holds the whole
Ah, two cluster barriers per frame, partials exchanged through distributed shared memory) against the default
L2-exchange kernel and the oracle: static, informative (with and without replacement) and norm_cap runs at
several cluster sizes. The two kernels sum the column norms in different orders, so they agree to rounding
(gamma 1e-5) with identical masks."""

import numpy as np
import pytest

from conftest import rel
from oracle import tt_oracle as O

pytestmark = pytest.mark.gpu


def _run(monkeypatch, mirror, *args, **kw):
    import paper_1609_04104_b200 as tt
    from paper_1609_04104_b200 import _lib as L

    monkeypatch.setenv("TT_ROWS_MIRROR", "1" if mirror else "0")
    return tt.run_online(*args, **kw), L


@pytest.mark.parametrize("n,R,cluster,kind", [(64, 6, 4, "informative"), (128, 10, 16, "static"),
                                              (96, 8, 2, "wor"), (64, 5, 1, "informative")])
def test_mirrored_kernel_matches_default_and_oracle(monkeypatch, n, R, cluster, kind):
    import paper_1609_04104_b200 as tt
    from paper_1609_04104_b200.phantom import cine_phantom

    T = 8
    ph = cine_phantom(n, n, T, period=8.0, seed=90 + n)
    A0, B0 = O.random_subspace(n, n, R, seed=91)
    if kind == "static":
        gen = np.random.Generator(np.random.Philox(key=92))
        S = n // 4
        rows = [O.vd_rows(n, -1.0, S / n, gen.random) for _ in range(T)]
        pol = tt.StaticRows(np.stack(rows)[:, None, :], np.full((T, 1), S))
        opol = {"kind": "static", "rows": rows}
    else:
        pol = tt.Informative(k=n // 4, forced=(0, 1), beta=0.1, key0=93, replacement=kind != "wor")
        opol = {"kind": "informative", "k": n // 4, "forced": [0, 1], "beta": 0.1, "key": (93, 0),
                "replacement": kind != "wor"}
    args = (ph.kspace, A0[None], B0[None], 0.1, tt.Fixed(0.01), pol)
    kw = dict(clean=ph.clean, cluster=cluster, norm_cap=25.0)
    res_m, L = _run(monkeypatch, True, *args, **kw)
    assert L.lib().tt_rows_mirror_fits(n, n, R, n // 4, cluster) == 1
    res_d, _ = _run(monkeypatch, False, *args, **kw)
    ref = O.online_run(ph.kspace, A0, B0, 0.1, ("fixed", 0.01), opol, clean=ph.clean)
    for f in range(T):
        np.testing.assert_array_equal(res_m.rows[f][0], res_d.rows[f][0])
        np.testing.assert_array_equal(np.sort(res_m.rows[f][0]), np.sort(ref["rows"][f]))
        assert rel(res_m.gamma[f, 0], res_d.gamma[f, 0]) < 1e-5
        assert rel(res_m.gamma[f, 0], ref["gamma"][f]) < 1e-4
    assert rel(res_m.final_A, res_d.final_A) < 1e-5 and rel(res_m.final_B, res_d.final_B) < 1e-5
    np.testing.assert_array_equal(res_m.norm_exceeded, res_d.norm_exceeded)
    assert np.max(np.abs(np.sqrt(res_m.nmse[:, 0]) - np.sqrt(ref["nmse"]))) < 1e-3
