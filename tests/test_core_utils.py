"""Host utilities of tensortrack.core (core.py:76-190) restated in the package: unfold / refold
(mode-m matricisation and its exact inverse, test_core.py's round trip), outer_rank_one,
singular_values (product of per-component column norms) and rank_surrogate."""

import numpy as np
import pytest

import paper_1609_04104_b200 as tt


def test_unfold_refold_roundtrip_and_layout():
    x = np.arange(2 * 3 * 4).reshape(2, 3, 4)
    for mode in (1, 2, 3):
        m = tt.unfold(x, mode)
        assert m.shape == (x.shape[mode - 1], x.size // x.shape[mode - 1])
        np.testing.assert_array_equal(tt.refold(m, mode, x.shape), x)
    np.testing.assert_array_equal(tt.unfold(x, 2)[1], x[:, 1, :].ravel())
    with pytest.raises(ValueError):
        tt.unfold(x, 4)
    with pytest.raises(ValueError):
        tt.refold(x.reshape(2, -1), 0, x.shape)


@pytest.mark.gpu
def test_outer_rank_one_and_norm_helpers():  # TensorSubspace holds device buffers
    a, b, c = np.array([1, 2j]), np.array([3, 4, 5]), np.array([1, -1])
    t = tt.outer_rank_one([a, b, c])
    assert t.shape == (2, 3, 2) and t[1, 2, 1] == 2j * 5 * -1
    with pytest.raises(ValueError):
        tt.outer_rank_one([])
    rng = np.random.default_rng(0)
    A = rng.standard_normal((6, 3)) + 1j * rng.standard_normal((6, 3))
    B = rng.standard_normal((5, 3)) + 1j * rng.standard_normal((5, 3))
    sub = tt.TensorSubspace((A, B))
    np.testing.assert_allclose(tt.singular_values(sub), np.linalg.norm(A, axis=0) * np.linalg.norm(B, axis=0),
                               rtol=1e-6)
    assert tt.rank_surrogate([A, B]) == pytest.approx((np.linalg.norm(A) ** 2 + np.linalg.norm(B) ** 2) / 2)
    # balanced factors: (1/M) sum ||A_m||_F^2 = sum_r sigma_r^(2/M) at M = 2
    Ab, Bb = tt.rebalance(sub).factors
    assert tt.rank_surrogate([Ab, Bb]) == pytest.approx(np.sum(tt.singular_values(sub)), rel=1e-5)


def test_config_error_and_metric_exports():
    """ConfigError (config.py:19) is a ValueError; nmse / ConfigError exported like the reference's
    package namespace (__init__.py:3-62)."""
    import paper_1609_04104_b200 as tt

    assert issubclass(tt.ConfigError, ValueError)
    for name in ("ConfigError", "nmse", "nmse_frames"):
        assert name in tt.__all__ and hasattr(tt, name)


def test_frame_rows_sequence():
    """OnlineResult.rows: a lazy per-frame / per-slice view over the run's row tables (several run
    segments concatenated), list-of-lists semantics."""
    from paper_1609_04104_b200.engine import FrameRows

    r = np.arange(2 * 3 * 5).reshape(2, 3, 5).astype(np.int32)
    c = np.array([[1, 2, 3], [5, 0, 4]], np.int32)
    fr = FrameRows([(r, c), (r + 100, c)])
    assert len(fr) == 4 and fr.total() == 30
    assert fr[1][0].dtype == np.int64 and fr[1][0].tolist() == [15, 16, 17, 18, 19]
    assert fr[3][2].tolist() == [125, 126, 127, 128] and fr[-1][1].size == 0
    assert [len(x) for x in fr] == [3, 3, 3, 3]
    assert sum(len(s) for f in fr for s in f) == 30
    assert [a.tolist() for a in fr[1:3][1]] == [a.tolist() for a in fr[2]]
    with pytest.raises(IndexError):
        fr[4]
