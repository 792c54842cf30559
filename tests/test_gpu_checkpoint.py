"""GPU: checkpoint / resume of the device engine (A, B, t, alpha_bar + Philox positions over CTEN):
a sequence run in one go equals the same sequence split at a checkpoint, saved, loaded into a fresh
engine and continued — bit for bit (rows, gamma, cost, final factors), for informative draws with
HessianBound steps (alpha_bar carries) over several slices."""

import numpy as np
import pytest

from oracle import tt_oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("replacement", [True, False])
def test_resume_from_checkpoint_is_bit_identical(tmp_path, replacement):
    import torch

    import paper_1609_04104_b200 as tt
    from paper_1609_04104_b200 import checkpoint
    from paper_1609_04104_b200.phantom import cine_phantom

    n, R, T, T1, ns = 64, 6, 12, 5, 3
    ks = np.stack([cine_phantom(n, n, T, period=8.0, seed=70 + s).kspace for s in range(ns)], axis=1)
    A0 = np.stack([O.random_subspace(n, n, R, seed=80 + s)[0] for s in range(ns)])
    B0 = np.stack([O.random_subspace(n, n, R, seed=80 + s)[1] for s in range(ns)])
    pol = tt.Informative(k=16, forced=(0,), beta=0.1, key0=5, replacement=replacement, pos0=3)
    step = tt.HessianBound(1e-3, 1e9)
    kd = torch.from_numpy(ks.astype(np.complex64)).cuda()

    def engine():
        e = tt.OnlineEngine(n, n, R, ns, 0.1, step, pol, t0=4)
        e.set_image_factors(A0, B0)
        return e

    full = engine()
    out_full = full.run(kd, T)
    first = engine()
    out1 = first.run(kd, T1)
    checkpoint.save_engine(first, tmp_path / "ck")
    second = tt.OnlineEngine(n, n, R, ns, 0.1, step, pol)
    checkpoint.load_engine(second, tmp_path / "ck")
    assert second.t == 4 + T1 and second.frame == T1
    out2 = second.run(kd, T - T1)
    torch.cuda.synchronize()
    for k in ("gamma", "cost", "mu", "cnt", "rows", "alpha"):
        got = torch.cat([out1[k], out2[k]]).cpu().numpy()
        np.testing.assert_array_equal(got, out_full[k].cpu().numpy(), err_msg=k)
    np.testing.assert_array_equal(second.ah.cpu().numpy(), full.ah.cpu().numpy())
    np.testing.assert_array_equal(second.bh.cpu().numpy(), full.bh.cpu().numpy())
    np.testing.assert_array_equal(second.alpha_bar.cpu().numpy(), full.alpha_bar.cpu().numpy())
    np.testing.assert_array_equal(second.philox_pos.cpu().numpy(), full.philox_pos.cpu().numpy())
    bad = tt.OnlineEngine(n, n, R + 1, ns, 0.1, step, pol)
    with pytest.raises(ValueError):
        checkpoint.load_engine(bad, tmp_path / "ck")
