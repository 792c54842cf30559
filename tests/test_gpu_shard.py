"""GPU: the row-sharded two-phase step (config 4 decomposition) on one GPU,
ranks emulated one after the other (no kernel waits on another): the summed
payloads give every rank the same gamma and the concatenated owned rows
equal the unsharded fused run."""

import numpy as np
import pytest

from conftest import rel
from oracle import tt_oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world,n,R,S,T", [(1, 128, 10, 32, 3), (2, 128, 10, 32, 4), (4, 256, 16, 64, 3),
                                           (3, 200, 12, 40, 3)])
def test_row_sharded_equals_unsharded(world, n, R, S, T):
    import torch

    import paper_1609_04104_b200 as tt
    from paper_1609_04104_b200.engine import RowShardedEngine
    from paper_1609_04104_b200.phantom import cine_phantom

    ph = cine_phantom(n, n, T, period=8.0, seed=5)
    A0, B0 = O.random_subspace(n, n, R, seed=6)
    gen = np.random.Generator(np.random.Philox(key=13))
    rows = np.stack([O.vd_rows(n, -1.0, S / n, gen.random) for _ in range(T)])
    ks = torch.from_numpy(ph.kspace).cuda()
    # unsharded reference run (fused kernel)
    ref = tt.run_online(ph.kspace, A0[None], B0[None], 0.1, tt.Fixed(0.01),
                        tt.StaticRows(rows[:, None, :], np.full((T, 1), S)))
    ranks = []
    for r in range(world):
        e = RowShardedEngine(n, n, R, 0.1, tt.Fixed(0.01), rows, np.full(T, S), world, r, allreduce=lambda t: None)
        e.set_image_factors(A0, B0)
        ranks.append((e, e.make_outputs(T)))
    for f in range(T):
        for e, _ in ranks:
            e.partial(ks, f)
        xw = sum(e.xw for e, _ in ranks)
        xg = sum(e.xg for e, _ in ranks)
        for e, out in ranks:
            e.xw.copy_(xw)
            e.xg.copy_(xg)
            e.finish(ks, f, out, f)
    torch.cuda.synchronize()
    g0 = ranks[0][1]["gamma"].cpu().numpy()
    for e, out in ranks:
        np.testing.assert_array_equal(out["gamma"].cpu().numpy(), g0)       # identical on every rank
        np.testing.assert_array_equal(e.bh.cpu().numpy(), ranks[0][0].bh.cpu().numpy())
    for f in range(T):
        assert rel(g0[f], ref.gamma[f, 0]) < 1e-5
    ah = torch.cat([e.ah for e, _ in ranks]).cpu().numpy()
    assert rel(O.fft_cols(ah, inverse=True), ref.final_A[0]) < 1e-5
    assert rel(O.fft_cols(ranks[0][0].bh.cpu().numpy(), inverse=True), ref.final_B[0]) < 1e-5
    np.testing.assert_allclose(ranks[0][1]["cost"].cpu().numpy(), ref.cost[:, 0], rtol=1e-5)
