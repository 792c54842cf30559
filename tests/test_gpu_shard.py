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


@pytest.mark.parametrize("ranks,n,R,S,T", [(1, 128, 10, 32, 3), (4, 256, 16, 64, 4), (3, 200, 12, 40, 3),
                                           (8, 512, 32, 64, 3)])
def test_local_multi_rank_launch_equals_unsharded(ranks, n, R, S, T):
    """Every rank of the sharding as a cluster of one launch (phase 1), the payload slots summed on the
    device, phase 2: equals the unsharded fused run and the host-reduced emulation; graph == eager; the
    fused cooperative launch (both phases of every frame, in-kernel reduction, GB split over the ranks)
    agrees with the 3-launch frames to rounding."""
    import torch

    import paper_1609_04104_b200 as tt
    from paper_1609_04104_b200.phantom import cine_phantom

    ph = cine_phantom(n, n, T, period=8.0, seed=15)
    A0, B0 = O.random_subspace(n, n, R, seed=16)
    gen = np.random.Generator(np.random.Philox(key=17))
    rows = np.stack([O.vd_rows(n, -1.0, S / n, gen.random) for _ in range(T)])
    ks = torch.from_numpy(ph.kspace).cuda()
    ref = tt.run_online(ph.kspace, A0[None], B0[None], 0.1, tt.Fixed(0.01),
                        tt.StaticRows(rows[:, None, :], np.full((T, 1), S)))
    outs = []
    for fused, graph in ((False, True), (False, False), (True, False)):
        e = tt.LocalShardedEngine(n, n, R, 0.1, tt.Fixed(0.01), rows, np.full(T, S), ranks, fused=fused)
        e.set_image_factors(A0, B0)
        out = e.run(ks, T, graph=graph)
        torch.cuda.synchronize()
        e.check_status()
        outs.append(({k: v.cpu().numpy() for k, v in out.items()}, e.ah.cpu().numpy(), e.bh.cpu().numpy()))
    # graph == eager bit for bit; the fused single launch sums GB over the ranks' column subsets (another
    # fp64 order), so it agrees to rounding
    for k in outs[0][0]:
        np.testing.assert_array_equal(outs[0][0][k], outs[1][0][k])
    np.testing.assert_array_equal(outs[0][1], outs[1][1])
    np.testing.assert_array_equal(outs[0][2], outs[1][2])
    fo = outs[2]
    for f in range(T):
        assert rel(fo[0]["gamma"][f], outs[0][0]["gamma"][f]) < 1e-5, f
    assert rel(fo[1], outs[0][1]) < 1e-5 and rel(fo[2], outs[0][2]) < 1e-5
    np.testing.assert_allclose(fo[0]["cost"], outs[0][0]["cost"], rtol=1e-5)
    out, ah, bh = outs[0]
    # the fp32 W partials are summed over the ranks in another order than the unsharded kernel's k
    # tiles (~1e-5 at 8 ranks, R = 32): the BASELINE parity bar, 1e-4 relative, is the tolerance
    for f in range(T):
        assert rel(out["gamma"][f], ref.gamma[f, 0]) < 1e-4, f
    assert rel(O.fft_cols(ah, inverse=True), ref.final_A[0]) < 1e-4
    assert rel(O.fft_cols(bh, inverse=True), ref.final_B[0]) < 1e-4
    np.testing.assert_allclose(out["cost"], ref.cost[:, 0], rtol=1e-4)


def test_rank_without_samples_still_steps():
    """A rank whose row block holds no sampled row in a frame must still solve (gamma is global) and
    scale its rows by the step's cfac: only the top rows are sampled here, so most ranks are empty."""
    import torch

    import paper_1609_04104_b200 as tt
    from paper_1609_04104_b200.phantom import cine_phantom

    n, R, S, T, ranks = 128, 8, 12, 3, 8
    ph = cine_phantom(n, n, T, period=8.0, seed=25)
    A0, B0 = O.random_subspace(n, n, R, seed=26)
    rows = np.stack([np.arange(S) + f for f in range(T)])  # rows 0..13: ranks 1..7 see none
    ks = torch.from_numpy(ph.kspace).cuda()
    ref = tt.run_online(ph.kspace, A0[None], B0[None], 0.1, tt.Fixed(0.01),
                        tt.StaticRows(rows[:, None, :], np.full((T, 1), S)))
    e = tt.LocalShardedEngine(n, n, R, 0.1, tt.Fixed(0.01), rows, np.full(T, S), ranks)
    e.set_image_factors(A0, B0)
    out = e.run(ks, T)
    torch.cuda.synchronize()
    for f in range(T):
        assert rel(out["gamma"][f].cpu().numpy(), ref.gamma[f, 0]) < 1e-5
    assert rel(O.fft_cols(e.ah.cpu().numpy(), inverse=True), ref.final_A[0]) < 1e-5


@pytest.mark.parametrize("world,n,R,K,T", [(2, 128, 10, 24, 5), (3, 200, 12, 30, 4)])
def test_row_sharded_informative_equals_unsharded(world, n, R, K, T):
    """Informative draws under row sharding, ranks emulated one after the other on one GPU (no kernel waits
    on another): each rank's row energies (zero elsewhere) summed on the host stand in for the energy
    all-reduce, every rank's scores kernel and phase-1 draw give the same rows, the summed payloads the
    same gamma; rows, gamma and factors equal the unsharded informative run."""
    import torch

    import paper_1609_04104_b200 as tt
    from paper_1609_04104_b200.engine import RowShardedEngine
    from paper_1609_04104_b200.phantom import cine_phantom

    ph = cine_phantom(n, n, T, period=8.0, seed=35)
    A0, B0 = O.random_subspace(n, n, R, seed=36)
    pol = tt.Informative(k=K, forced=(0, 1, n - 1), beta=0.1, key0=17, pos0=5)
    ks = torch.from_numpy(ph.kspace).cuda()
    ref = tt.run_online(ph.kspace, A0[None], B0[None], 0.1, tt.Fixed(0.01), pol)
    ranks = []
    for r in range(world):
        e = RowShardedEngine(n, n, R, 0.1, tt.Fixed(0.01), pol, None, world, r, allreduce=lambda t: None)
        e.set_image_factors(A0, B0)
        ranks.append((e, e.make_outputs(T)))
    for f in range(T):
        for e, _ in ranks:
            e._energy()
        en = sum(e.energy for e, _ in ranks)
        for e, out in ranks:
            e.energy.copy_(en)
            e._scores()
            e._out, e._fo = out, f
            e._phase1(ks, f)
        xw = sum(e.xw for e, _ in ranks)
        xg = sum(e.xg for e, _ in ranks)
        for e, out in ranks:
            e.xw.copy_(xw)
            e.xg.copy_(xg)
            e.finish(ks, f, out, f)
    torch.cuda.synchronize()
    for e, _ in ranks:
        e.check_status()
    outs = [{k: v.cpu().numpy() for k, v in out.items()} for _, out in ranks]
    for f in range(T):
        got = outs[0]["rows"][f, :outs[0]["cnt"][f]]
        np.testing.assert_array_equal(got, ref.rows[f][0])
        for o in outs[1:]:
            np.testing.assert_array_equal(o["rows"][f], outs[0]["rows"][f])
            np.testing.assert_array_equal(o["gamma"][f], outs[0]["gamma"][f])
        assert rel(outs[0]["gamma"][f], ref.gamma[f, 0]) < 1e-5
    ah = torch.cat([e.ah for e, _ in ranks]).cpu().numpy()
    assert rel(O.fft_cols(ah, inverse=True), ref.final_A[0]) < 1e-5
    assert rel(O.fft_cols(ranks[0][0].bh.cpu().numpy(), inverse=True), ref.final_B[0]) < 1e-5


@pytest.mark.parametrize("informative", [False, True])
def test_row_sharded_graph_with_nccl_world1(informative):
    """The captured T-frame chain with real NCCL collectives (a one-rank NCCL process group on this GPU:
    the collectives are graph nodes, nothing waits on another rank): graph replay == eager frames bit for
    bit, == the unsharded run to rounding; replay after restore() repeats the bits."""
    import os

    import torch
    import torch.distributed as dist

    import paper_1609_04104_b200 as tt
    from paper_1609_04104_b200.engine import RowShardedEngine
    from paper_1609_04104_b200.phantom import cine_phantom

    n, R, T, S = 128, 8, 6, 32
    ph = cine_phantom(n, n, T, period=8.0, seed=45)
    A0, B0 = O.random_subspace(n, n, R, seed=46)
    ks = torch.from_numpy(ph.kspace).cuda()
    if informative:
        pol = tt.Informative(k=S, forced=(0,), beta=0.1, key0=3)
        args = (pol, None)
    else:
        gen = np.random.Generator(np.random.Philox(key=47))
        rows = np.stack([O.vd_rows(n, -1.0, S / n, gen.random) for _ in range(T)])
        pol = tt.StaticRows(rows[:, None, :], np.full((T, 1), S))
        args = (rows, np.full(T, S))
    ref = tt.run_online(ph.kspace, A0[None], B0[None], 0.1, tt.Fixed(0.01), pol)
    own_pg = not dist.is_initialized()
    if own_pg:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        import socket

        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        os.environ["MASTER_PORT"] = str(s.getsockname()[1])
        s.close()
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        runs = []
        for graph in (False, True):
            e = RowShardedEngine(n, n, R, 0.1, tt.Fixed(0.01), *args, world=1, rank_id=0)
            e.set_image_factors(A0, B0)
            init = e.save()
            out = e.run(ks, T, graph=graph)
            torch.cuda.synchronize()
            e.check_status()
            runs.append(({k: v.cpu().numpy() for k, v in out.items()}, e.ah.cpu().numpy(), e.bh.cpu().numpy()))
            if graph:  # replay from the restored initial state
                e.restore(init)
                e.replay()
                torch.cuda.synchronize()
                np.testing.assert_array_equal(e.ah.cpu().numpy(), runs[-1][1])
                np.testing.assert_array_equal(out["gamma"].cpu().numpy(), runs[-1][0]["gamma"])
    finally:
        if own_pg:
            dist.destroy_process_group()
    for k in runs[0][0]:
        np.testing.assert_array_equal(runs[0][0][k], runs[1][0][k])
    np.testing.assert_array_equal(runs[0][1], runs[1][1])
    for f in range(T):
        assert rel(runs[0][0]["gamma"][f], ref.gamma[f, 0]) < 1e-5
    assert rel(O.fft_cols(runs[0][1], inverse=True), ref.final_A[0]) < 1e-5
