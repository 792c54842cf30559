"""CPU, world size 2 over gloo: the multi-GPU decompositions.

* row sharding (config 4): per-rank partials all-reduced with
  torch.distributed (gloo) then a redundant solve reproduce the unsharded
  oracle step (which is pinned to the reference);
* slice sharding (config 3): the partition covers every slice exactly once.
"""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import tt_oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _case(seed=3, n1=64, n2=48, R=5, S=20):
    rng = np.random.default_rng(seed)
    A = (rng.standard_normal((n1, R)) + 1j * rng.standard_normal((n1, R))) / np.sqrt(2 * n1)
    B = (rng.standard_normal((n2, R)) + 1j * rng.standard_normal((n2, R))) / np.sqrt(2 * n2)
    rows = rng.choice(n1, size=S, replace=False)
    Ah, Bh = O.fft_cols(A), O.fft_cols(B)
    g = rng.standard_normal(R) + 1j * rng.standard_normal(R)
    Y = (Ah[rows] * g[None, :]) @ Bh.T + 0.05 * (rng.standard_normal((S, n2)) + 1j * rng.standard_normal((S, n2)))
    return A, B, Ah, Bh, rows, Y


def _worker(rank, world, port, out):
    import torch

    from paper_1609_04104_b200.sharding import row_partition, slice_partition

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    A, B, Ah, Bh, rows, Y = _case()
    n1, R = Ah.shape
    r0, r1 = row_partition(n1, world, rank)
    part = O.row_shard_partials(Ah, Bh, rows, Y, r0, r1)
    # pack the payload as float64 (re, im) and all-reduce — one collective per frame
    payload = np.concatenate([part["W"].ravel(), part["GA"].ravel(), [part["yn"] + 1j * part["an"]]])
    buf = torch.from_numpy(np.stack([payload.real, payload.imag], axis=1).copy())
    dist.all_reduce(buf, op=dist.ReduceOp.SUM)
    red_c = buf[:, 0].numpy() + 1j * buf[:, 1].numpy()
    ny = Bh.shape[0]
    red = dict(W=red_c[:ny * R].reshape(ny, R), GA=red_c[ny * R:ny * R + R * R].reshape(R, R),
               yn=red_c[-1].real, an=red_c[-1].imag)
    A_own, B_new, gamma, cost = O.row_shard_finish(Ah, Bh, rows, Y, r0, r1, red, 0.2, 5, 0.03)
    gathered = [None] * world
    dist.all_gather_object(gathered, (r0, r1, A_own, B_new, gamma, cost))
    sl = [None] * world
    dist.all_gather_object(sl, slice_partition(64, world, rank))
    if rank == 0:
        out.put((gathered, sl))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_row_sharded_step_equals_unsharded(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    gathered, sl = q.get(timeout=120)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    A, B, Ah, Bh, rows, Y = _case()
    idx = O.rows_to_entries(rows, Bh.shape[0])
    want = O.track_step(A, B, 5, 0.0, Y.ravel(), idx, "fourier", 0.2, ("fixed", 0.03))
    Ah_want, Bh_want = O.fft_cols(want["A"]), O.fft_cols(want["B"])
    A_sh = np.zeros_like(Ah)
    for (r0, r1, A_own, B_new, gamma, cost) in gathered:
        A_sh[r0:r1] = A_own
        np.testing.assert_allclose(gamma, want["gamma"], rtol=1e-10)
        np.testing.assert_allclose(B_new, Bh_want, rtol=1e-10, atol=1e-12)
        assert cost == pytest.approx(want["cost"], rel=1e-10)
    np.testing.assert_allclose(A_sh, Ah_want, rtol=1e-10, atol=1e-12)
    # every rank holds an identical replica of Bh and gamma
    for g in gathered[1:]:
        np.testing.assert_array_equal(g[3], gathered[0][3])
    # slice sharding covers 64 slices exactly once
    flat = sorted(s for part in sl for s in part)
    assert flat == list(range(64))


def test_partitions():
    from paper_1609_04104_b200.sharding import block_range, row_partition, slice_partition

    for n in (1, 7, 64, 1024):
        for parts in (1, 2, 3, 4, 8):
            cover = []
            for p in range(parts):
                b, e = block_range(n, parts, p)
                assert e - b in (n // parts, n // parts + 1)
                cover += list(range(b, e))
            assert cover == list(range(n))
    assert row_partition(1024, 8, 7) == (896, 1024)
    assert slice_partition(64, 8, 2) == list(range(16, 24))
