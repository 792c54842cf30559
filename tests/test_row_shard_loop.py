"""CPU, world size 2 over gloo: the row-sharded engine's host orchestration (engine.RowShardLoop, the loop
RowShardedEngine runs on the GPUs) with the phases restated in numpy on the kernel's payload layout
(sharding.pack_payload / unpack_payload): per frame [row energies -> sum all-reduce -> scores -> the same
draw on every rank] -> phase 1 partials packed -> ONE all-reduce of the payload -> phase 2 unpacked,
redundant solve, update of the owned rows and the replicated Bh. Over a whole sequence (static rows and
informative draws) the ranks' concatenated rows and Bh equal the unsharded oracle loop (pinned to the
reference), and the collective count is one payload all-reduce per frame (+ one energy all-reduce for
informative draws)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import tt_oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


N, R, T, LAM, MU, K, BETA, KEY = 48, 4, 7, 0.1, 0.02, 12, 0.1, (9, 0)


def _problem():
    from paper_1609_04104_b200.phantom import cine_phantom

    ph = cine_phantom(N, N, T, period=8.0, seed=3)
    A0, B0 = O.random_subspace(N, N, R, seed=4)
    gen = np.random.Generator(np.random.Philox(key=5))
    rows = [O.vd_rows(N, -1.0, 0.25, gen.random) for _ in range(T)]
    return ph, A0, B0, rows


def _worker(rank, world, port, informative, q):
    import torch
    import torch.distributed as dist

    from paper_1609_04104_b200.engine import RowShardLoop
    from paper_1609_04104_b200.sharding import pack_payload, payload_doubles, row_partition, unpack_payload

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ph, A0, B0, rows = _problem()
    calls = []

    def allreduce(t):
        calls.append(t.numel())
        dist.all_reduce(t, op=dist.ReduceOp.SUM)

    class HostRowShard(RowShardLoop):
        def __init__(self):
            self.r0, self.r1 = row_partition(N, world, rank)
            Ah, self.Bh = O.fft_cols(A0), O.fft_cols(B0)
            self.Ah = Ah.copy()  # only rows [r0, r1) are this rank's; the rest is never read below
            self.informative = informative
            self.payload = torch.zeros(payload_doubles(N, R), dtype=torch.float64)
            self.energy = torch.zeros(N, R, dtype=torch.float64)
            self.allreduce = allreduce
            self.t, self.frame, self.pos = 1, 0, 0
            self.rows_f = None

        def _energy(self):  # tt_rows_shard_energy: own rows, zeros elsewhere
            e = np.zeros((N, R))
            e[self.r0:self.r1] = np.abs(self.Ah[self.r0:self.r1]) ** 2
            self.energy.copy_(torch.from_numpy(e))

        def _scores(self):  # tt_rows_shard_scores + the blend of row_scores (sampler.py:115-128, :88-92)
            E = self.energy.numpy()
            s = (N * (E / E.sum(axis=0)).sum(axis=1) + R) / (R * (N + N))
            p = O._blend(s / s.sum(), BETA)
            self.rows_f, used = O.draw_rows(p, K, [0], KEY, self.pos)
            self.pos += used

        def _phase1(self, kspace, f):
            rw = self.rows_f if informative else np.asarray(rows[f])
            self.rows_cur = rw
            Y = kspace[f][rw]
            Ah_loc = np.zeros_like(self.Ah)
            Ah_loc[self.r0:self.r1] = self.Ah[self.r0:self.r1]
            part = O.row_shard_partials(Ah_loc, self.Bh, rw, Y, self.r0, self.r1)
            self.payload.copy_(torch.from_numpy(pack_payload(part["W"], part["GA"], part["yn"], part["an"])))

        def _phase2(self, kspace, f, out, fo):
            red = unpack_payload(self.payload.numpy(), N, R)
            rw = self.rows_cur
            A_own, B_new, gamma, cost = O.row_shard_finish(self.Ah, self.Bh, rw, kspace[f][rw], self.r0, self.r1,
                                                           red, LAM, self.t, MU)
            self.Ah[self.r0:self.r1] = A_own
            self.Bh = B_new
            out.append((np.sort(rw), gamma, cost))

    eng = HostRowShard()
    out = []
    eng.run_frames(ph.kspace.astype(np.complex128), T, out)
    res = (eng.r0, eng.r1, eng.Ah[eng.r0:eng.r1], eng.Bh, out, calls)
    gathered = [None] * world
    dist.all_gather_object(gathered, res)
    if rank == 0:
        q.put(gathered)
    dist.destroy_process_group()


@pytest.mark.parametrize("informative", [False, True])
def test_row_shard_loop_over_gloo_equals_unsharded(informative):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, informative, q)) for r in range(world)]
    for p in ps:
        p.start()
    gathered = q.get(timeout=300)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    ph, A0, B0, rows = _problem()
    pol = ({"kind": "informative", "k": K, "forced": [0], "beta": BETA, "key": KEY} if informative
           else {"kind": "static", "rows": rows})
    ref = O.online_run(ph.kspace, A0, B0, LAM, ("fixed", MU), pol)
    Ah = np.zeros((N, R), np.complex128)
    for r0, r1, A_own, Bh, out, calls in gathered:
        Ah[r0:r1] = A_own
        np.testing.assert_allclose(Bh, O.fft_cols(ref["final"][1]), rtol=1e-9, atol=1e-12)
        for f, (rw, gamma, cost) in enumerate(out):
            np.testing.assert_array_equal(rw, np.sort(ref["rows"][f]))
            np.testing.assert_allclose(gamma, ref["gamma"][f], rtol=1e-9, atol=1e-12)
            assert cost == pytest.approx(ref["cost"][f], rel=1e-9)
        # one payload all-reduce per frame (+ one energy all-reduce per frame for informative draws)
        per_frame = [N * R, 2 * N * R + R * (R + 1) + 2] if informative else [2 * N * R + R * (R + 1) + 2]
        assert calls == per_frame * T
    np.testing.assert_allclose(Ah, O.fft_cols(ref["final"][0]), rtol=1e-9, atol=1e-12)
    # the replicas agree exactly
    np.testing.assert_array_equal(gathered[0][3], gathered[1][3])
