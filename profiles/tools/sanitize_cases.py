"""Tiny-shape runs of every kernel family, for compute-sanitizer (memcheck / racecheck / synccheck).

Usage (GPU box):  compute-sanitizer --tool racecheck python profiles/tools/sanitize_cases.py [case ...]
Cases: rows_static16, rows_static2, rows_inf16, rows_inf2, rows_wor, shard_fused, shard3, entries, patched,
fft, recon, draws. Default: all. Shapes are small so the instrumented run takes seconds per case.
"""

import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))

import numpy as np
import torch

import paper_1609_04104_b200 as tt
from paper_1609_04104_b200 import _ops as K
from paper_1609_04104_b200.phantom import cine_phantom


def _rand_subspace(n1, n2, R, seed):
    g = np.random.default_rng(seed)
    A = (g.standard_normal((n1, R)) + 1j * g.standard_normal((n1, R))) / np.sqrt(2 * n1)
    B = (g.standard_normal((n2, R)) + 1j * g.standard_normal((n2, R))) / np.sqrt(2 * n2)
    return A, B


def _vd_table(n, S, T, key):
    gen = np.random.Generator(np.random.Philox(key=key))
    return np.stack([tt.variable_density_rows(n, -1.0, S / n, gen) for _ in range(T)])


def rows_case(cluster, informative, replacement=True, n=64, R=6, T=3):
    ph = cine_phantom(n, n, T, period=8.0, seed=1)
    A0, B0 = _rand_subspace(n, n, R, 2)
    if informative:
        kw = {} if replacement else {"replacement": False}
        pol = tt.Informative(k=16, forced=(0, 1, n - 1), beta=0.1, key0=7, **kw)
    else:
        S = 16
        pol = tt.StaticRows(_vd_table(n, S, T, 3)[:, None, :], np.full((T, 1), S))
    eng = tt.OnlineEngine(n, n, R, 1, 0.1, tt.Fixed(0.01), pol, cluster=cluster)
    eng.set_image_factors(A0[None], B0[None])
    kd = torch.from_numpy(ph.kspace[:, None].astype(np.complex64)).cuda()
    out = eng.run(kd, T)
    eng.reconstruct(out)
    torch.cuda.synchronize()
    eng.check_status()


def shard_case(fused, ranks=3, n=96, R=6, S=24, T=3):
    ph = cine_phantom(n, n, T, period=8.0, seed=4)
    A0, B0 = _rand_subspace(n, n, R, 5)
    rows = _vd_table(n, S, T, 6)
    e = tt.LocalShardedEngine(n, n, R, 0.1, tt.Fixed(0.01), rows, np.full(T, S), ranks, fused=fused)
    e.set_image_factors(A0, B0)
    e.run(torch.from_numpy(ph.kspace).cuda(), T, graph=False)
    torch.cuda.synchronize()
    e.check_status()


def entries_case(n=32, R=4, T=3):
    ph = cine_phantom(n, n, T, period=8.0, seed=8)
    A0, B0 = _rand_subspace(n, n, R, 9)
    pol = tt.InformativeEntries(k=200, forced=(0, 1), beta=0.1, key0=11)
    eng = tt.EntryEngine(n, n, R, 0.1, tt.Fixed(0.01), pol)
    eng.set_image_factors(A0, B0)
    eng.run(torch.from_numpy(ph.kspace.astype(np.complex64)).cuda(), T, graph=False)
    torch.cuda.synchronize()
    eng.check_status()


def patched_case(N=32, n=16, rho=3, T=4, warm=1):
    grid = tt.PatchGrid((N, N), n, n, rho)
    rng = np.random.Generator(np.random.Philox(5))
    A0s, B0s = tt.init_patch_factors(grid, rng)
    masks = [tt.full_entries((N, N))] * warm + [tt.draw_frame_entries("variable_density", (N, N), rng, 0.3)
                                                 for _ in range(T - warm)]
    g = np.random.default_rng(6)
    frames = g.standard_normal((T, N, N)) + 1j * g.standard_normal((T, N, N))
    tt.run_tracking_patched(frames, grid, 0.05, tt.Fixed(0.01), masks, warm_n=warm, warm_epochs=2, epochs=2,
                            rng=rng, reshuffle=True, A0s=A0s, B0s=B0s)
    torch.cuda.synchronize()


def fft_case():
    for n in (1, 7, 64, 100, 256):
        x = torch.randn(3, n, 5, dtype=torch.complex64, device="cuda")
        K.fft_cols(x)
        K.fft_cols(x, inverse=True)
    torch.cuda.synchronize()


def recon_case():
    a = torch.randn(4, 70, 9, dtype=torch.complex64, device="cuda")
    b = torch.randn(4, 66, 9, dtype=torch.complex64, device="cuda")
    g = torch.randn(4, 9, dtype=torch.complex64, device="cuda")
    K.reconstruct(a, b, g)
    torch.cuda.synchronize()


def draws_case():
    rng = np.random.Generator(np.random.Philox(3))
    p = np.random.default_rng(1).random(300)
    p /= p.sum()
    d = tt.SamplingDistribution(p, "rows")
    tt.draw_samples(d, 40, True, rng, forced=[0, 5])
    tt.draw_samples(d, 40, False, rng, forced=[0, 5])
    tt.variable_density_rows(128, -1.0, 0.25, rng)
    torch.cuda.synchronize()


CASES = {
    "rows_static16": lambda: rows_case(16, False),
    "rows_static2": lambda: rows_case(2, False),
    "rows_inf16": lambda: rows_case(16, True),
    "rows_inf2": lambda: rows_case(2, True),
    "rows_wor": lambda: rows_case(4, True, replacement=False),
    "shard_fused": lambda: shard_case(True),
    "shard3": lambda: shard_case(False),
    "entries": entries_case,
    "patched": patched_case,
    "fft": fft_case,
    "recon": recon_case,
    "draws": draws_case,
}

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for nm in names:
        CASES[nm]()
        print("case ok:", nm, flush=True)
