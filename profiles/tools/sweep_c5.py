#!/usr/bin/env python
"""BASELINE.json configs[4] (C5): shape sweep for roofline characterisation.

Nx = Ny in {128, 256, 512, 1024}, R in {4, 8, 16, 32, 64}, sampling fraction in
{10%, 25%, 50%}, T = 64 frames of the seeded cine phantom (period 16), masks
both fixed (variable-density rows, alpha = -1, Philox stream per point) and
informative (K = ceil(frac N) trials with replacement, forced DC, beta = 0.1).
Each point runs what `bench.py` times for config 2: the fused online loop
(`tt_rows_kernel`, T frames in one launch) and the reconstruction of all T frames in k-space
(Ah diag(gamma) Bh^T, what run_adaptive records for k-space data), device-timed with
CUDA events, L2 flushed between steps. Reported per point:

* fps            reconstructed frames / s (device, inputs resident)
* us_frame_trk   tracking kernel time per frame
* hbm_frac       SURVEY §8d byte model (B_upd + B_rec) x fps / measured HBM peak
* hbm_frac_trk   B_upd x tracking frames/s / peak (the tracking kernel alone)
* fp32_frac_trk  F_upd (separable) x tracking frames/s / fp32 CUDA-core peak
* cpu_fps        the oracle port of the reference algorithm (numpy SVD ridge,
                 pocketfft, all host threads) on the first few frames of the
                 same point (fixed masks only; same cost for informative ones)

Output: one JSON object per point on stdout and in --out (jsonl).
Usage: python profiles/tools/sweep_c5.py [--n 128 256] [--R 4 8] [--frac .1] [--no-cpu]
"""

from __future__ import annotations

import argparse
import itertools
import json
import math
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import bench  # noqa: E402  (helpers: ClockSampler, measured_peaks, init_factors)

CPU_FRAMES = {128: 16, 256: 8, 512: 3, 1024: 2}
CLUSTER = 0  # --cluster: CTAs per slice (0: the library's choice)


def byte_model(n, R, S, informative):
    b_upd = 8 * S * n + 4 * S + 16 * R * (2 * n) + 8 * R + (8 * n if informative else 0)
    b_rec = 8 * n * n
    f_sep = 16 * S * n * R + 16 * (S + n) * R * R + 10 * R * 2 * n * math.log2(n) + 16 * R * 2 * n
    return b_upd, b_rec, f_sep


def run_point(n, R, frac, kind, ks_dev, clean_dev, T, steps, warmup, flush, hbm_peak, fp32_peak):
    import torch

    import paper_1609_04104_b200 as tt
    from paper_1609_04104_b200 import _lib as L
    from paper_1609_04104_b200 import _ops as K

    lib = L.lib()
    cfg = dict(n=n, R=R)
    A0, B0 = bench.init_factors(cfg, [0])
    S_max = int(math.ceil(frac * n))
    if kind == "fixed":
        gen = np.random.Generator(np.random.Philox(key=2024 + n * 1000 + R))
        tab = np.zeros((T, 1, S_max), np.int64)
        for f in range(T):
            tab[f, 0] = tt.variable_density_rows(n, -1.0, frac, gen)
        pol = tt.StaticRows(tab, np.full((T, 1), S_max))
    else:
        pol = tt.Informative(k=S_max, forced=(0,), beta=0.1, key0=2024, key1=n * 1000 + R)
    lam = 0.05
    eng = tt.OnlineEngine(n, n, R, 1, lam, tt.Fixed(0.01), pol, cluster=CLUSTER)
    eng.set_image_factors(A0, B0)
    ah0, bh0 = eng.ah.clone(), eng.bh.clone()
    ahf, bhf = torch.empty_like(ah0), torch.empty_like(bh0)
    out = eng.make_outputs(T, history=True)
    X = torch.empty(T, n, n, dtype=torch.complex64, device=ks_dev.device)
    args = eng.args(ks_dev, T, out, ah_in=ah0, bh_in=bh0, ah_out=ahf, bh_out=bhf, frame0=0, t0=1)
    stream = torch.cuda.current_stream()

    def step(evs=None):
        eng.philox_pos.zero_()
        eng.alpha_bar.zero_()
        if evs:
            evs[0].record(stream)
        K.track_rows(args)
        if evs:
            evs[1].record(stream)
        # the k-space frames Ah diag(gamma) Bh^T (run_adaptive's record for k-space data, as bench.py's step)
        L.check(lib.tt_reconstruct(stream.cuda_stream, T, n, n, R, out["ah"].data_ptr(), out["bh"].data_ptr(),
                                   out["gamma"].data_ptr(), X.data_ptr()), "reconstruct")
        if evs:
            evs[2].record(stream)

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    eng.check_status()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(steps)]
    with bench.ClockSampler(torch.cuda.current_device()) as clk:
        for i in range(steps):
            flush.zero_()
            step(evs[i])
        torch.cuda.synchronize()
    eng.check_status()
    tot = sum(e[0].elapsed_time(e[2]) for e in evs) / 1e3
    trk = sum(e[0].elapsed_time(e[1]) for e in evs) / 1e3
    fps = T * steps / tot
    fps_trk = T * steps / trk
    S_avg = float(out["cnt"].double().mean())
    b_upd, b_rec, f_sep = byte_model(n, R, S_avg, kind == "informative")
    nm = ((clean_dev - X).abs().pow(2).sum((-1, -2)) / clean_dev.abs().pow(2).sum((-1, -2))).double().sqrt()
    return {
        "n": n, "R": R, "frac": frac, "mask": kind, "T": T, "cluster": eng.cluster, "rows_avg": S_avg,
        "fps": fps, "us_frame": 1e6 / fps, "us_frame_trk": 1e6 / fps_trk,
        "hbm_frac": (b_upd + b_rec) * fps / 1e9 / hbm_peak,
        "hbm_frac_trk": b_upd * fps_trk / 1e9 / hbm_peak,
        "fp32_frac_trk": f_sep * fps_trk / 1e12 / fp32_peak,
        "bytes_upd": b_upd, "bytes_rec": b_rec, "flops_upd_sep": f_sep,
        "last_nrmse": float(nm[-1]), "mean_nrmse": float(nm.mean()),
        "clocks": clk.summary(),
    }


def cpu_point(n, R, frac, ks_np, A0, B0, frames):
    from oracle import tt_oracle as O

    gen = np.random.Generator(np.random.Philox(key=2024 + n * 1000 + R))
    pol = {"kind": "static", "rows": [O.vd_rows(n, -1.0, frac, gen.random) for _ in range(frames)]}
    O.online_run(ks_np[:1], A0[0], B0[0], 0.05, ("fixed", 0.01), dict(pol, rows=pol["rows"][:1]))  # warm
    t0 = time.perf_counter()
    O.online_run(ks_np[:frames], A0[0], B0[0], 0.05, ("fixed", 0.01), pol)
    dt = time.perf_counter() - t0
    return frames / dt, dt


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, nargs="*", default=[128, 256, 512, 1024])
    ap.add_argument("--R", type=int, nargs="*", default=[4, 8, 16, 32, 64])
    ap.add_argument("--frac", type=float, nargs="*", default=[0.1, 0.25, 0.5])
    ap.add_argument("--mask", nargs="*", default=["fixed", "informative"])
    ap.add_argument("--T", type=int, default=64)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cluster", type=int, default=0, help="CTAs per slice (0: the library's choice)")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "sweep_c5.jsonl"))
    args = ap.parse_args()
    global CLUSTER
    CLUSTER = args.cluster

    import torch

    from paper_1609_04104_b200 import _lib as L
    from paper_1609_04104_b200.phantom import cine_phantom

    torch.cuda.set_device(0)
    L.load()
    dev = torch.device("cuda", 0)
    hbm_peak, sm_max, _ = bench.measured_peaks()
    fp32_peak = 148 * 128 * 2 * sm_max * 1e6 / 1e12
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    fo = open(args.out, "a")
    for n in args.n:
        ph = cine_phantom(n, n, args.T, period=16.0, seed=2024)
        ks_np = np.ascontiguousarray(ph.kspace)
        ks_dev = torch.from_numpy(ks_np).to(dev).reshape(args.T, 1, n, n)
        clean_dev = torch.from_numpy(np.ascontiguousarray(ph.clean)).to(dev)
        for R, frac in itertools.product(args.R, args.frac):
            cpu = None
            if not args.no_cpu and "fixed" in args.mask:
                A0, B0 = bench.init_factors(dict(n=n, R=R), [0])
                fps, dt = cpu_point(n, R, frac, ks_np, A0, B0, CPU_FRAMES.get(n, 2))
                cpu = {"fps": fps, "seconds": dt, "frames": CPU_FRAMES.get(n, 2), "cores": os.cpu_count(),
                       "kind": "port"}
            for kind in args.mask:
                try:
                    rec = run_point(n, R, frac, kind, ks_dev, clean_dev, args.T, args.steps, args.warmup, flush,
                                    hbm_peak, fp32_peak)
                except Exception as e:  # unsupported shapes are reported, not skipped silently
                    rec = {"n": n, "R": R, "frac": frac, "mask": kind, "error": f"{type(e).__name__}: {e}"}
                rec["cpu"] = cpu
                if cpu and "fps" in rec:
                    rec["speedup_vs_cpu"] = rec["fps"] / cpu["fps"]
                s = json.dumps(rec)
                print(s, flush=True)
                fo.write(s + "\n")
                fo.flush()
        del ks_dev, clean_dev
        torch.cuda.empty_cache()
    return 0


if __name__ == "__main__":
    sys.exit(main())
