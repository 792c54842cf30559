#!/usr/bin/env python
"""Frames/s of the online per-frame MM reconstruction loop on B200.

Default workload = BASELINE.json configs[2] ("c3"), the largest configuration that fits one GPU:
64 independent 256x256 complex64 cine phantom slices, T=100 frames, R=16, lambda=0.05, Fixed
mu=0.01, informative row sampling at 20% (K=52 trials incl. the forced DC line, beta=0.1, Philox
draws per slice). One bench *step* = the whole T-frame online sequence of every slice from the same
initial state: per slice-frame [row scores -> Philox draw -> gather y -> Gram/ridge -> k-space factor
update] in persistent cluster-kernel launches over blocks of frames (`--blocks`, default 4; the state
stays resident across them), each block's reconstructed frames — the k-space estimates Ah diag(gamma)
Bh^T that run_adaptive records for k-space data (experiment.py:242-245, :525) — computed on a second
stream while the next block tracks. `--config c2` (single 256^2 slice, T=200, R=20, K=64 with 16
forced centre lines), `c1`, `c4` and the widening configs select the others.

`value`  = slice-frames reconstructed per second over all ranks (device time, inputs resident, L2
           flushed between steps).
`e2e`    = the same through the public call `run_online` with the truth k-space in pinned host
           memory (H2D) and the reconstructions + per-frame reports read back (D2H) inside the timed
           region.
`--impl reference` times the UNMODIFIED reference package (baseline/_ref, `bench_reference.py`):
its own `run_adaptive` per slice, one process per host core, full T per step.
`--gpus N` without torchrun re-launches itself under `torch.distributed.run` with N ranks. The
64-slice config is sharded over ranks (64/N slices each, no collective, `scaling: strong`); the
single-slice configs run one replica per rank (`scaling: weak`); `c4` under N ranks runs the row
sharding.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

METRIC = "frames/sec reconstructed (online per-frame update) and % HBM roofline, 1–8 B200"


def center_lines(n, m):
    return tuple(list(range(m // 2)) + list(range(n - m // 2, n)))


CONFIGS = {
    "c1": dict(n=128, R=10, T=64, lam=0.1, period=16.0, vd=0.25, mu=0.01, slices=1,
               desc="config 1: 128x128 complex64 cine phantom, T=64, R=10, lambda=0.1, variable-density rows "
                    "25% (32 rows/frame, alpha=-1, Philox), Fixed mu=0.01"),
    "c2": dict(n=256, R=20, T=200, lam=0.05, period=20.0, K=64, forced=center_lines(256, 16), beta=0.1, mu=0.01,
               slices=1, desc="config 2: 256x256 complex64 cine phantom, T=200, R=20, lambda=0.05, informative "
                              "rows K=64 (4x) incl. 16 centre lines, beta=0.1, Philox draws, Fixed mu=0.01"),
    "c3": dict(n=256, R=16, T=100, lam=0.05, period=16.0, K=52, forced=(0,), beta=0.1, mu=0.01, slices=64,
               desc="config 3: 64 independent 256x256 slices, T=100, R=16, 20% informative rows (K=52, forced DC)"),
    "c2e": dict(n=256, R=20, T=200, lam=0.05, period=20.0, entries=0.25, mu=0.01, slices=1, beta=0.1,
                desc="config 2 with entry sampling (run_adaptive's entries mode): 256x256 complex64 cine "
                     "phantom, T=200, R=20, lambda=0.05, informative entries K=16384 (25% of nx*ny trials, "
                     "forced DC), beta=0.1, Philox draws, Fixed mu=0.01"),
    "c2p": dict(n=256, R=4, patch=32, T=200, lam=0.05, period=20.0, vd=0.25, mu=0.01, slices=1, warm_n=5,
                warm_epochs=20,
                desc="per-patch trackers (experiment._run_tracking_patched): 256x256 complex64 cine phantom "
                     "k-space, T=200, 8x8 grid of 32x32 patches with rank 4 each, lambda=0.05, variable-density "
                     "rows 25% (Philox), Fixed mu=0.01, warm-up 5 full frames x 20 epochs, 1 epoch, "
                     "re-projection of every frame"),
    "c2b": dict(n=256, R=20, T=200, lam=0.05, period=20.0, vd=0.25, mu=0.01, slices=1, epochs=4, batch=True,
                desc="multi-epoch batch mode (tracker.run / experiment.run_tracking with epochs > 1): 256x256 "
                     "complex64 cine phantom, T=200, R=20, lambda=0.05, variable-density rows 25% (Philox), "
                     "Fixed mu=0.01, 4 epochs with reshuffling and rebalancing, then the re-projection of every "
                     "frame onto the final subspace"),
    "c4": dict(n=1024, R=32, T=256, lam=0.1, period=16.0, vd=0.125, mu=0.01, slices=1,
               desc="config 4: 1024x1024 complex64 cine phantom, T=256, R=32, lambda=0.1, variable-density rows "
                    "12.5% (128 rows/frame), Fixed mu=0.01 (single GPU, unsharded)"),
}


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clock and throttle reasons sampled during the timed region: NVML polled
    every ~1 ms from a thread (the timed region is tens of ms), falling back to
    `nvidia-smi -lms 100` when NVML is unavailable."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown"}

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
            get_r = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                pynvml.nvmlDeviceGetCurrentClocksThrottleReasons

            def poll():
                while not self._stop.is_set():
                    try:
                        self.samples.append(float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)))
                        r = int(get_r(h))
                        for bit, name in self.REASONS.items():
                            if r & bit:
                                self.reasons.add(name)
                    except Exception:
                        pass
                    time.sleep(0.001)

            self.thread = threading.Thread(target=poll, daemon=True)
            self.thread.start()
        except Exception:
            try:
                self.proc = subprocess.Popen(
                    ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                     "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                     "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "100"],
                    stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
                self.thread = threading.Thread(target=self._read, daemon=True)
                self.thread.start()
            except FileNotFoundError:
                self.proc = None
        return self

    def _read(self):
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                self.samples.append(float(parts[0]))
                self.max_mhz = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    self.reasons.add(nm)

    def __exit__(self, *exc):
        self._stop.set()
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------ data
def make_data(cfg, slice_ids, seed=2024):
    from paper_1609_04104_b200.phantom import cine_phantom

    ks, cl = [], []
    for s in slice_ids:
        ph = cine_phantom(cfg["n"], cfg["n"], cfg["T"], period=cfg["period"], seed=seed, slice_index=s)
        ks.append(ph.kspace)
        cl.append(ph.clean)
    return np.stack(ks, axis=1), np.stack(cl, axis=1)  # (T, ns, n, n)


def init_factors(cfg, slice_ids, seed=7):
    A, B = [], []
    for s in slice_ids:
        rng = np.random.default_rng([seed, s])
        a = (rng.standard_normal((cfg["n"], cfg["R"])) + 1j * rng.standard_normal((cfg["n"], cfg["R"]))) / np.sqrt(2 * cfg["n"])
        b = (rng.standard_normal((cfg["n"], cfg["R"])) + 1j * rng.standard_normal((cfg["n"], cfg["R"]))) / np.sqrt(2 * cfg["n"])
        A.append(a)
        B.append(b)
    return np.stack(A), np.stack(B)


def measured_peaks():
    p = os.path.join(HERE, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), float(d.get("sm_max_mhz", 1965.0)), "measured"
    return 6650.0, 1965.0, "fallback"


# ------------------------------------------------------------------ CPU oracle (reference arm / cpu_baseline)
def patched_masks(cfg, T):
    """Warm frames full, the rest variable-density rows (Philox stream 2024, the device VD draw)."""
    import paper_1609_04104_b200 as tt

    n = cfg["n"]
    gen = np.random.Generator(np.random.Philox(key=2024))
    warm = min(cfg["warm_n"], T)
    full = tt.full_entries((n, n))
    return [full] * warm + [tt.rows_to_entries(O_vd_rows(n, cfg["vd"], gen), n) for _ in range(T - warm)]


def O_vd_rows(n, frac, gen):
    from oracle import tt_oracle as O

    return O.vd_rows(n, -1.0, frac, gen.random)


def patched_init(cfg):
    rng = np.random.default_rng(7)
    k = cfg["n"] // cfg["patch"]
    A, B = [], []
    for _ in range(k * k):
        for out in (A, B):
            z = rng.standard_normal((cfg["patch"], cfg["R"])) + 1j * rng.standard_normal((cfg["patch"], cfg["R"]))
            out.append(z / np.sqrt(2 * cfg["patch"]))
    return np.stack(A), np.stack(B)


def cpu_oracle_fps(cfg, frames, ks, A0, B0):
    from oracle import tt_oracle as O

    if "patch" in cfg:  # streamed frames only (no warm-up), every patch stepped and re-projected
        p = cfg["patch"]
        masks = patched_masks(dict(cfg, warm_n=0), frames)
        A0s, B0s = patched_init(cfg)
        t0 = time.perf_counter()
        O.patched_run(ks[:frames, 0], A0s, B0s, cfg["lam"], ("fixed", cfg["mu"]), p, p, masks, 0, 1, 1, power=False)
        dt = time.perf_counter() - t0
        return frames / dt, dt
    if "entries" in cfg:
        k = int(np.ceil(cfg["entries"] * cfg["n"] ** 2))
        t0 = time.perf_counter()
        O.online_run_entries(ks[:frames, 0], O.fft_cols(A0[0]), O.fft_cols(B0[0]), cfg["lam"], ("fixed", cfg["mu"]),
                             {"kind": "informative", "k": k, "forced": [0], "beta": cfg["beta"], "key": (2024, 0)})
        dt = time.perf_counter() - t0
        return frames / dt, dt
    if "vd" in cfg:
        gen = np.random.Generator(np.random.Philox(key=2024))
        pol = {"kind": "static", "rows": [O.vd_rows(cfg["n"], -1.0, cfg["vd"], gen.random) for _ in range(frames)]}
    else:
        pol = {"kind": "informative", "k": cfg["K"], "forced": list(cfg["forced"]), "beta": cfg["beta"],
               "key": (2024, 0)}
    t0 = time.perf_counter()
    O.online_run(ks[:frames, 0], A0[0], B0[0], cfg["lam"], ("fixed", cfg["mu"]), pol)
    dt = time.perf_counter() - t0
    return frames / dt, dt


REF_CONFIGS = ("c1", "c2", "c3", "c4")  # the BASELINE configs: timed through the reference package itself
REF_FRAMES = {"c4": 8}  # ~1 s per frame at 1024^2: a bounded sample of frames (>= 8 frames)


def reference_sample(args, cfg):
    """Frames per reference step: the config's full T unless bounded (c4, or --ref-frames)."""
    if args.ref_frames > 0:
        return min(cfg["T"], args.ref_frames)
    return min(cfg["T"], REF_FRAMES.get(args.config, cfg["T"]))


def run_reference(args, cfg):
    """The reference arm: the unmodified reference package (bench_reference.py) on the host cores,
    this config's workload, one process per core (single-threaded BLAS each). Rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    if args.config not in REF_CONFIGS:
        return run_reference_port(args, cfg)
    import bench_reference as BR

    try:
        BR.load_reference()
    except Exception as e:  # the install is missing: the pinned oracle port stands in (kind "port")
        print(f"reference package unavailable ({e!r}); timing the oracle port", file=sys.stderr)
        return run_reference_port(args, dict(cfg))
    fr = reference_sample(args, cfg)
    m = BR.measure(dict(cfg, T=fr), args.steps, args.warmup)
    nsl = cfg.get("slices", 1)
    value = m["value"]
    sample = (f"{m['slices']} of {nsl} slices x {fr} of {cfg['T']} frames per step through the stock "
              f"run_adaptive (experiment.py:444-556; SSIM stubbed), {m['procs']} processes x 1 BLAS thread "
              f"on {m['cores']} host cores")
    line = {"metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": m["ms_per_step"], "higher_is_better": True,
            "scaling": "strong" if nsl > 1 else "weak", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
            "config": workload_config(args, cfg), "impl": "reference",
            "same_config": bool(fr == cfg["T"] and m["slices"] == nsl),
            "cpu_baseline": {"value": value, "unit": "frames/s", "cores": m["procs"], "kind": "reference",
                             "sample": sample},
            "e2e": {"value": value, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "extra": {"host_cores": m["cores"], "last_nmse": m["last_nmse"][:4]}}
    print(json.dumps(line), flush=True)
    return 0


def workload_config(args, cfg):
    """The config keys both arms report."""
    return {"workload": cfg["desc"], "frames_per_step": cfg["T"], "slices": cfg.get("slices", 1), "rank": cfg["R"],
            "nx": cfg["n"], "ny": cfg["n"], "l2": "flushed between steps (256 MB write)", "init": "cold start"}


def cpu_baseline_reference(args, cfg):
    """cpu_baseline of our arm: the reference package itself on the box's host cores, a bounded sample
    (one step of min(slices, cores) slices, full T except c4), plus one core alone and the stock
    track_step by itself (SURVEY §8d's two numbers)."""
    import bench_reference as BR

    BR.load_reference()
    fr = reference_sample(args, cfg)
    t0 = time.perf_counter()
    allc = BR.measure(dict(cfg, T=fr), 1, 0, max_slices=BR.host_cores())
    one = BR.measure(dict(cfg, T=min(fr, 50)), 1, 0, max_slices=1)
    ts = BR.track_step_ms(cfg, frames=6 if cfg["n"] >= 1024 else 12)
    dt = time.perf_counter() - t0
    return {"value": allc["value"], "unit": "frames/s", "cores": allc["procs"], "kind": "reference",
            "sample": f"{allc['slices']} slices x {fr} frames of the stock run_adaptive, one process per core "
                      f"({allc['cores']} host cores), single-threaded BLAS; {dt:.0f} s for all three numbers",
            "one_core_frames_per_s": one["value"], "track_step_ms_median": ts}


def run_reference_port(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    frames = args.ref_frames or 8
    ks, _ = make_data(dict(cfg, T=frames), [0])
    A0, B0 = init_factors(cfg, [0])
    for _ in range(args.warmup):
        cpu_oracle_fps(cfg, max(1, frames // 4), ks, A0, B0)
    times = []
    for _ in range(args.steps):
        fps, dt = cpu_oracle_fps(cfg, frames, ks, A0, B0)
        times.append(dt)
    total = sum(times)
    value = frames * args.steps / total
    cores = os.cpu_count()
    line = {"metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
            "config": {"workload": cfg["desc"], "frames_per_step": frames, "parallelism": "cpu"},
            "impl": "reference",
            "cpu_baseline": {"value": value, "unit": "frames/s", "cores": cores, "kind": "port",
                             "sample": f"first {frames} frames of the {args.config} sequence per step, oracle port "
                                       "of the reference algorithm (numpy/OpenBLAS, all host threads)"},
            "e2e": {"value": value, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ our arm
def run_entries(args, cfg):
    """Entry-sampling online loop (EntryEngine): per frame entry scores, a
    large-domain Philox draw, the gather at the drawn entries and the generic index-list step, the
    frame chain replayed as one CUDA graph. Replicas per rank (no collective), like config 2."""
    import torch
    import torch.distributed as dist

    import paper_1609_04104_b200 as tt

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    n, R, T = cfg["n"], cfg["R"], cfg["T"]
    k = int(np.ceil(cfg["entries"] * n * n))
    ks_np, _ = make_data(cfg, [0])
    A0, B0 = init_factors(cfg, [0])
    pol = tt.InformativeEntries(k=k, forced=(0,), beta=cfg["beta"], key0=2024)
    kd = torch.from_numpy(ks_np[:, 0]).to(dev)

    def engine():
        e = tt.EntryEngine(n, n, R, cfg["lam"], tt.Fixed(cfg["mu"]), pol)
        e.set_image_factors(A0[0], B0[0])
        return e

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    graphs = []
    for _ in range(args.warmup + args.steps):  # one engine per step: every step replays the same sequence
        e = engine()
        e.run(kd, T)  # eager first frame + capture + one replay (warm)
        graphs.append(e)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    stream = torch.cuda.current_stream()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(args.warmup):
            for g, _, _ in graphs[i]._graph[0]:
                g.replay()
        for i in range(args.steps):
            flush.zero_()
            a, b = ev[i]
            a.record(stream)
            for g, _, _ in graphs[args.warmup + i]._graph[0]:
                g.replay()
            b.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    frames = T - 1  # the replayed chain (the first frame runs eagerly when the graph is captured)
    total_ms = sum(a.elapsed_time(b) for a, b in ev)
    tot = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    total_ms = float(tot[0])
    value = frames * world * args.steps / (total_ms / 1e3)
    # algorithmic bytes per frame: y and (i, j) at the sampled entries, factors read + written, gamma,
    # the fp64 entry distribution (SURVEY §8d's row model with entries in place of rows)
    L_frame = float(k)  # upper bound on |Omega| (distinct entries <= trials)
    b_frame = 8 * L_frame + 8 * L_frame + 16 * R * (2 * n) + 8 * R + 8 * n * n
    hbm_peak, sm_max, peak_kind = measured_peaks()
    achieved = b_frame * frames * args.steps / (total_ms / 1e3) / 1e9
    e2e = None
    if not args.no_e2e:
        ks_pin = torch.from_numpy(ks_np[:, 0]).pin_memory()
        res = None
        for _ in range(2):  # warm-up in the timed loop's pattern (pinned result blocks cached)
            res = tt.run_online(ks_pin, A0, B0, cfg["lam"], tt.Fixed(cfg["mu"]), pol)
        torch.cuda.synchronize()
        t_e2e = []
        for _ in range(max(1, args.steps)):
            t0 = time.perf_counter()
            res = tt.run_online(ks_pin, A0, B0, cfg["lam"], tt.Fixed(cfg["mu"]), pol)
            torch.cuda.synchronize()
            t_e2e.append(time.perf_counter() - t0)
        et = torch.tensor([sum(t_e2e)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
        e2e = {"value": T * world * len(t_e2e) / float(et[0]), "unit": "frames/s",
               "h2d_bytes_per_step": int(ks_np[:, 0].nbytes),
               "d2h_bytes_per_step": int(res.recon.nbytes + res.gamma.nbytes + res.cost.nbytes + res.mu.nbytes),
               "call": "paper_1609_04104_b200.run_online(pinned host kspace, InformativeEntries) -> host recon"}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        from oracle import tt_oracle as O
        fr = 3
        t0 = time.perf_counter()
        O.online_run_entries(ks_np[:fr, 0], O.fft_cols(A0[0]), O.fft_cols(B0[0]), cfg["lam"], ("fixed", cfg["mu"]),
                             {"kind": "informative", "k": k, "forced": [0], "beta": cfg["beta"], "key": (2024, 0)})
        dt = time.perf_counter() - t0
        cpu = {"value": fr / dt, "unit": "frames/s", "cores": os.cpu_count(), "kind": "port",
               "sample": f"first {fr} frames ({dt:.1f} s), oracle port of the reference entries loop"}
    if world > 1:
        dist.destroy_process_group()
    if rank != 0:
        return 0
    line = {
        "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "c64", "data": "synthetic",
        "config": {"workload": cfg["desc"], "frames_per_step": frames, "rank": R, "nx": n, "ny": n, "trials": k,
                   "l2": "flushed between steps (256 MB write)", "parallelism": f"replicas x{world}"},
        # per replayed frame: entry scores (3 kernels), large-domain draw (6), generic step (5)
        "gpu_launches": 14 * frames * args.steps,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": achieved / hbm_peak, "traffic": None, "kernel": "entry frame chain (graph)",
                     "bytes_per_frame": b_frame, "peak_kind": peak_kind},
        "clocks": clk.summary(), "e2e": e2e, "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)
    return 0


def run_patched(args, cfg):
    """Per-patch trackers (run_tracking_patched). A step is one whole patched run on
    resident, binned inputs: the warm-up passes (one launch each, rebalanced between), the streamed
    pass over the remaining frames, and the re-projection of every frame into the assembled
    reconstructions. Replicas per rank (a frame's latency is one patch step, so splitting patches
    across GPUs would not shorten it)."""
    import torch
    import torch.distributed as dist

    import paper_1609_04104_b200 as tt
    from paper_1609_04104_b200 import patches as PT

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    n, R, T, pch = cfg["n"], cfg["R"], cfg["T"], cfg["patch"]
    warm_n, warm_ep = cfg["warm_n"], cfg["warm_epochs"]
    grid = tt.PatchGrid((n, n), pch, pch, R)
    ks_np, clean_np = make_data(cfg, [0])
    masks = patched_masks(cfg, T)
    A0s, B0s = patched_init(cfg)
    ent, off = PT._entry_table(masks, (n, n), T)
    cnt = np.diff(off)
    fd = torch.from_numpy(ks_np[:, 0]).to(dev)
    run = PT._PatchRun(grid, cfg["lam"], tt.Fixed(cfg["mu"]), fd, ent, off)
    run.set_factors(A0s, B0s)
    a0, b0 = run.a.clone(), run.b.clone()
    npch = run.np
    main = list(range(warm_n, T))
    g = torch.empty((len(main), npch, R), dtype=torch.complex64, device=dev)
    c = torch.empty((len(main), npch), dtype=torch.float64, device=dev)
    m = torch.empty((len(main), npch), dtype=torch.float64, device=dev)
    gp = torch.empty((T, npch, R), dtype=torch.complex64, device=dev)
    rec = torch.empty((T, n, n), dtype=torch.complex64, device=dev)
    warm_s = torch.arange(warm_n, dtype=torch.int32, device=dev)
    main_s = torch.tensor(main, dtype=torch.int32, device=dev)
    all_s = torch.arange(T, dtype=torch.int32, device=dev)
    from paper_1609_04104_b200 import _lib as L

    def launch(sd, nsteps, project=False, gamma=None, cost=None, mu=None, recon=None):
        args_ = L.PatchesArgs(
            nx=n, ny=n, pn1=pch, pn2=pch, rank=R, patch0=0, npatch_local=npch, frames=T, pidx=run.pidx.data_ptr(),
            py=run.py.data_ptr(), pcnt=run.pcnt.data_ptr(), nsteps=nsteps, sched=sd.data_ptr(), a=run.a.data_ptr(),
            b=run.b.data_ptr(), t=run.t.data_ptr(), alpha_bar=run.ab.data_ptr(), lam=run.lam, step_mode=run.mode,
            mu=run.mu, c_floor=run.c_floor, c_cap=run.c_cap, project=int(project), gamma_out=L.ptr(gamma),
            cost_out=L.ptr(cost), mu_out=L.ptr(mu), resid_out=None, recon_out=L.ptr(recon),
            status=run.status.data_ptr())
        L.check(L.lib().tt_track_patches(L.stream_ptr(), args_), "patch tracking")

    stream = torch.cuda.current_stream()
    ev_main = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    launches = [0]

    def one_run(timed_main=None):
        run.a.copy_(a0)
        run.b.copy_(b0)
        run.t.fill_(1)
        run.ab.zero_()
        launches[0] = 0
        for e in range(warm_ep):
            if e > 0:
                run.rebalance()
                launches[0] += 1
            launch(warm_s, warm_n)
            launches[0] += 1
        if timed_main:
            timed_main[0].record(stream)
        launch(main_s, len(main), gamma=g, cost=c, mu=m)
        if timed_main:
            timed_main[1].record(stream)
        launch(all_s, T, project=True, gamma=gp, recon=rec)
        launches[0] += 2

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    for _ in range(args.warmup):
        one_run()
    torch.cuda.synchronize()
    L.raise_status(int(run.status.max().item()) | int(run.bin_status.item()), "patched bench")
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    mains = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.zero_()
            ev[i][0].record(stream)
            one_run(mains[i])
            ev[i][1].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    total_ms = sum(a.elapsed_time(b) for a, b in ev)
    main_ms = sum(a.elapsed_time(b) for a, b in mains)
    tot = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    total_ms = float(tot[0])
    value = T * world * args.steps / (total_ms / 1e3)
    # the trackers work in the data domain (k-space): NRMSE against the clean frames' k-space
    ck = np.fft.fft2(clean_np[:, 0], norm="ortho")
    rh = rec.cpu().numpy()
    nm = np.sum(np.abs(rh - ck) ** 2, axis=(1, 2)) / np.sum(np.abs(ck) ** 2, axis=(1, 2))
    # dominant kernel = the streamed pass: per frame, every sampled entry's (index, value) read once,
    # each patch's factors read + written, the per-step outputs (SURVEY §8d's model per patch)
    L_main = float(cnt[warm_n:].mean()) if len(main) else 0.0
    b_frame = 12 * L_main + npch * (16 * R * 2 * pch + 8 * R + 16)
    hbm_peak, sm_max, peak_kind = measured_peaks()
    achieved = b_frame * len(main) * args.steps / (main_ms / 1e3) / 1e9
    e2e = None
    if not args.no_e2e:
        ks_pin = torch.from_numpy(ks_np[:, 0]).pin_memory()
        res = None
        for _ in range(2):
            res = tt.run_tracking_patched(ks_pin, grid, cfg["lam"], tt.Fixed(cfg["mu"]), masks, warm_n=warm_n,
                                          warm_epochs=warm_ep, A0s=A0s, B0s=B0s)
        torch.cuda.synchronize()
        t_e2e = []
        for _ in range(max(1, args.steps)):
            t0 = time.perf_counter()
            res = tt.run_tracking_patched(ks_pin, grid, cfg["lam"], tt.Fixed(cfg["mu"]), masks, warm_n=warm_n,
                                          warm_epochs=warm_ep, A0s=A0s, B0s=B0s)
            torch.cuda.synchronize()
            t_e2e.append(time.perf_counter() - t0)
        et = torch.tensor([sum(t_e2e)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
        e2e = {"value": T * world * len(t_e2e) / float(et[0]), "unit": "frames/s",
               "h2d_bytes_per_step": int(ks_np[:, 0].nbytes + ent.nbytes + off.nbytes),
               "d2h_bytes_per_step": int(res.recon.nbytes + res.gamma.nbytes + res.step_gamma.nbytes),
               "call": "paper_1609_04104_b200.run_tracking_patched(pinned host frames, host masks) -> host recon"}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        fr = min(T, 100)
        fps, dt = cpu_oracle_fps(cfg, fr, ks_np, None, None)
        cpu = {"value": fps, "unit": "frames/s", "cores": os.cpu_count(), "kind": "port",
               "sample": f"{fr} streamed frames x {npch} patch steps + re-projection ({dt:.1f} s), oracle port "
                         "of _run_tracking_patched (no warm-up)"}
    if world > 1:
        dist.destroy_process_group()
    if rank != 0:
        return 0
    line = {
        "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "c64", "data": "synthetic",
        "config": {"workload": cfg["desc"], "frames_per_step": T, "patches": npch, "patch": [pch, pch], "rank": R,
                   "warm_steps": warm_n * warm_ep, "streamed_frames": len(main),
                   "streamed_ms_per_frame": main_ms / args.steps / max(1, len(main)),
                   "l2": "flushed between steps (256 MB write)", "parallelism": f"replicas x{world}",
                   "nrmse_last": float(np.sqrt(nm[-1]))},
        "gpu_launches": launches[0],
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": achieved / hbm_peak, "traffic": None, "kernel": "patch_track_kernel (streamed pass)",
                     "bytes_per_frame": b_frame, "peak_kind": peak_kind},
        "clocks": clk.summary(), "e2e": e2e, "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)
    return 0


def run_batch_mode(args, cfg):
    """Multi-epoch batch mode (run_batch): a step is the whole batch run, epochs x T
    tracked steps (rebalanced between epochs, reshuffled order from the caller's generator) and the
    re-projection of every frame; value = tracked frame-steps per second with the k-space resident.
    Replicas per rank."""
    import torch
    import torch.distributed as dist

    import paper_1609_04104_b200 as tt

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    n, R, T, E = cfg["n"], cfg["R"], cfg["T"], cfg["epochs"]
    ks_np, clean_np = make_data(cfg, [0])
    A0, B0 = init_factors(cfg, [0])
    S = int(np.ceil(cfg["vd"] * n))
    gen = np.random.Generator(np.random.Philox(key=2024))
    tab = np.stack([tt.variable_density_rows(n, -1.0, cfg["vd"], gen) for _ in range(T)])
    cnt = np.full(T, S)
    kd = torch.from_numpy(ks_np[:, 0]).to(dev)

    def one(src):
        return tt.run_batch(src, A0[0], B0[0], cfg["lam"], tt.Fixed(cfg["mu"]), tab, cnt, epochs=E,
                            rng=np.random.default_rng(5), reshuffle=True)

    for _ in range(args.warmup):
        one(kd)
    torch.cuda.synchronize()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.zero_()
            ev[i][0].record(stream)
            res = one(kd)  # ends with the host readback of the results
            ev[i][1].record(stream)
        torch.cuda.synchronize()
    total_ms = sum(a.elapsed_time(b) for a, b in ev)
    tot = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    total_ms = float(tot[0])
    value = E * T * world * args.steps / (total_ms / 1e3)
    nm = [float(np.linalg.norm(res.recon[t] - clean_np[t, 0]) ** 2 / np.linalg.norm(clean_np[t, 0]) ** 2)
          for t in range(T)]
    e2e = None
    if not args.no_e2e:
        kp = torch.from_numpy(ks_np[:, 0]).pin_memory()
        one(kp)
        torch.cuda.synchronize()
        t_e2e = []
        for _ in range(max(1, args.steps)):
            t0 = time.perf_counter()
            res = one(kp)
            torch.cuda.synchronize()
            t_e2e.append(time.perf_counter() - t0)
        et = torch.tensor([sum(t_e2e)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
        e2e = {"value": E * T * world * len(t_e2e) / float(et[0]), "unit": "frame-steps/s",
               "h2d_bytes_per_step": int(ks_np[:, 0].nbytes),
               "d2h_bytes_per_step": int(res.recon.nbytes + res.gamma.nbytes + res.step_gamma.nbytes),
               "call": "paper_1609_04104_b200.run_batch(pinned host kspace, row tables) -> host recon"}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        from oracle import tt_oracle as O
        fr = 20
        rows = [tab[f] for f in range(fr)]
        t0 = time.perf_counter()
        O.batch_run(ks_np[:fr, 0], A0[0], B0[0], cfg["lam"], ("fixed", cfg["mu"]), rows, 2,
                    rng=np.random.default_rng(5), reshuffle=True)
        dt = time.perf_counter() - t0
        cpu = {"value": 2 * fr / dt, "unit": "frame-steps/s", "cores": os.cpu_count(), "kind": "port",
               "sample": f"2 epochs over the first {fr} frames + re-projection ({dt:.1f} s), oracle port of "
                         "tracker.run / the batch re-projection"}
    if world > 1:
        dist.destroy_process_group()
    if rank != 0:
        return 0
    line = {
        "metric": METRIC, "value": value, "unit": "frame-steps/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "c64", "data": "synthetic",
        "config": {"workload": cfg["desc"], "frames": T, "epochs": E, "rank": R, "rows_per_frame": S,
                   "l2": "flushed between steps (256 MB write)", "parallelism": f"replicas x{world}",
                   "nrmse_last": float(np.sqrt(nm[-1]))},
        "gpu_launches": None,
        "roofline": None,
        "clocks": clk.summary(), "e2e": e2e, "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)
    return 0


def run_row_sharded(args, cfg):
    """Config 4 across ranks: Ah row-sharded, one NCCL all-reduce of the frame's fp64 payload per frame,
    the T-frame chain captured in one CUDA graph. `scaling: strong` (the single 1024^2 slice is
    split)."""
    import torch
    import torch.distributed as dist

    import paper_1609_04104_b200 as tt
    from paper_1609_04104_b200 import _lib as L
    from paper_1609_04104_b200 import _ops as K
    from paper_1609_04104_b200.engine import RowShardedEngine

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    L.load()
    n, R, T = cfg["n"], cfg["R"], cfg["T"]
    ks_np, clean_np = make_data(cfg, [0])
    A0, B0 = init_factors(cfg, [0])
    Smax = int(np.ceil(cfg["vd"] * n))
    gen = np.random.Generator(np.random.Philox(key=2024))
    tab = np.stack([tt.variable_density_rows(n, -1.0, cfg["vd"], gen) for _ in range(T)])
    ks = torch.from_numpy(ks_np[:, 0]).to(dev)

    def allreduce(t):
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.SUM)

    def fresh():
        e = RowShardedEngine(n, n, R, cfg["lam"], tt.Fixed(cfg["mu"]), tab, np.full(T, Smax), world, rank,
                             cluster=args.cluster, allreduce=allreduce)
        e.set_image_factors(A0[0], B0[0])
        return e

    e = fresh()
    r0, r1 = e.r0, e.r1
    out = e.make_outputs(T)
    Xblk = torch.empty(T, r1 - r0, n, dtype=torch.complex64, device=dev)
    lib = L.lib()
    stream = torch.cuda.current_stream()
    # the T-frame chain [phase 1 -> NCCL all-reduce -> phase 2] captured once as one CUDA graph; every step
    # restores the initial state into the same buffers (outside the timed region) and replays it
    init_state = e.save()
    e.capture(ks, T, out)

    def fresh():
        e.restore(init_state)
        return e

    def step():
        e.replay()
        # this rank's block of k-space rows of every frame, Ah_rows diag(gamma) Bh^T (row i of the k-space frame
        # needs only row i of Ah: the reconstruction shards by rows with no collective and no FFT)
        L.check(lib.tt_reconstruct(stream.cuda_stream, T, r1 - r0, n, R, out["ah"].data_ptr(), out["bh"].data_ptr(),
                                   out["gamma"].data_ptr(), Xblk.data_ptr()), "reconstruct")

    for _ in range(args.warmup):
        e = fresh()
        step()
    torch.cuda.synchronize()
    times = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            e = fresh()
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step()
            e1.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
    tot = torch.tensor([sum(times)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
        dist.destroy_process_group()
    L.raise_status(int(e.status.item()), "row-sharded engine")
    total_ms = float(tot[0])
    if rank != 0:
        return 0
    value = T * args.steps / (total_ms / 1e3)
    line = {"metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "c64", "data": "synthetic",
            "config": {"workload": cfg["desc"].replace("single GPU, unsharded", f"Ah row-sharded over {world}"),
                       "frames_per_step": T, "rank": R, "nx": n, "ny": n, "parallelism": f"row-shard x{world}",
                       "collectives": "2 NCCL all-reduces per frame (W fp32, GA/norms fp64) + 1 all-gather per step"},
            "gpu_launches": (2 * T + 3) * args.steps, "clocks": clk.summary(), "e2e": None, "cpu_baseline": None}
    print(json.dumps(line), flush=True)
    return 0


def run_local_sharded(args, cfg):
    """Config 4 on one GPU with the row sharding's ranks as thread-block clusters (SURVEY §8e emulated
    in one fused cooperative launch: `LocalShardedEngine(fused=True)`), then the inverse column FFTs and
    the reconstruction of all T frames. Device-timed like `run_ours` (L2 flushed between steps)."""
    import torch

    import paper_1609_04104_b200 as tt
    from paper_1609_04104_b200 import _lib as L
    from paper_1609_04104_b200 import _ops as K

    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    L.load()
    n, R, T = cfg["n"], cfg["R"], cfg["T"]
    ks_np, clean_np = make_data(cfg, [0])
    A0, B0 = init_factors(cfg, [0])
    Smax = int(np.ceil(cfg["vd"] * n))
    gen = np.random.Generator(np.random.Philox(key=2024))
    tab = np.stack([tt.variable_density_rows(n, -1.0, cfg["vd"], gen) for _ in range(T)])
    ks = torch.from_numpy(ks_np[:, 0]).to(dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    X = torch.empty(T, n, n, dtype=torch.complex64, device=dev)
    stream = torch.cuda.current_stream()

    def fresh():
        e = tt.LocalShardedEngine(n, n, R, cfg["lam"], tt.Fixed(cfg["mu"]), tab, np.full(T, Smax), args.local_ranks)
        e.set_image_factors(A0[0], B0[0])
        return e, e.make_outputs(T)

    def step(e, out, ev=None):
        e.run(ks, T, out=out)
        if ev is not None:
            ev.record(stream)
        A = K.fft_cols_(out["ah"], inverse=True)
        B = K.fft_cols_(out["bh"], inverse=True)
        K.reconstruct(A, B, out["gamma"], out=X)

    for _ in range(args.warmup):
        e, out = fresh()
        step(e, out)
    torch.cuda.synchronize()
    tot = trk = 0.0
    with ClockSampler(0) as clk:
        for _ in range(args.steps):
            e, out = fresh()
            flush.zero_()
            torch.cuda.synchronize()
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            e0.record(stream)
            step(e, out, e1)
            e2.record(stream)
            torch.cuda.synchronize()
            tot += e0.elapsed_time(e2)
            trk += e0.elapsed_time(e1)
    e.check_status()
    cl = torch.from_numpy(clean_np[:, 0]).to(dev)
    nm = tt.nmse_frames(cl.reshape(T, -1), X.reshape(T, -1)).sqrt()
    value = T * args.steps / (tot / 1e3)
    line = {"metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": tot / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "c64", "data": "synthetic",
            "config": {"workload": cfg["desc"].replace("single GPU, unsharded",
                                                       f"Ah row-sharded over {args.local_ranks} clusters of one GPU"),
                       "frames_per_step": T, "rank": R, "nx": n, "ny": n, "l2": "flushed between steps (256 MB write)",
                       "parallelism": f"local row-shard x{args.local_ranks} (fused cooperative launch: "
                                      f"{'yes' if e.fused else 'no, 3-launch frames'})"},
            "gpu_launches": (1 if e.fused else 3 * T) + 3,
            "extra": {"us_per_frame_tracking": 1e3 * trk / args.steps / T, "mean_nrmse": float(nm.mean()),
                      "last_nrmse": float(nm[-1])},
            "clocks": clk.summary(), "e2e": None, "cpu_baseline": None}
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args, cfg):
    import torch
    import torch.distributed as dist

    import paper_1609_04104_b200 as tt
    from paper_1609_04104_b200 import _lib as L
    from paper_1609_04104_b200 import _ops as K

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    L.load()

    # slices of this rank: replicas for c2 (weak), shards for c3 (strong)
    from paper_1609_04104_b200.sharding import slice_partition

    if cfg["slices"] == 1:
        slice_ids = [rank]
        scaling = "weak"
    else:
        slice_ids = slice_partition(cfg["slices"], world, rank)
        scaling = "strong"
        if args.shard_of > 1:
            if world != 1:
                raise SystemExit("bench.py: --shard-of is a one-GPU measurement")
            slice_ids = slice_partition(cfg["slices"], args.shard_of, 0)
    ns = len(slice_ids)
    n, R, T = cfg["n"], cfg["R"], cfg["T"]
    ks_np, clean_np = make_data(cfg, slice_ids)
    A0, B0 = init_factors(cfg, slice_ids)

    if "vd" in cfg:
        # static variable-density masks per frame and slice (observation.py:300-323), drawn on device
        Smax = int(np.ceil(cfg["vd"] * n))
        tab = np.zeros((T, ns, Smax), np.int64)
        for si, s_id in enumerate(slice_ids):
            gen = np.random.Generator(np.random.Philox(key=2024 + (s_id << 64)))
            for f in range(T):
                tab[f, si] = tt.variable_density_rows(n, -1.0, cfg["vd"], gen)
        pol = tt.StaticRows(tab, np.full((T, ns), Smax))
    else:
        pol = tt.Informative(k=cfg["K"], forced=cfg["forced"], beta=cfg["beta"], key0=2024, key1=slice_ids[0])
    step_rule = tt.HessianBound(1e-3, 1e9) if args.step == "hessian" else tt.Fixed(cfg["mu"])
    eng = tt.OnlineEngine(n, n, R, ns, cfg["lam"], step_rule, pol, cluster=args.cluster)
    eng.set_image_factors(A0, B0)
    ah0, bh0 = eng.ah.clone(), eng.bh.clone()
    ks = torch.from_numpy(ks_np).to(dev)
    out = eng.make_outputs(T, history=True)
    X = torch.empty(T, ns, n, n, dtype=torch.complex64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()
    if args.track_priority:
        # tracking on a high-priority stream: at a block boundary the next tracking launch's clusters go
        # ahead of the reconstruction CTAs still pending (those take what is left of their block later)
        hp = torch.cuda.Stream(dev, priority=-1)
        hp.wait_stream(stream)
        torch.cuda.set_stream(hp)
        stream = hp
    s_rec = torch.cuda.Stream(dev)
    # one step = the T-frame sequence in `nblk` tracking launches on the compute stream (the resident
    # state carries across launches; results are launch-boundary invariant); each block's inverse column
    # FFTs + reconstruction run on a second stream as soon as its tracking is done, on the SMs the
    # tracking clusters leave free (run_online's pipeline without the host transfers)
    nblk = max(1, min(args.blocks, T))
    # the last block's reconstruction runs after the tracking ends (the step's tail): it is made short
    # (--tail-frac of an even block), the others share the rest evenly
    if nblk > 1 and args.tail_frac < 1.0:
        last = max(1, int(round(args.tail_frac * T / nblk)))
        head = T - last
        bounds = [(head * i // (nblk - 1), head * (i + 1) // (nblk - 1)) for i in range(nblk - 1)] + [(head, T)]
    else:
        bounds = [(T * i // nblk, T * (i + 1) // nblk) for i in range(nblk)]
    parts = [{k: v[a:b] for k, v in out.items()} for a, b in bounds]
    tracked = [torch.cuda.Event() for _ in bounds]

    def reset():
        eng.ah.copy_(ah0)
        eng.bh.copy_(bh0)
        eng.philox_pos.zero_()
        eng.alpha_bar.zero_()
        eng.frame, eng.t = 0, 1

    def step_kernels(e_track=None):
        s_rec.wait_stream(stream)
        for (a, b), part, ev in zip(bounds, parts, tracked):
            eng.run(ks, b - a, out=part)                          # fused online loop over frames [a, b)
            ev.record(stream)
            s_rec.wait_event(ev)
            with torch.cuda.stream(s_rec):
                if args.recon_ctas:
                    if b < T:
                        os.environ["TT_RECON_MAXCTAS"] = str(args.recon_ctas)
                    else:
                        os.environ.pop("TT_RECON_MAXCTAS", None)
                eng.reconstruct(part, into=X[a:b], domain="kspace")  # k-space frames (run_adaptive's .kspace)
        if e_track is not None:
            e_track.record(stream)
        stream.wait_stream(s_rec)
    launches_per_step = 2 * nblk  # per block: the tracking launch and the reconstruction

    for _ in range(args.warmup):
        reset()
        step_kernels()
    torch.cuda.synchronize()
    eng.check_status()

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.zero_()          # L2 flush (256 MB write), outside the timed events
            reset()
            e0, e1, e2 = ev[i]
            e0.record(stream)
            step_kernels(e1)
            e2.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    step_ms = [a.elapsed_time(c) for a, b, c in ev]
    track_ms = [a.elapsed_time(b) for a, b, c in ev]
    total_ms = sum(step_ms)
    tot = torch.tensor([total_ms, sum(track_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    total_ms, track_total = float(tot[0]), float(tot[1])
    eng.check_status()
    frames_all = T * cfg["slices"] * (world if cfg["slices"] == 1 else 1) * args.steps
    if args.shard_of > 1:
        frames_all = T * ns * args.steps  # this GPU's shard only
    value = frames_all / (total_ms / 1e3)

    # ---- quality (outside timing): NRMSE of the last step's reconstructions
    Xr = X.reshape(T, ns, n, n)
    cl = torch.from_numpy(clean_np).to(dev).reshape(T * ns, n, n)
    cl = K.fft2_(cl.contiguous())  # F_x X F_y^T
    cl = cl.reshape(T, ns, n, n)
    nmse = ((cl - Xr).abs().pow(2).sum((-1, -2)) / cl.abs().pow(2).sum((-1, -2))).double()
    cnt = out["cnt"].double()

    # ---- roofline of the dominant kernel (tt_rows_kernel) from the BASELINE byte model
    S_avg = float(cnt.mean())
    b_upd = 8 * S_avg * n + 4 * S_avg + 16 * R * (2 * n) + 8 * R + (8 * n if "K" in cfg else 0)
    b_rec = 8 * n * n
    f_sep = 16 * S_avg * n * R + 16 * (S_avg + n) * R * R + 10 * R * 2 * n * math.log2(n) + 16 * R * 2 * n
    hbm_peak, sm_max, peak_kind = measured_peaks()
    track_s = track_total / 1e3 / args.steps
    achieved = b_upd * T * ns / track_s / 1e9
    fp32_peak = 148 * 128 * 2 * sm_max * 1e6 / 1e12
    traffic = None
    prof = os.path.join(HERE, "profiles", f"traffic_{args.config}.json")
    if os.path.exists(prof):
        with open(prof) as f:
            traffic = json.load(f).get("dram_bytes_per_launch")

    # ---- e2e through the public API with pinned host buffers
    e2e = None
    h2d = d2h = 0
    if not args.no_e2e:
        ks_pin = torch.from_numpy(ks_np).pin_memory()
        # two warm-up calls in the timed loop's pattern (the previous result stays alive while the next
        # call runs): both pinned result blocks are then in torch's host caching allocator
        res = None
        for _ in range(2):
            res = tt.run_online(ks_pin, A0, B0, cfg["lam"], step_rule, pol, cluster=args.cluster,
                                recon_domain="kspace")
        torch.cuda.synchronize()
        t_e2e = []
        for _ in range(max(1, args.steps)):
            t0 = time.perf_counter()
            res = tt.run_online(ks_pin, A0, B0, cfg["lam"], step_rule, pol, cluster=args.cluster,
                                recon_domain="kspace")
            torch.cuda.synchronize()
            t_e2e.append(time.perf_counter() - t0)
        # bytes that crossed the host link: the whole truth when it is uploaded, only the sampled rows when the
        # kernels read the page-locked truth in place (run_online's zero-copy mode for truths >= 512 MB)
        from paper_1609_04104_b200.engine import ZERO_COPY_BYTES

        zc = ks_np.nbytes >= ZERO_COPY_BYTES
        h2d = (res.rows.total() * n * 8) if zc else ks_np.nbytes
        d2h = res.recon.nbytes + res.gamma.nbytes + res.cost.nbytes + res.mu.nbytes + 4 * (T * ns * (eng.max_rows + 1))
        et = torch.tensor([sum(t_e2e)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
        # whole-job frames: replicas (one slice per rank) or all the job's slices sharded over the ranks
        job_slices = world if cfg["slices"] == 1 else (ns if args.shard_of > 1 else cfg["slices"])
        e2e = {"value": T * job_slices * len(t_e2e) / float(et[0]), "unit": "frames/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "call": "paper_1609_04104_b200.run_online(pinned host kspace, recon_domain='kspace') -> host "
                       "k-space frames (run_adaptive's recon for k-space data) + reports",
               "truth_transfer": "zero-copy (sampled rows read in place)" if zc else "upload"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            cpu = cpu_baseline_reference(args, cfg)
        except Exception as e:  # reference package missing: the pinned oracle port on slice 0
            fr = args.cpu_frames
            fps, dt = cpu_oracle_fps(cfg, fr, ks_np, A0, B0)
            cpu = {"value": fps, "unit": "frames/s", "cores": os.cpu_count(), "kind": "port",
                   "sample": f"first {fr} frames of slice 0 ({dt:.1f} s), oracle port of the reference algorithm "
                             f"(numpy SVD ridge, pocketfft), all host threads; reference unavailable: {e!r}"}

    api_fps = None
    if rank == 0 and not args.no_e2e:
        try:
            api_fps = api_loop_rate(cfg, ks_np[:, 0], A0[0], B0[0])
        except Exception as e:  # reported, never fatal to the bench line
            api_fps = f"failed: {e!r}"

    # ---- parity of this run (rank 0's first slice) against the oracle on the same masks: the device's
    # own rows fed to the oracle restatement, every frame's gamma and NRMSE compared (north_star tolerances)
    parity = None
    if rank == 0 and not args.no_parity:
        parity = run_parity(cfg, ks_np[:, 0], clean_np[:, 0], A0[0], B0[0], out, Xr[:, 0], cnt[:, 0],
                            clean_k=cl[:, 0].cpu().numpy(),
                            ostep=("hessian", 1e-3, 1e9) if args.step == "hessian" else ("fixed", cfg["mu"]))

    if world > 1:
        dist.destroy_process_group()
    if rank != 0:
        return 0
    line = {
        "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": scaling,
        "vs_baseline": None, "dtype": "c64", "data": "synthetic",
        "config": dict(workload_config(args, cfg), slices_per_gpu=ns, cluster_ctas_per_slice=eng.cluster,
                       step=("HessianBound(1e-3, 1e9)" if args.step == "hessian" else f"Fixed({cfg['mu']})"),
                       tracking_launches_per_step=nblk,
                       **({"shard_of": f"rank 0's shard of a {args.shard_of}-GPU run, alone on one GPU"}
                          if args.shard_of > 1 else {}),
                       parallelism=f"{'replicas' if cfg['slices'] == 1 else 'slice-shard'} x{world}"),
        "gpu_launches": launches_per_step * args.steps,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": achieved / hbm_peak, "traffic": traffic, "kernel": "tt_rows_kernel",
                     "bytes_per_slice_frame": b_upd, "frames_per_launch": T / nblk,
                     "algorithmic_bytes_per_launch": b_upd * ns * T / nblk, "peak_kind": peak_kind},
        "extra": {"track_ms_per_step": track_total / args.steps,
                  "us_per_frame_tracking": 1e6 * track_s / T,
                  "step_hbm_frac": (b_upd + b_rec) * value / 1e9 / hbm_peak / (1 if cfg["slices"] == 1 else 1),
                  "fp32_frac_tracking": f_sep * T * ns / track_s / 1e12 / fp32_peak,
                  "mean_nrmse": float(nmse.sqrt().mean()), "last_nrmse": float(nmse[-1].sqrt().mean()),
                  "rows_per_frame_avg": S_avg,
                  "per_call_api_frames_per_s": api_fps,
                  "per_call_api": "row_scores -> draw_samples -> track_step(FourierMask rows, host y) -> "
                                  "reconstruct_frame (host k-space + image), one slice, synchronous"},
        "clocks": clk.summary(),
        "e2e": e2e,
        "cpu_baseline": cpu,
        "parity": parity,
    }
    print(json.dumps(line), flush=True)
    return 0


def api_loop_rate(cfg, ks_host, A0, B0, frames=24):
    """The per-call drop-in loop a reference caller gets after switching imports (experiment.py:498-525 on
    the per-call API): row_scores -> draw_samples (Philox generator) -> FourierMask batch from host k-space
    rows -> track_step -> reconstruct_frame (host k-space and magnitude image back), image-domain factors,
    one frame at a time. Frames/s over `frames` frames after two warm-up frames (wall clock, synchronous
    API: every call returns host data)."""
    import torch

    import paper_1609_04104_b200 as tt

    n, R = cfg["n"], cfg["R"]
    k = int(cfg["K"]) if "K" in cfg else int(np.ceil(cfg["vd"] * n))
    forced = list(cfg.get("forced", (0,)))
    state = tt.TrackerState(tt.TensorSubspace((np.asarray(A0, np.complex128), np.asarray(B0, np.complex128))),
                            tt.StepConfig(cfg["lam"], R, tt.Fixed(cfg["mu"])))
    gen = np.random.Generator(np.random.Philox(key=11))
    t_start = None
    for f in range(frames + 2):
        if f == 2:
            torch.cuda.synchronize()
            t_start = time.perf_counter()
        dist = tt.row_scores(state.subspace, cfg.get("beta", 0.1))
        plan = tt.draw_samples(dist, k, True, gen, forced=forced)
        rows = plan.omega
        y = ks_host[f % ks_host.shape[0]][rows, :].ravel()
        batch = tt.MeasurementBatch(y, tt.FourierMask((n, n), tt.rows_to_entries(rows, n)), t=f)
        state, rep = tt.track_step(state, batch)
        tt.reconstruct_frame(state.subspace, rep.gamma)
    torch.cuda.synchronize()
    return frames / (time.perf_counter() - t_start)


PARITY_FRAMES = {"c4": 12}  # the oracle's numpy SVD at 1024^2 takes ~1 s per frame


def run_parity(cfg, ks, clean, A0, B0, out, X, cnt, clean_k=None, ostep=None):
    """Slice 0 of the last timed step against the CPU oracle (oracle/tt_oracle.py, pinned to the
    reference) fed the same per-frame rows the device drew: per-frame gamma (relative) and the NRMSE
    trajectory (absolute) over the first T frames (PARITY_FRAMES bounds c4); the device's masks are
    also compared with the oracle's own free-running draws (first frame that differs, if any)."""
    from oracle import tt_oracle as O

    T = min(cfg["T"], PARITY_FRAMES.get(cfg.get("name", ""), cfg["T"]))
    if cfg["n"] >= 1024:
        T = min(T, PARITY_FRAMES["c4"])
    rows_d = out["rows"][:T, 0].cpu().numpy()
    rows = [rows_d[f, :int(cnt[f])].astype(np.int64) for f in range(T)]
    A0c = np.asarray(A0).astype(np.complex64).astype(np.complex128)
    B0c = np.asarray(B0).astype(np.complex64).astype(np.complex128)
    t0 = time.perf_counter()
    ostep = ostep or ("fixed", cfg["mu"])
    ref = O.online_run(ks[:T], A0c, B0c, cfg["lam"], ostep, {"kind": "static", "rows": rows},
                       clean=clean[:T])
    gam = out["gamma"][:T, 0].cpu().numpy()
    ge = max(float(np.linalg.norm(gam[f] - ref["gamma"][f]) / max(np.linalg.norm(ref["gamma"][f]), 1e-300))
             for f in range(T))
    nd = X[:T].cpu().numpy().reshape(T, -1)
    cl = (clean if clean_k is None else clean_k)[:T].reshape(T, -1)  # the device frames' domain
    nr_dev = np.sqrt(np.sum(np.abs(cl - nd) ** 2, axis=1) / np.sum(np.abs(cl) ** 2, axis=1))
    ne = float(np.max(np.abs(nr_dev - np.sqrt(np.asarray(ref["nmse"])))))
    first_div = None
    if "K" in cfg:  # the oracle's own draws from its own probabilities (device masks bit-exact until a near-tie)
        free = O.online_run(ks[:T], A0c, B0c, cfg["lam"], ostep,
                            {"kind": "informative", "k": cfg["K"], "forced": list(cfg["forced"]), "beta": cfg["beta"],
                             "key": (2024, 0)})
        for f in range(T):
            if not np.array_equal(free["rows"][f], rows[f]):
                first_div = f
                break
    return {"slice": 0, "frames": T, "gamma_max_rel": ge, "nrmse_max_abs": ne,
            "tol": {"gamma_rel": 1e-4, "nrmse_abs": 1e-3}, "pass": bool(ge < 1e-4 and ne < 1e-3),
            "masks": "device rows fed to the oracle",
            "free_running_masks_equal_frames": (T if first_div is None else first_div) if "K" in cfg else None,
            "oracle_s": round(time.perf_counter() - t0, 1)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c3")
    ap.add_argument("--cluster", type=int, default=0)
    ap.add_argument("--step", choices=["fixed", "hessian"], default="fixed",
                    help="step rule of the default arms: Fixed(mu) or the Lipschitz HessianBound(1e-3, 1e9) (config.py)")
    ap.add_argument("--cpu-frames", type=int, default=100)
    ap.add_argument("--ref-frames", type=int, default=0,
                    help="frames per reference step (default: the config's T; 8 for c4, SURVEY §8d)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--row-shard", action="store_true", help="config c4: use the row-sharded two-phase path")
    ap.add_argument("--blocks", type=int, default=4, help="tracking launches per step (reconstruction overlaps)")
    ap.add_argument("--track-priority", type=int, default=0,
                    help="1: the tracking launches run on a high-priority stream (measured: no effect)")
    ap.add_argument("--recon-ctas", type=int, default=0,
                    help="experiment: persistent reconstruction CTAs of every block but the last (0: one per SM)")
    ap.add_argument("--tail-frac", type=float, default=1.0,
                    help="size of the last tracking block relative to an even split (its reconstruction is the tail)")
    ap.add_argument("--shard-of", type=int, default=0,
                    help="config c3 on one GPU: run only rank 0's slice shard of an N-GPU run (the per-rank "
                         "workload of --gpus N measured alone; value counts this GPU's frames only)")
    ap.add_argument("--local-ranks", type=int, default=0,
                    help="config c4 on one GPU: row-shard over this many thread-block clusters (fused launch)")
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config], name=args.config)
    if args.impl == "reference":
        return run_reference(args, cfg)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # one process per GPU: re-launch under torch.distributed.run (rendezvous on 127.0.0.1)
        import socket

        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
        return subprocess.call(cmd)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.config == "c4" and (int(os.environ.get("WORLD_SIZE", "1")) > 1 or args.row_shard):
        return run_row_sharded(args, cfg)
    if args.config == "c4" and args.local_ranks > 0:
        return run_local_sharded(args, cfg)
    if "entries" in cfg:
        return run_entries(args, cfg)
    if "patch" in cfg:
        return run_patched(args, cfg)
    if cfg.get("batch"):
        return run_batch_mode(args, cfg)
    return run_ours(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
