"""The reference arm of bench.py: the UNMODIFIED reference package timed on the host cores.

Bench infrastructure, never the product. The reference (`tensortrack`, pure Python/NumPy) is
installed once into ``baseline/_ref`` (``pip install --no-index --no-build-isolation --no-deps
--target baseline/_ref``). Its ``__init__`` imports scikit-image through
``metrics.py``, which this image lacks, so the package module is pre-registered (``__init__`` never
runs) and ``skimage.metrics.structural_similarity`` is stubbed: SSIM is an evaluation metric
outside the reconstruction path and is "stubbed" exactly as SURVEY §8d prescribes. Everything
else runs the reference's own code:

* ``run_adaptive`` (experiment.py:444-556) per slice: the whole per-frame body — row_scores,
  draw_samples, EntryMask + MeasurementBatch validation, acquisition from the StreamingProvider,
  track_step, reconstruct_frame, per-frame NMSE (+ the stubbed SSIM) — for the config's full T,
  cold-started (warm_start_frames=0, so every frame is informative from frame 0, the bench's
  workload) with the config's rank, lambda, Fixed mu, fraction and beta;
* ``track_step`` alone (tracker.py:367-411) on FourierMask batches with image-domain factors, the
  north-star call, median per frame.

Slices are independent, so the CPU's best throughput is one process per core, each with a
single BLAS thread (multi-threaded OpenBLAS is several times slower on these small SVDs:
SURVEY §8d). ``WorkerPool`` keeps one process per slice, each holding its slice's truth, and times
a step as the wall time from "go" to the last "done".
"""

from __future__ import annotations

import importlib
import multiprocessing as mp
import os
import sys
import time
import types

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIRS = (os.path.join(HERE, "baseline", "_ref", "tensortrack"), "/root/reference/pkg/src/tensortrack")


def reference_dir():
    for d in REF_DIRS:
        if os.path.exists(os.path.join(d, "tracker.py")):
            return d
    return None


def load_reference():
    """The stock reference modules (experiment, config, tracker, observation, core, mri)."""
    d = reference_dir()
    if d is None:
        raise ImportError("reference package not installed (baseline/_ref)")
    if "tensortrack" not in sys.modules:
        pkg = types.ModuleType("tensortrack")
        pkg.__path__ = [d]
        sys.modules["tensortrack"] = pkg
    if "skimage.metrics" not in sys.modules:
        sk = types.ModuleType("skimage")
        skm = types.ModuleType("skimage.metrics")
        skm.structural_similarity = lambda *a, **k: 0.0  # SSIM stubbed (evaluation only)
        sk.metrics = skm
        sys.modules["skimage"] = sk
        sys.modules["skimage.metrics"] = skm
    mods = {m: importlib.import_module(f"tensortrack.{m}")
            for m in ("experiment", "config", "tracker", "observation", "core", "mri")}
    return types.SimpleNamespace(**mods), d


def adaptive_config(ref, cfg):
    """ExperimentConfig of the bench config for the stock run_adaptive."""
    C = ref.config
    n = cfg["n"]
    if "K" in cfg:
        samp = C.SamplingConfig(mode="adaptive", fraction=cfg["K"] / n, k=int(cfg["K"]), beta=cfg["beta"],
                                replacement=True, domain="rows")
    else:  # variable-density configs: the VD branch of run_adaptive (switch frame after the run)
        samp = C.SamplingConfig(mode="variable_density", fraction=cfg["vd"], switch_frame=cfg["T"] + 1,
                                domain="rows")
    return C.ExperimentConfig(seed=7, rank=cfg["R"], lam=cfg["lam"], mu=cfg["mu"], warm_start_frames=0,
                              sampling=samp)


def _truth(cfg, s, frames):
    import numpy as np

    sys.path.insert(0, HERE)
    from paper_1609_04104_b200.phantom import cine_phantom

    ph = cine_phantom(cfg["n"], cfg["n"], frames, period=cfg["period"], seed=2024, slice_index=s)
    return np.ascontiguousarray(np.moveaxis(ph.kspace, 0, -1).astype(np.complex128))  # frames last


_THREAD_VARS = ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS")


def _worker(conn, cfg, slices, frames):
    try:
        ref, _ = load_reference()
        truths = [_truth(cfg, s, frames) for s in slices]
        ecfg = adaptive_config(ref, cfg)
        conn.send(("ready", None))
        while True:
            msg = conn.recv()
            if msg == "stop":
                break
            nf = int(msg)
            t0 = time.perf_counter()
            nm = [float(ref.experiment.run_adaptive(tr[..., :nf], ecfg).metrics[-1].nmse) for tr in truths]
            dt = time.perf_counter() - t0
            conn.send(("done", (dt, nm[0])))
    except Exception as e:  # report, never hang the parent
        conn.send(("error", repr(e)))


class WorkerPool:
    """``procs`` processes (single BLAS thread each) sharing the slices round-robin, each slice's truth
    resident in its worker; a step runs every slice once."""

    def __init__(self, cfg, slices, frames, procs):
        ctx = mp.get_context("spawn")
        self.conns, self.procs = [], []
        # one BLAS thread per worker: set before the children start (a spawned child imports numpy, and
        # so initialises OpenBLAS, while unpickling its target, before _worker runs)
        saved = {k: os.environ.get(k) for k in _THREAD_VARS}
        os.environ.update({k: "1" for k in _THREAD_VARS})
        try:
            for w in range(procs):
                a, b = ctx.Pipe()
                p = ctx.Process(target=_worker, args=(b, cfg, list(slices[w::procs]), frames), daemon=True)
                p.start()
                self.conns.append(a)
                self.procs.append(p)
        finally:
            for k, v in saved.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
        for c in self.conns:
            kind, val = c.recv()
            if kind != "ready":
                raise RuntimeError(f"reference worker failed: {val}")

    def step(self, frames):
        t0 = time.perf_counter()
        for c in self.conns:
            c.send(frames)
        out = []
        for c in self.conns:
            kind, val = c.recv()
            if kind != "done":
                raise RuntimeError(f"reference worker failed: {val}")
            out.append(val)
        return time.perf_counter() - t0, out

    def close(self):
        for c in self.conns:
            try:
                c.send("stop")
            except (BrokenPipeError, OSError):
                pass
        for p in self.procs:
            p.join(timeout=10)
            if p.is_alive():
                p.kill()


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def track_step_ms(cfg, frames=12):
    """Median ms of the stock track_step on FourierMask batches (image-domain factors, Fixed mu),
    one BLAS thread, informative-like row counts (the config's K rows or VD fraction)."""
    import numpy as np
    from threadpoolctl import threadpool_limits

    ref, _ = load_reference()
    Tr, Ob, Co = ref.tracker, ref.observation, ref.core
    n, R = cfg["n"], cfg["R"]
    k = int(cfg["K"]) if "K" in cfg else int(np.ceil(cfg["vd"] * n))
    truth = _truth(cfg, 0, frames)
    rng = np.random.default_rng(7)
    gen = np.random.Generator(np.random.Philox(key=2024))
    state = Tr.init_state(Tr.StepConfig(cfg["lam"], R, Tr.Fixed(cfg["mu"])), (n, n), rng)
    times = []
    with threadpool_limits(limits=1):
        for f in range(frames):
            rows = np.sort(gen.choice(n, size=k, replace=False))
            ent = Ob.rows_to_entries(rows, n)
            y = truth[..., f][rows, :].ravel()
            t0 = time.perf_counter()
            batch = Ob.MeasurementBatch(y, Ob.FourierMask((n, n), ent), t=f)
            state, _ = Tr.track_step(state, batch)
            times.append(time.perf_counter() - t0)
    return 1e3 * float(np.median(times[2:] if len(times) > 4 else times))


def measure(cfg, steps, warmup, max_slices=None):
    """Slice-frames/s of the stock run_adaptive over the config's slices (all of them, or the first
    ``max_slices``) for the config's T per step, one process per host core (at most one per slice).
    Returns a dict for the bench line."""
    cores = host_cores()
    nsl = cfg.get("slices", 1)
    take = max(1, min(nsl, nsl if max_slices is None else max_slices))
    procs = max(1, min(take, cores))
    T = cfg["T"]
    pool = WorkerPool(cfg, list(range(take)), T, procs)
    try:
        for _ in range(warmup):
            pool.step(min(T, 4))
        dts, nm = [], []
        for _ in range(steps):
            dt, out = pool.step(T)
            dts.append(dt)
            nm = [v[1] for v in out]
    finally:
        pool.close()
    total = sum(dts)
    return dict(value=take * T * steps / total, ms_per_step=1e3 * total / steps, slices=take, procs=procs,
                cores=cores, frames=T, last_nmse=nm)
