"""Checkpoint / resume of the online loop's state (A, B, t, alpha_bar) over CTEN.

The reference has no checkpoint: its state is the frozen ``TrackerState`` (subspace factors, t,
alpha_bar; tracker.py:99-106) and runs return ``final_subspace`` without persisting it
(experiment.py:122). Here a checkpoint is a directory holding

* ``A.cten``, ``B.cten`` — the factors in the reference's CTEN container (cten.py:1-74): the device
  engine's resident k-space factors [nslices][N][R] stored as float32 pairs (dtype 0, the exact bits of
  the complex64 state), or a host ``TrackerState``'s factors as float64 pairs (dtype 1);
* ``state.json`` — t, alpha_bar per slice (exact: the float's hex form), the Philox stream position of
  each slice's informative draws, the frame index, the factor domain ("kspace" for the engine's
  Ah = F_x A, "image" for a TrackerState) and the shape.

Resuming an ``OnlineEngine`` from its checkpoint continues the sequence bit for bit: the same resident
factors, step accumulator, time index and draw positions (tests/test_gpu_checkpoint.py). Host file I/O
only (the native CTEN reader/writer); the engine's tensors are read back once per save.
"""

from __future__ import annotations

import json
import os

import numpy as np
import torch

from . import cten

__all__ = ["save_engine", "load_engine", "save_state", "load_state"]

_VERSION = 1


def _write_json(path, obj) -> None:
    tmp = path + ".tmp"
    with open(tmp, "w", encoding="utf-8") as fh:
        json.dump(obj, fh, indent=2, sort_keys=True)
        fh.write("\n")
    os.replace(tmp, path)


def _read_json(path) -> dict:
    with open(path, encoding="utf-8") as fh:
        meta = json.load(fh)
    if meta.get("version") != _VERSION:
        raise ValueError(f"unsupported checkpoint version {meta.get('version')!r}")
    return meta


def save_engine(engine, path) -> None:
    """Write an ``OnlineEngine``'s resident state (k-space factors of every slice, t, alpha_bar, Philox
    positions, frame index) to the directory ``path``."""
    os.makedirs(path, exist_ok=True)
    torch.cuda.current_stream(engine.dev).synchronize()
    ah = engine.ah.detach().cpu().numpy()
    bh = engine.bh.detach().cpu().numpy()
    cten.write_cten(os.path.join(path, "A.cten"), ah, dtype_code=0)  # complex64 bits, exact
    cten.write_cten(os.path.join(path, "B.cten"), bh, dtype_code=0)
    meta = {
        "version": _VERSION,
        "kind": "engine",
        "domain": "kspace",
        "nslices": engine.nslices, "nx": engine.nx, "ny": engine.ny, "rank": engine.rank,
        "t": int(engine.t),
        "frame": int(engine.frame),
        "alpha_bar": [float(v).hex() for v in engine.alpha_bar.cpu().numpy()],
        "philox_pos": [int(v) for v in engine.philox_pos.cpu().numpy()],
    }
    _write_json(os.path.join(path, "state.json"), meta)


def load_engine(engine, path) -> None:
    """Restore a checkpoint written by :func:`save_engine` into an ``OnlineEngine`` of the same shape
    (the policy, step and lambda are the engine's own, as a resumed run's configuration is)."""
    meta = _read_json(os.path.join(path, "state.json"))
    if meta.get("kind") != "engine":
        raise ValueError("not an engine checkpoint")
    shape = (meta["nslices"], meta["nx"], meta["ny"], meta["rank"])
    if shape != (engine.nslices, engine.nx, engine.ny, engine.rank):
        raise ValueError(f"checkpoint shape {shape} does not match the engine "
                         f"{(engine.nslices, engine.nx, engine.ny, engine.rank)}")
    dev = engine.dev
    ah = cten.read_cten_tensor(os.path.join(path, "A.cten"), pin=False)
    bh = cten.read_cten_tensor(os.path.join(path, "B.cten"), pin=False)
    if tuple(ah.shape) != (engine.nslices, engine.nx, engine.rank) or \
            tuple(bh.shape) != (engine.nslices, engine.ny, engine.rank):
        raise ValueError("checkpoint factor shapes do not match the engine")
    engine.ah = ah.to(dev).contiguous()
    engine.bh = bh.to(dev).contiguous()
    engine.alpha_bar = torch.tensor([float.fromhex(v) for v in meta["alpha_bar"]], dtype=torch.float64, device=dev)
    engine.philox_pos = torch.tensor(meta["philox_pos"], dtype=torch.int64, device=dev)
    engine.status = torch.zeros(engine.nslices, dtype=torch.int32, device=dev)
    engine.t = int(meta["t"])
    engine.frame = int(meta["frame"])


def save_state(state, path) -> None:
    """Write a host-API ``TrackerState`` (tracker.py:99-106: factors, t, alpha_bar) to ``path``; the
    factors as float64 pairs (the reference's complex128 state)."""
    os.makedirs(path, exist_ok=True)
    A, B = state.subspace.factors
    cten.write_cten(os.path.join(path, "A.cten"), np.asarray(A), dtype_code=1)
    cten.write_cten(os.path.join(path, "B.cten"), np.asarray(B), dtype_code=1)
    cfg = state.config
    step = cfg.step
    meta = {
        "version": _VERSION,
        "kind": "state",
        "domain": "image",
        "t": int(state.t),
        "alpha_bar": float(state.alpha_bar).hex(),
        "config": {"lam": float(cfg.lam), "rank": int(cfg.rank), "init_scale": float(cfg.init_scale),
                   "norm_cap": None if cfg.norm_cap is None else float(cfg.norm_cap),
                   "step": ({"fixed": float(step.mu)} if hasattr(step, "mu")
                            else {"hessian": [float(step.c_floor), float(step.c_cap)]})},
    }
    _write_json(os.path.join(path, "state.json"), meta)


def load_state(path):
    """The ``TrackerState`` saved by :func:`save_state`."""
    from .core import TensorSubspace
    from .tracker import Fixed, HessianBound, StepConfig, TrackerState

    meta = _read_json(os.path.join(path, "state.json"))
    if meta.get("kind") != "state":
        raise ValueError("not a TrackerState checkpoint")
    A = cten.read_cten(os.path.join(path, "A.cten"))
    B = cten.read_cten(os.path.join(path, "B.cten"))
    c = meta["config"]
    st = c["step"]
    step = Fixed(st["fixed"]) if "fixed" in st else HessianBound(*st["hessian"])
    cfg = StepConfig(c["lam"], c["rank"], step, init_scale=c["init_scale"], norm_cap=c["norm_cap"])
    return TrackerState(TensorSubspace((A, B)), cfg, t=int(meta["t"]), alpha_bar=float.fromhex(meta["alpha_bar"]))
