"""Run artefacts in the reference's formats (experiment.py:641-675): metrics,
mask, trace and budget CSVs, byte-for-byte (same headers, `%.17g` floats,
LF line ends), plus the rows of an online run built from its device results.

The writers mirror ``experiment.write_metrics_csv`` / ``write_mask_csv`` /
``write_trace_csv`` / ``write_budget_csv``; ``online_mask_rows`` and
``online_budget_rows`` derive run_adaptive's mask and budget rows
(experiment.py:495-510) from an :class:`engine.OnlineResult`, the budget's
expected sample count (sampler.py:173-178) from the device row scores of each
frame's pre-update factors.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _ops as K

__all__ = ["MetricRow", "write_metrics_csv", "write_mask_csv", "write_trace_csv", "write_budget_csv",
           "online_mask_rows", "online_budget_rows", "write_manifest"]


@dataclass
class MetricRow:
    """experiment.MetricRow: per-frame quality row."""
    t: int
    nmse: float
    ssim: float
    samples: int


def _fmt(x: float) -> str:
    return f"{x:.17g}"


def write_metrics_csv(path, rows) -> None:
    with open(path, "w", encoding="utf-8", newline="\n") as fh:
        fh.write("t,nmse,ssim,samples\n")
        for row in rows:
            fh.write(f"{row.t},{_fmt(row.nmse)},{_fmt(row.ssim)},{row.samples}\n")


def write_mask_csv(path, rows) -> None:
    width = max((len(r) for r in rows), default=2)
    header = "t,i" if width == 2 else "t,i,j"
    with open(path, "w", encoding="utf-8", newline="\n") as fh:
        fh.write(header + "\n")
        for row in rows:
            fh.write(",".join(str(int(v)) for v in row) + "\n")


def write_trace_csv(path, reports) -> None:
    with open(path, "w", encoding="utf-8", newline="\n") as fh:
        fh.write("t,f_t,step_size,gamma_norm,residual_norm\n")
        for rep in reports:
            fh.write(f"{rep.t},{_fmt(rep.instantaneous_cost)},{_fmt(rep.step_size)},"
                     f"{_fmt(float(np.linalg.norm(rep.gamma)))},"
                     f"{_fmt(float(np.linalg.norm(rep.residual)))}\n")


def write_budget_csv(path, rows) -> None:
    with open(path, "w", encoding="utf-8", newline="\n") as fh:
        fh.write("t,K,omega_size,expected\n")
        for t, k, size, expected in rows:
            fh.write(f"{t},{k},{size},{_fmt(expected)}\n")


def online_mask_rows(result, t0: int = 0, slice_index: int = 0) -> list[tuple]:
    """(t, i) per sampled row, frames numbered from ``t0``, each frame's rows ascending as the reference
    records both its variable-density and its informative masks (experiment.py:495, :507)."""
    return [(t0 + f, int(i)) for f, rows in enumerate(result.rows) for i in np.sort(rows[slice_index])]


def online_budget_rows(result, A0, B0, k_draws: int, beta: float = 0.1, t0: int = 0,
                       slice_index: int = 0, replacement: bool = True, vd_frames: int = 0) -> list[tuple]:
    """(t, K, |Omega_t|, E|Omega_t|) per frame (experiment.py:496, :508-509): for the first ``vd_frames``
    (an AdaptiveSchedule's variable-density frames) (t, |rows|, |rows|, |rows|); for informative frames
    with replacement the expected distinct count sum_i 1 - (1 - p_i)^K under frame t's row scores,
    computed on the device from the pre-update factors (A0 for the first frame, then the previous
    frame's factors from the run's history); without replacement the plan size."""
    if not replacement or len(result.rows) <= vd_frames:
        out = []
        for f in range(len(result.rows)):
            m = len(result.rows[f][slice_index])
            out.append((t0 + f, m, m, float(m)) if f < vd_frames else (t0 + f, int(k_draws), m, float(m)))
        return out
    hist = getattr(result, "factor_history", None)
    if hist is None:
        raise ValueError("the result carries no factor history (run_online(..., keep_history=True))")
    ah_hist = hist  # (T, nx, R) k-space factors after each frame
    a_prev = torch.from_numpy(np.ascontiguousarray(np.fft.fft(np.asarray(A0), axis=0, norm="ortho"),
                                                   dtype=np.complex64))
    dev = ah_hist.device
    pre = torch.cat([a_prev.to(dev)[None], ah_hist[:-1]], dim=0)  # (T, nx, R)
    ny = int(np.asarray(B0).shape[0])
    p = K.row_scores(pre.contiguous(), ny, beta)  # (T, nx) fp64
    expected = (1.0 - (1.0 - p) ** int(k_draws)).sum(dim=1).cpu().numpy()
    out = []
    for f in range(len(result.rows)):
        m = len(result.rows[f][slice_index])
        out.append((t0 + f, m, m, float(m)) if f < vd_frames else (t0 + f, int(k_draws), m, float(expected[f])))
    return out


def write_manifest(path, mode: str, input_path, config: dict, per_frame_ms, nmse_values, total_s: float,
                   commit: str | None = None) -> dict:
    """manifest.json as run_experiment writes it (experiment.py:727-741): mode, input path, the config
    echo, the git commit, timings (total seconds, per-frame milliseconds rounded to 3 places) and the
    mean NMSE; indent 2, sorted keys, trailing newline. Returns the dict."""
    import json
    import subprocess

    if commit is None:
        try:
            out = subprocess.run(["git", "rev-parse", "HEAD"], capture_output=True, text=True, timeout=5, check=False)
            commit = out.stdout.strip() if out.returncode == 0 else "unknown"
        except OSError:
            commit = "unknown"
    manifest = {
        "mode": mode,
        "input": str(input_path),
        "config": config,
        "commit": commit,
        "timings": {"total_s": float(total_s), "per_frame_ms": [round(float(x), 3) for x in per_frame_ms]},
        "mean_nmse": float(np.mean(np.asarray(nmse_values, dtype=float))),
    }
    with open(path, "w", encoding="utf-8") as fh:
        json.dump(manifest, fh, indent=2, sort_keys=True)
        fh.write("\n")
    return manifest
