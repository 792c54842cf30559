"""Reconstruction quality, mirroring the reference's ``metrics.nmse``
(`pkg/src/tensortrack/metrics.py:53-62`).

``nmse`` runs on the device (``tt_nmse``: fp64 sums of complex64 frames in a
fixed order) and, like the reference, raises ``ValueError`` for a shape
mismatch or an all-zero truth. ``nmse_frames`` is the batched form the online
engines use for their per-frame NRMSE trajectories. SSIM and the
differential-CS baseline are evaluation code outside the hot path.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib as L

__all__ = ["nmse", "nmse_frames"]


def _dev_c64(x, dev) -> torch.Tensor:
    t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(np.asarray(x)))
    if not t.is_complex():
        t = t.to(torch.float64)
    return t.to(dev, torch.complex64).contiguous()


def nmse_frames(truth, estimate) -> torch.Tensor:
    """Per-frame NMSE of (F, ...) stacks (the leading axis indexes frames) -> (F,) float64 on the device.
    A frame with an all-zero truth gives NaN."""
    dev = L.device()
    t, e = _dev_c64(truth, dev), _dev_c64(estimate, dev)
    if t.shape != e.shape:
        raise ValueError(f"shape mismatch {tuple(t.shape)} vs {tuple(e.shape)}")
    F = t.shape[0] if t.dim() > 0 else 1
    n = t.numel() // max(F, 1)
    out = torch.empty(F, dtype=torch.float64, device=dev)
    if F == 0:
        return out
    lib = L.lib()
    done = 0
    while done < F:
        nf = min(65535, F - done)
        work = torch.empty(int(lib.tt_nmse_work_doubles(nf)), dtype=torch.float64, device=dev)
        L.check(lib.tt_nmse(L.stream_ptr(), nf, n, t.view(F, n)[done].data_ptr(), e.view(F, n)[done].data_ptr(),
                            work.data_ptr(), out[done].data_ptr()), "nmse")
        done += nf
    return out


def nmse(truth, estimate) -> float:
    """Squared Frobenius error normalised by the truth's squared norm (metrics.py:53-62)."""
    ts = tuple(truth.shape) if isinstance(truth, torch.Tensor) else np.shape(truth)
    es = tuple(estimate.shape) if isinstance(estimate, torch.Tensor) else np.shape(estimate)
    if tuple(ts) != tuple(es):
        raise ValueError(f"shape mismatch {tuple(ts)} vs {tuple(es)}")
    t = truth.reshape(1, -1) if isinstance(truth, torch.Tensor) else np.asarray(truth).reshape(1, -1)
    e = estimate.reshape(1, -1) if isinstance(estimate, torch.Tensor) else np.asarray(estimate).reshape(1, -1)
    v = float(nmse_frames(t, e)[0].item())
    if v != v:  # NaN: all-zero truth
        raise ValueError("NMSE is undefined for an all-zero reference")
    return v
