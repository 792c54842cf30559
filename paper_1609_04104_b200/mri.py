"""MRI specialisations on the hot path — drop-in for the ``reconstruct_frame``
and ``interp_track_step`` parts of ``tensortrack.mri``
(`pkg/src/tensortrack/mri.py:40-45, 107-135`). Patches, coils and the coil
residual image are out of scope.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _ops as K
from .core import TensorSubspace, synthesize_device
from .observation import EntryMask, MeasurementBatch
from .tracker import TrackerState, track_step

__all__ = ["FrameEstimate", "reconstruct_frame", "interp_track_step"]


@dataclass(frozen=True)
class FrameEstimate:
    """Interpolated k-space frame and the magnitude image it implies (mri.py:40-45)."""

    kspace: np.ndarray
    image: np.ndarray


def reconstruct_frame(subspace, gamma) -> FrameEstimate:
    """A1 diag(gamma) A2^T (plain transpose) and |F^-1(.)| (mri.py:107-121):
    the outer-product kernel, then two column-FFT passes for the image."""
    if not isinstance(subspace, TensorSubspace):
        subspace = TensorSubspace(subspace.factors)
    if subspace.nmodes != 2:
        raise ValueError("frame reconstruction needs a two-mode (matrix) subspace")
    g = np.asarray(gamma).ravel() if not hasattr(gamma, "device") else gamma
    if (g.size if isinstance(g, np.ndarray) else g.numel()) != subspace.rank:
        raise ValueError("gamma length does not match subspace rank")
    ks = synthesize_device(subspace, gamma)
    img = K.fft_cols(ks, inverse=True)
    img = K.fft_cols(img.transpose(0, 1).contiguous(), inverse=True).transpose(0, 1)
    return FrameEstimate(kspace=ks.cpu().numpy().astype(np.complex128),
                         image=img.abs().cpu().numpy().astype(np.float64))


def interp_track_step(state: TrackerState, batch: MeasurementBatch):
    """k-space interpolation step: track_step over an entry mask (mri.py:124-135)."""
    if not isinstance(batch.descriptor, EntryMask):
        raise TypeError("interpolation steps take entry-mask batches")
    if state.subspace.nmodes != 2:
        raise ValueError("interpolation tracking needs a two-mode subspace")
    return track_step(state, batch)
