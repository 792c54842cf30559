"""MRI specialisations on the hot path — drop-in for the ``reconstruct_frame``,
``interp_track_step`` and patch-grid parts of ``tensortrack.mri``
(`pkg/src/tensortrack/mri.py:40-177`). The per-patch trackers themselves run in
``patches.py`` (one CTA per patch). Coils and the coil residual image are out of
scope.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _ops as K
from .core import TensorSubspace, synthesize_device
from .observation import EntryMask, MeasurementBatch
from .tracker import TrackerState, track_step

__all__ = ["FrameEstimate", "reconstruct_frame", "interp_track_step", "PatchGrid", "patch_partition",
           "patch_assemble"]


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
    img = K.fft2(ks, inverse=True)
    return FrameEstimate(kspace=ks.cpu().numpy().astype(np.complex128),
                         image=img.abs().cpu().numpy().astype(np.float64))


def interp_track_step(state: TrackerState, batch: MeasurementBatch):
    """k-space interpolation step: track_step over an entry mask (mri.py:124-135)."""
    if not isinstance(batch.descriptor, EntryMask):
        raise TypeError("interpolation steps take entry-mask batches")
    if state.subspace.nmodes != 2:
        raise ValueError("interpolation tracking needs a two-mode subspace")
    return track_step(state, batch)


@dataclass(frozen=True)
class PatchGrid:
    """Non-overlapping tiling of an N1 x N2 frame into n1 x n2 patches with per-patch rank ``rho``
    (mri.py:48-80): the extents must divide the frame exactly."""

    frame_shape: tuple
    n1: int
    n2: int
    rho: int = 1

    def __post_init__(self):
        shape = tuple(int(n) for n in self.frame_shape)
        if len(shape) != 2:
            raise ValueError("patch grids tile 2-D frames")
        if self.n1 < 1 or self.n2 < 1 or self.rho < 1:
            raise ValueError("patch extents and rank must be positive")
        if shape[0] % self.n1 or shape[1] % self.n2:
            raise ValueError(f"patch size ({self.n1}, {self.n2}) does not tile frame {shape}")
        object.__setattr__(self, "frame_shape", shape)

    @property
    def k1(self) -> int:
        return self.frame_shape[0] // self.n1

    @property
    def k2(self) -> int:
        return self.frame_shape[1] // self.n2


def patch_partition(frame, grid: PatchGrid) -> list:
    """Row-major list of the grid's patches (mri.py:151-162). Works on host arrays and on device
    tensors (copies of the tiles either way)."""
    shape = tuple(frame.shape)
    if shape != grid.frame_shape:
        raise ValueError(f"frame shape {shape} does not match grid {grid.frame_shape}")
    out = []
    for p in range(grid.k1):
        for q in range(grid.k2):
            tile = frame[p * grid.n1:(p + 1) * grid.n1, q * grid.n2:(q + 1) * grid.n2]
            out.append(tile.clone() if hasattr(tile, "clone") else np.array(tile, copy=True))
    return out


def patch_assemble(patches, grid: PatchGrid):
    """Exact inverse of patch_partition (mri.py:165-177)."""
    patches = list(patches)
    if len(patches) != grid.k1 * grid.k2:
        raise ValueError(f"expected {grid.k1 * grid.k2} patches, got {len(patches)}")
    if patches and hasattr(patches[0], "device"):
        import torch

        out = torch.empty(grid.frame_shape, dtype=patches[0].dtype, device=patches[0].device)
    else:
        patches = [np.asarray(p) for p in patches]
        out = np.empty(grid.frame_shape, dtype=np.result_type(*[p.dtype for p in patches]))
    for p in range(grid.k1):
        for q in range(grid.k2):
            tile = patches[p * grid.k2 + q]
            if tuple(tile.shape) != (grid.n1, grid.n2):
                raise ValueError("patch shape does not match the grid")
            out[p * grid.n1:(p + 1) * grid.n1, q * grid.n2:(q + 1) * grid.n2] = tile
    return out
