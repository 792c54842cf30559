"""Acquisition (the S0 step): experiment.StreamingProvider
(experiment.py:70-111) and observation.project / measure
(observation.py:186-204, :335-353) over a device-resident truth tensor.

The truth (frames on the last axis, as the reference stores it) is uploaded
once in the engines' layout (frames leading, one frame contiguous). Frame
requests keep the reference's tripwire: asking for a frame beyond the first
unserved one raises RuntimeError (out of range: IndexError), which keeps
streaming runs honest. Entry reads are device gathers; a FourierMask sketch
transforms the frame with the device column FFT (two passes). Noise is drawn
from the caller's ``rng`` exactly as the reference does (host
``standard_normal``), so the generator stream stays in step; the device
engines themselves consume pre-noised truth, in frame order by construction.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib as L
from . import _ops as K
from .observation import EntryMask, FourierMask, MeasurementBatch

__all__ = ["StreamingProvider", "project", "measure"]


class StreamingProvider:
    """Serves ground-truth frames strictly in order (experiment.py:70-111), from the GPU."""

    def __init__(self, tensor):
        t = tensor if isinstance(tensor, torch.Tensor) else torch.from_numpy(np.asarray(tensor))
        if t.dim() < 2:
            raise ValueError("truth tensor needs at least one frame axis")
        self._frame_shape = tuple(t.shape[:-1])
        self._frames = int(t.shape[-1])
        self._truth = t.movedim(-1, 0).to(L.device(), torch.complex64).contiguous()  # (T, ...)
        self._next = 0

    @property
    def frames(self) -> int:
        return self._frames

    @property
    def frame_shape(self) -> tuple[int, ...]:
        return self._frame_shape

    @property
    def truth_device(self) -> torch.Tensor:
        """(T, *frame_shape) complex64 on the device: the engines' resident truth."""
        return self._truth

    def _claim(self, t: int) -> None:
        if t < 0 or t >= self._frames:
            raise IndexError(f"frame {t} out of range")
        if t > self._next:
            raise RuntimeError(f"frame {t} requested before frame {self._next} was processed")
        if t == self._next:
            self._next += 1

    def full_frame_device(self, t: int) -> torch.Tensor:
        self._claim(t)
        return self._truth[t]

    def full_frame(self, t: int) -> np.ndarray:
        return self.full_frame_device(t).cpu().numpy().astype(np.complex128)

    def entries_device(self, t: int, indices) -> torch.Tensor:
        self._claim(t)
        return _gather(self._truth[t], indices)

    def entries(self, t: int, indices) -> np.ndarray:
        return self.entries_device(t, indices).cpu().numpy().astype(np.complex128)

    def sketch(self, t: int, descriptor, noise_sigma: float, rng) -> MeasurementBatch:
        self._claim(t)
        return measure(self._truth[t], descriptor, noise_sigma, rng, t=t)


def _gather(frame: torch.Tensor, indices) -> torch.Tensor:
    """frame (n1, n2) complex64 on the device, indices (L, 2) -> (L,) complex64 by tt_gather_entries."""
    n1, n2 = frame.shape
    idx = np.asarray(indices, dtype=np.int64).reshape(-1, 2)
    if idx.size and (idx.min() < 0 or idx[:, 0].max() >= n1 or idx[:, 1].max() >= n2):
        raise IndexError("entry index out of range")
    flat = torch.from_numpy((idx[:, 0] * n2 + idx[:, 1]).astype(np.int32)).to(frame.device)
    cnt = torch.tensor([flat.numel()], dtype=torch.int32, device=frame.device)
    y = torch.empty(max(1, flat.numel()), dtype=torch.complex64, device=frame.device)
    ij = torch.empty(max(1, flat.numel()), 2, dtype=torch.int32, device=frame.device)
    if flat.numel():
        L.check(L.lib().tt_gather_entries(L.stream_ptr(), n1, n2, frame.contiguous().data_ptr(), flat.data_ptr(),
                                          cnt.data_ptr(), flat.numel(), ij.data_ptr(), y.data_ptr()), "gather")
    return y[:flat.numel()]


def project(frame, descriptor) -> np.ndarray:
    """observation.project (observation.py:186-204) for EntryMask / FourierMask on the device."""
    x = frame if isinstance(frame, torch.Tensor) else torch.from_numpy(np.asarray(frame, dtype=np.complex64))
    x = x.to(L.device(), torch.complex64)
    if tuple(x.shape) != tuple(descriptor.shape):
        raise ValueError(f"frame shape {tuple(x.shape)} does not match descriptor {descriptor.shape}")
    if isinstance(descriptor, EntryMask):
        y = _gather(x, descriptor.indices)
    elif isinstance(descriptor, FourierMask):
        k = K.fft2(x.contiguous())                                       # F1 X F2^T
        y = _gather(k, descriptor.indices)
    else:
        raise TypeError(f"unknown descriptor type {type(descriptor).__name__}")
    return y.cpu().numpy().astype(np.complex128)


def measure(frame, descriptor, noise_sigma: float, rng, t: int = 0) -> MeasurementBatch:
    """observation.measure (observation.py:335-353): project, then circular complex Gaussian noise
    from ``rng`` (real and imaginary parts i.i.d. with standard deviation ``noise_sigma``)."""
    if noise_sigma < 0:
        raise ValueError("noise_sigma must be nonnegative")
    y = project(frame, descriptor)
    if noise_sigma > 0 and y.size:
        noise = rng.standard_normal(y.size) + 1j * rng.standard_normal(y.size)
        y = y + noise_sigma * noise
    return MeasurementBatch(y, descriptor, t=t, noise_sigma=noise_sigma)
