"""Seeded synthetic cine phantoms for the BASELINE.json configurations.

Host-side data generation only (it stands in for the scanner). Nothing here
is on the timed path. The reference ships a two-ellipse phantom
(`pkg/src/tensortrack/synth.py:50-71`); BASELINE.json asks for a different
construction, so this is written new:

* 6 static background ellipses, magnitude U[0.2, 1], random centre, axes and
  rotation, layered with soft edges;
* a smooth random phase (a random quadratic polynomial over the frame);
* a "heart" ellipse whose radius follows r0 * (1 + a * sin(2 pi t / P));
* additive complex Gaussian noise, sigma per real/imaginary component (the
  reference convention, `observation.py:343-352`).

The truth k-space is the unitary (ortho), unshifted 2-D DFT of the noisy
frame, row 0 = DC (`observation.py:9-11`, `:171-178`).

Layout: frames first, ``(T, Nx, Ny)`` C-contiguous, so one frame is one
contiguous block in HBM.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = ["CinePhantom", "cine_phantom", "truth_kspace"]


@dataclass(frozen=True)
class CinePhantom:
    clean: np.ndarray      # (T, Nx, Ny) complex64, noiseless image frames
    image: np.ndarray      # (T, Nx, Ny) complex64, noisy image frames
    kspace: np.ndarray     # (T, Nx, Ny) complex64, fft2(image, ortho)


def _soft(level: np.ndarray, soft: float) -> np.ndarray:
    return 0.5 * (1.0 - np.tanh((level - 1.0) / soft))


def _ellipse_level(u, v, cu, cv, au, av, theta):
    c, s = np.cos(theta), np.sin(theta)
    du, dv = u - cu, v - cv
    p = (c * du + s * dv) / au
    q = (-s * du + c * dv) / av
    return np.sqrt(p * p + q * q)


def cine_phantom(
    n1: int,
    n2: int,
    frames: int,
    period: float = 16.0,
    seed: int = 0,
    slice_index: int = 0,
    noise_sigma: float = 0.01,
    n_background: int = 6,
    pulse_amplitude: float = 0.25,
) -> CinePhantom:
    """Deterministic phantom for ``(seed, slice_index)``; different slices get
    different ellipse layouts (BASELINE config 3)."""
    if n1 < 4 or n2 < 4 or frames < 1:
        raise ValueError("phantom needs at least a 4x4 frame and one frame")
    rng = np.random.default_rng([int(seed), int(slice_index), 0x7A11])
    yy, xx = np.meshgrid(np.arange(n1), np.arange(n2), indexing="ij")
    u = (yy - (n1 - 1) / 2.0) / (n1 / 2.0)
    v = (xx - (n2 - 1) / 2.0) / (n2 / 2.0)
    soft = 1.5 / min(n1 / 2.0, n2 / 2.0)

    background = np.zeros((n1, n2))
    for _ in range(n_background):
        cu, cv = rng.uniform(-0.45, 0.45, size=2)
        au, av = rng.uniform(0.12, 0.45, size=2)
        theta = rng.uniform(0.0, np.pi)
        mag = rng.uniform(0.2, 1.0)
        ind = _soft(_ellipse_level(u, v, cu, cv, au, av, theta), soft)
        background = background * (1.0 - ind) + mag * ind

    coef = rng.uniform(-1.0, 1.0, size=6) * (np.pi / 2.0)
    phase = (coef[0] + coef[1] * u + coef[2] * v + coef[3] * u * u
             + coef[4] * u * v + coef[5] * v * v)
    carrier = np.exp(1j * phase)

    hu, hv = rng.uniform(-0.15, 0.15, size=2)
    r0 = rng.uniform(0.12, 0.2)
    heart_mag = 1.0
    t = np.arange(frames, dtype=np.float64)
    cycle = np.mod(t, period) / period
    radius = r0 * (1.0 + pulse_amplitude * np.sin(2.0 * np.pi * cycle))
    rho = np.sqrt((u - hu) ** 2 + (v - hv) ** 2)

    clean = np.empty((frames, n1, n2), dtype=np.complex64)
    image = np.empty((frames, n1, n2), dtype=np.complex64)
    kspace = np.empty((frames, n1, n2), dtype=np.complex64)
    for k in range(frames):
        ind = _soft(rho / radius[k], soft)
        mag = background * (1.0 - ind) + heart_mag * ind
        x = mag * carrier
        clean[k] = x
        if noise_sigma > 0:
            x = x + noise_sigma * (rng.standard_normal((n1, n2)) + 1j * rng.standard_normal((n1, n2)))
        image[k] = x
        kspace[k] = np.fft.fft2(x, norm="ortho")
    return CinePhantom(clean=clean, image=image, kspace=kspace)


def truth_kspace(n1, n2, frames, period=16.0, seed=0, slice_index=0, noise_sigma=0.01):
    return cine_phantom(n1, n2, frames, period, seed, slice_index, noise_sigma).kspace
