"""Measurement descriptors and operators — drop-in for
``tensortrack.observation`` (`pkg/src/tensortrack/observation.py`) on the
hot path: ``EntryMask``/``FourierMask`` (:58-90), ``MeasurementBatch``
(:153-168), ``unitary_dft2`` (:171-178), ``unitary_dft_matrix`` (:181-183),
``build_phi`` (:207-244, Entry/Fourier branches), ``row_distances``
(:274-276), ``weighted_draw_without_replacement`` (:279-297),
``variable_density_rows`` (:300-323) and ``rows_to_entries`` (:326-332).

Descriptors are host index bookkeeping with the reference's validation
(range, no duplicates). A Fourier/entry mask whose indices are whole
phase-encode lines in row-major order is recognised once (``row_lines``) and
routed to the fused row-mask kernel; anything else takes the generic index
kernels. Coil / dense descriptors are out of scope and raise
TypeError in ``track_step``.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib as L
from . import _ops as K
from .core import TensorSubspace

__all__ = [
    "EntryMask",
    "FourierMask",
    "MeasurementBatch",
    "unitary_dft2",
    "unitary_dft_matrix",
    "build_phi",
    "row_distances",
    "weighted_draw_without_replacement",
    "variable_density_rows",
    "rows_to_entries",
    "philox_position",
]


def _as_indices(indices, shape) -> np.ndarray:
    """Validation of observation.py:41-55 (range, duplicates). The duplicate
    test runs on linear indices (O(L + N)) instead of a row-wise unique."""
    idx = np.ascontiguousarray(np.atleast_2d(np.asarray(indices, dtype=np.int64)))
    if idx.size == 0:
        idx = idx.reshape(0, len(shape))
    if idx.shape[1] != len(shape):
        raise ValueError(f"indices have {idx.shape[1]} coordinates for a {len(shape)}-way frame")
    for axis, extent in enumerate(shape):
        col = idx[:, axis]
        if col.size and (col.min() < 0 or col.max() >= extent):
            raise ValueError(f"index out of range on axis {axis} (extent {extent})")
    if len(idx) > 1:
        lin = np.ravel_multi_index(tuple(idx.T), shape)
        if np.bincount(lin, minlength=1).max() > 1:
            raise ValueError("duplicate indices within one descriptor")
    return idx


def _row_lines(idx: np.ndarray, shape) -> np.ndarray | None:
    """Rows if ``idx`` is rows_to_entries(rows, n2) for distinct rows, else None."""
    if len(shape) != 2 or idx.shape[0] == 0:
        return None
    n2 = shape[1]
    if idx.shape[0] % n2:
        return None
    blk = idx.reshape(-1, n2, 2)
    if not np.array_equal(blk[:, :, 1], np.broadcast_to(np.arange(n2), blk[:, :, 1].shape)):
        return None
    rows = blk[:, 0, 0]
    if not np.array_equal(blk[:, :, 0], np.broadcast_to(rows[:, None], blk[:, :, 0].shape)):
        return None
    return rows.astype(np.int64)


@dataclass(frozen=True)
class EntryMask:
    """Entry subsampling: measurement l picks the entry at ``indices[l]``."""

    shape: tuple
    indices: np.ndarray
    _rows: object = field(default=None, repr=False, compare=False)

    def __post_init__(self):
        object.__setattr__(self, "shape", tuple(int(n) for n in self.shape))
        object.__setattr__(self, "indices", _as_indices(self.indices, self.shape))
        object.__setattr__(self, "_rows", _row_lines(self.indices, self.shape))

    @property
    def nmeas(self) -> int:
        return len(self.indices)

    @property
    def row_lines(self):
        return self._rows


@dataclass(frozen=True)
class FourierMask:
    """k-space subsampling: measurement l picks DFT coefficient (i, j)."""

    shape: tuple
    indices: np.ndarray
    _rows: object = field(default=None, repr=False, compare=False)

    def __post_init__(self):
        shape = tuple(int(n) for n in self.shape)
        if len(shape) != 2:
            raise ValueError("Fourier masks are defined for 2-D frames")
        object.__setattr__(self, "shape", shape)
        object.__setattr__(self, "indices", _as_indices(self.indices, shape))
        object.__setattr__(self, "_rows", _row_lines(self.indices, shape))

    @property
    def nmeas(self) -> int:
        return len(self.indices)

    @property
    def row_lines(self):
        return self._rows


def descriptor_kind(descriptor) -> str:
    if isinstance(descriptor, FourierMask):
        return "fourier"
    if isinstance(descriptor, EntryMask):
        return "entry"
    raise TypeError(f"unknown descriptor type {type(descriptor).__name__}")


@dataclass(frozen=True)
class MeasurementBatch:
    """One frame's measurements plus the descriptor (observation.py:153-168).
    ``y`` may be a host array or a CUDA tensor; it is kept as given."""

    y: object
    descriptor: object
    t: int = 0
    noise_sigma: float = 0.0

    def __post_init__(self):
        y = self.y
        if isinstance(y, torch.Tensor):
            y = y.reshape(-1)
            n = y.numel()
        else:
            y = np.asarray(y, dtype=np.complex128).ravel()
            n = y.size
        if n != self.descriptor.nmeas:
            raise ValueError(f"batch holds {n} values for {self.descriptor.nmeas} projections")
        object.__setattr__(self, "y", y)

    def y_device(self) -> torch.Tensor:
        y = self.y
        if isinstance(y, torch.Tensor):
            return y.to(device=L.device(), dtype=torch.complex64).contiguous()
        return torch.from_numpy(y.astype(np.complex64)).to(L.device())


# ------------------------------------------------------------------ DFT
def unitary_dft2(image, inverse: bool = False) -> np.ndarray:
    """Unitary 2-D DFT (F1 X F2^T): the column FFT kernel, then the row FFT kernel."""
    x = np.asarray(image, dtype=np.complex128) if not isinstance(image, torch.Tensor) else image
    if x.ndim != 2 or (x.size if isinstance(x, np.ndarray) else x.numel()) == 0:
        raise ValueError("unitary_dft2 expects a nonempty 2-D array")
    t = x.to(L.device(), torch.complex64) if isinstance(x, torch.Tensor) else \
        torch.from_numpy(x.astype(np.complex64)).to(L.device())
    t = K.fft2(t.contiguous(), inverse)                           # F1 X F2^T: a column and a row pass
    return t.cpu().numpy().astype(np.complex128)


def unitary_dft_matrix(n: int) -> np.ndarray:
    """Symmetric unitary 1-D DFT matrix F with F @ x == fft(x, ortho)."""
    eye = torch.eye(n, dtype=torch.complex64, device=L.device())
    return K.fft_cols_(eye).cpu().numpy().astype(np.complex128)


# ------------------------------------------------------------------ build_phi
def build_phi(subspace: TensorSubspace, descriptor) -> np.ndarray:
    """Phi[l, r] = Ah[i_l, r] Bh[j_l, r] (observation.py:219-228) with the
    measurement factors from the column FFT kernel; gathered on device."""
    if subspace.dims != descriptor.shape:
        raise ValueError(f"subspace dims {subspace.dims} do not match descriptor {descriptor.shape}")
    kind = descriptor_kind(descriptor)
    ah, bh = subspace.measurement_factors(kind)
    idx = torch.from_numpy(descriptor.indices).to(ah.device)
    phi = ah.index_select(0, idx[:, 0]) * bh.index_select(0, idx[:, 1])
    return phi.cpu().numpy().astype(np.complex128)


# ------------------------------------------------------------------ masks
def row_distances(n1: int) -> np.ndarray:
    """|signed frequency offset| of each unshifted DFT row (observation.py:274-276)."""
    return np.abs(np.fft.fftfreq(n1, d=1.0 / n1)).astype(np.int64)


def rows_to_entries(rows, n2: int) -> np.ndarray:
    """Full phase-encode lines -> (i, j) entries, row-major (observation.py:326-332)."""
    rows = np.asarray(rows, dtype=np.int64).ravel()
    cols = np.arange(n2, dtype=np.int64)
    return np.stack([np.repeat(rows, n2), np.tile(cols, len(rows))], axis=1)


def philox_position(rng) -> tuple:
    """(key0, key1, position) of a numpy ``Generator(Philox(...))``: the
    stream index of the next 64-bit word (the device draws index the Philox
    stream directly, word n = block n // 4 + 1, lane n % 4)."""
    bg = getattr(rng, "bit_generator", None)
    if bg is None or type(bg).__name__ != "Philox":
        raise TypeError("device draws need a numpy Generator over the Philox bit generator "
                        "(np.random.Generator(np.random.Philox(key)))")
    st = bg.state
    ctr = [int(v) for v in st["state"]["counter"]]
    key = [int(v) for v in st["state"]["key"]]
    if ctr[1] or ctr[2] or ctr[3] or st.get("has_uint32", 0):
        raise TypeError("Philox generator state not supported for device draws (counter beyond 2^64 "
                        "or a buffered 32-bit half)")
    pos = (ctr[0] - 1) * 4 + int(st["buffer_pos"])
    return key[0], key[1], pos


def device_uniforms(rng, k: int):
    """Where the device draws take their k uniforms from: ``("philox", key0, key1, pos)`` for a
    Generator over Philox (the kernels index the stream directly; the host generator is advanced
    afterwards), else ``("table", u)`` with u = rng.random(k) uploaded — exactly the
    Generator.random() values numpy's choice / the sequential draws consume, one per draw, so any
    bit generator (np.random.default_rng(seed) is PCG64, as the reference builds them:
    experiment.py:257,338,453) gets numpy's draws."""
    try:
        return ("philox",) + tuple(philox_position(rng))
    except TypeError:
        u = np.ascontiguousarray(rng.random(int(k)), dtype=np.float64)
        return ("table", torch.from_numpy(u).to(L.device()))


def _advance(rng, n: int) -> None:
    """Keep the host Generator in step with the words consumed on device."""
    if n > 0:
        rng.random(n)


def weighted_draw_without_replacement(weights, k: int, rng) -> np.ndarray:
    """Sequential renormalised draws (observation.py:279-297), on device,
    bit-identical to numpy (any bit generator: ``device_uniforms``)."""
    w = np.asarray(weights, dtype=float)
    if k > np.count_nonzero(w):
        raise ValueError("cannot draw more items than have positive weight")
    if k == 0:
        return np.empty(0, dtype=np.int64)
    src = device_uniforms(rng, k)
    dev = L.device()
    wt = torch.from_numpy(np.ascontiguousarray(w)).to(dev)
    st = torch.zeros(1, dtype=torch.int32, device=dev)
    if src[0] == "philox":
        _, k0, k1, pos = src
        pt = torch.tensor([pos], dtype=torch.int64, device=dev)
        out = K.draw_without_replacement(wt, int(k), (k0, k1), pt, st)
        _advance(rng, int(k))
    else:
        out = K.draw_without_replacement(wt, int(k), None, None, st, uniforms=src[1])
    L.raise_status(int(st.item()), "weighted_draw_without_replacement")
    return out.cpu().numpy().astype(np.int64)


def variable_density_rows(n1: int, alpha: float, fraction: float, rng) -> np.ndarray:
    """Variable-density Cartesian rows (observation.py:300-323): DC first,
    then ceil(fraction n1) - 1 draws without replacement with weight
    d**alpha / 2, in draw order."""
    if not 0.0 < fraction <= 1.0:
        raise ValueError(f"fraction must be in (0, 1], got {fraction}")
    n_rows = int(np.ceil(fraction * n1))
    if n_rows < 1:
        raise ValueError("fraction selects no rows")
    dist = row_distances(n1)
    weights = np.zeros(n1)
    nz = dist > 0
    weights[nz] = dist[nz].astype(float) ** alpha / 2.0
    drawn = weighted_draw_without_replacement(weights, n_rows - 1, rng) if n_rows > 1 else np.empty(0, np.int64)
    return np.concatenate([np.zeros(1, dtype=np.int64), drawn])
