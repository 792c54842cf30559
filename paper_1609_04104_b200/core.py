"""Device-backed PARAFAC subspace values — drop-in for ``tensortrack.core``
(`pkg/src/tensortrack/core.py`).

``TensorSubspace`` keeps the reference constructor and accessors
(``factors``, ``rank``, ``dims``, ``nmodes``, ``basis_tensor``;
core.py:39-73) but owns device buffers. A subspace produced by the tracker
holds its *measurement-domain* factors on the GPU:

* ``kind == "image"``: the resident buffers are the k-space factors
  ``F_x A, F_y B`` of image-domain factors ``A, B`` (FourierMask tracking);
* ``kind == "direct"``: the resident buffers are the factors themselves
  (EntryMask tracking, i.e. k-space interpolation).

Host arrays (``.factors``, complex128 like the reference) are materialised
lazily, through the inverse column FFT kernel when needed. Values are never
mutated after construction (core.py:6-7), so buffers are shared freely.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib as L
from . import _ops as K

__all__ = ["TensorSubspace", "synthesize_slice", "rebalance", "outer_rank_one", "singular_values", "rank_surrogate",
           "unfold", "refold"]


def _as_factor(a) -> np.ndarray:
    a = np.asarray(a, dtype=np.complex128)
    if a.ndim != 2:
        raise ValueError(f"factor matrix must be 2-D, got shape {a.shape}")
    if a.shape[0] < 1 or a.shape[1] < 1:
        raise ValueError(f"factor matrix must be nonempty, got shape {a.shape}")
    return a


def _to_dev(a: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.complex64)).to(L.device(), non_blocking=False)


class TensorSubspace:
    """Rank-R subspace held as M-1 factor matrices (core.py:39-73)."""

    __slots__ = ("_host", "_dev", "_kind", "_dims", "_rank", "_cache")

    def __init__(self, factors):
        if isinstance(factors, TensorSubspace):
            factors = factors.factors
        factors = tuple(factors)
        if len(factors) == 2 and all(isinstance(f, torch.Tensor) and f.is_cuda for f in factors):
            # device factors stay on the device (no host round trip): copied once as complex64, the
            # reference's copy-on-construction (core.py:47-52), validated like host factors
            for f in factors:
                if f.dim() != 2:
                    raise ValueError(f"factor matrix must be 2-D, got shape {tuple(f.shape)}")
                if f.shape[0] < 1 or f.shape[1] < 1:
                    raise ValueError(f"factor matrix must be nonempty, got shape {tuple(f.shape)}")
            if factors[0].shape[1] != factors[1].shape[1]:
                raise ValueError(f"factor ranks differ: {sorted({int(f.shape[1]) for f in factors})}")
            dev = L.device()
            a, b = (f.detach().to(dev, torch.complex64).clone().contiguous() for f in factors)
            self._host, self._dev, self._kind = None, (a, b), "direct"
            self._dims = (int(a.shape[0]), int(b.shape[0]))
            self._rank = int(a.shape[1])
            self._cache = {}
            return
        facs = []
        for f in factors:
            if isinstance(f, torch.Tensor):
                f = f.detach().cpu().numpy()
            facs.append(_as_factor(f))
        facs = tuple(facs)
        if not facs:
            raise ValueError("subspace needs at least one factor matrix")
        ranks = {f.shape[1] for f in facs}
        if len(ranks) != 1:
            raise ValueError(f"factor ranks differ: {sorted(ranks)}")
        self._host = facs
        self._dev = None
        self._kind = None
        self._dims = tuple(f.shape[0] for f in facs)
        self._rank = facs[0].shape[1]
        self._cache = {}

    # ------------------------------------------------------------ construction from device
    @classmethod
    def _from_device(cls, ma: torch.Tensor, mb: torch.Tensor, kind: str) -> "TensorSubspace":
        obj = cls.__new__(cls)
        obj._host = None
        obj._dev = (ma, mb)
        obj._kind = kind
        obj._dims = (int(ma.shape[0]), int(mb.shape[0]))
        obj._rank = int(ma.shape[1])
        obj._cache = {}
        return obj

    # ------------------------------------------------------------ reference accessors
    @property
    def factors(self) -> tuple:
        if self._host is None:
            a, b = self.torch_factors()
            self._host = (a.cpu().numpy().astype(np.complex128), b.cpu().numpy().astype(np.complex128))
        return self._host

    @property
    def rank(self) -> int:
        return self._rank

    @property
    def dims(self) -> tuple:
        return self._dims

    @property
    def nmodes(self) -> int:
        return len(self._dims)

    def basis_tensor(self, r: int) -> np.ndarray:
        a, b = self.factors
        return np.multiply.outer(a[:, r], b[:, r])

    def __repr__(self):
        where = "host" if self._dev is None else f"cuda/{self._kind}"
        return f"TensorSubspace(dims={self.dims}, rank={self.rank}, {where})"

    # ------------------------------------------------------------ device views
    def _require_two_modes(self):
        if self.nmodes != 2:
            raise TypeError("the B200 tracker handles two-mode (matrix) subspaces only")

    def torch_factors(self) -> tuple:
        """Visible factors (A, B) as complex64 CUDA tensors."""
        self._require_two_modes()
        if "visible" in self._cache:
            return self._cache["visible"]
        if self._dev is None:
            out = (_to_dev(self._host[0]), _to_dev(self._host[1]))
        elif self._kind == "direct":
            out = self._dev
        else:
            out = (K.fft_cols(self._dev[0], inverse=True), K.fft_cols(self._dev[1], inverse=True))
        self._cache["visible"] = out
        return out

    def measurement_factors(self, kind: str) -> tuple:
        """Factors as the sketch sees them: (F_x A, F_y B) for ``"fourier"``
        (observation.py:225-226), (A, B) for ``"entry"``. Device tensors,
        read-only by convention."""
        self._require_two_modes()
        if kind == "entry":
            return self.torch_factors()
        if kind != "fourier":
            raise TypeError(f"unknown measurement kind {kind!r}")
        if self._dev is not None and self._kind == "image":
            return self._dev
        if "fourier" in self._cache:
            return self._cache["fourier"]
        a, b = self.torch_factors()
        out = (K.fft_cols(a), K.fft_cols(b))
        self._cache["fourier"] = out
        return out


def _gamma_dev(gamma, rank: int) -> torch.Tensor:
    if isinstance(gamma, torch.Tensor):
        g = gamma.to(device=L.device(), dtype=torch.complex64).reshape(-1)
    else:
        g = torch.from_numpy(np.asarray(gamma, dtype=np.complex128).ravel().astype(np.complex64)).to(L.device())
    if g.numel() != rank:
        raise ValueError(f"gamma length {g.numel()} does not match rank {rank}")
    return g.contiguous()


def synthesize_device(subspace: TensorSubspace, gamma) -> torch.Tensor:
    """sum_r gamma_r a_r b_r^T on the GPU (complex64, (N1, N2))."""
    a, b = subspace.torch_factors()
    g = _gamma_dev(gamma, subspace.rank)
    return K.reconstruct(a.unsqueeze(0).contiguous(), b.unsqueeze(0).contiguous(), g.unsqueeze(0))[0]


def synthesize_slice(subspace: TensorSubspace, gamma) -> np.ndarray:
    """Dense slice sum_r gamma_r a_r o b_r (core.py:91-104); plain transpose."""
    if not isinstance(subspace, TensorSubspace):
        subspace = TensorSubspace(subspace.factors)
    return synthesize_device(subspace, gamma).cpu().numpy().astype(np.complex128)


def rebalance(subspace: TensorSubspace) -> TensorSubspace:
    """Per-component geometric-mean column norms (core.py:138-166).

    The per-column scales are real, so they apply unchanged to the k-space
    factors (Parseval): a device subspace keeps its kind."""
    subspace._require_two_modes()
    if subspace._dev is not None:
        a, b = subspace._dev[0].clone(), subspace._dev[1].clone()
        kind = subspace._kind
    else:
        a, b = subspace.torch_factors()
        a, b = a.clone(), b.clone()
        kind = "direct"
    st = torch.zeros(1, dtype=torch.int32, device=a.device)
    K.rebalance_(a, b, st)
    if int(st.item()) & L.TT_ST_ZEROCOL:
        raise ValueError("a component is zero in some modes but not all")
    return TensorSubspace._from_device(a, b, kind)


# ---------------------------------------------------------------- small host utilities (core.py:76-190)
# Off the hot path: shape bookkeeping and norms the reference exposes next to the subspace type.
def outer_rank_one(vectors) -> np.ndarray:
    """Outer product of the given vectors (core.py:76-88)."""
    from functools import reduce

    vecs = [np.asarray(v, dtype=np.complex128).ravel() for v in vectors]
    if not vecs:
        raise ValueError("outer product of an empty vector list")
    if any(v.size == 0 for v in vecs):
        raise ValueError("outer product with an empty vector")
    return reduce(np.multiply.outer, vecs)


def singular_values(subspace: TensorSubspace, mode_m_factor=None) -> np.ndarray:
    """Per-component sigma_r = prod_m ||a_r^(m)|| over the factors (plus an optional trailing
    mode-M factor), in column order (core.py:107-121)."""
    mats = list(subspace.factors)
    if mode_m_factor is not None:
        f = _as_factor(mode_m_factor)
        if f.shape[1] != subspace.rank:
            raise ValueError("mode-M factor rank does not match subspace rank")
        mats.append(f)
    return np.prod(np.stack([np.linalg.norm(f, axis=0) for f in mats]), axis=0)


def rank_surrogate(factors) -> float:
    """(1/M) sum_m ||A_m||_F^2 (core.py:124-135)."""
    mats = [_as_factor(f) for f in factors]
    if not mats:
        raise ValueError("rank surrogate of an empty factor list")
    return float(sum(np.linalg.norm(f) ** 2 for f in mats)) / len(mats)


def unfold(tensor, mode: int) -> np.ndarray:
    """Mode-``mode`` (1-based) unfolding, remaining indices ascending, last fastest (core.py:169-178)."""
    tensor = np.asarray(tensor)
    if not 1 <= mode <= tensor.ndim:
        raise ValueError(f"mode {mode} out of range for {tensor.ndim}-way tensor")
    return np.moveaxis(tensor, mode - 1, 0).reshape(tensor.shape[mode - 1], -1)


def refold(matrix, mode: int, dims) -> np.ndarray:
    """Inverse of :func:`unfold` (core.py:181-190)."""
    dims = tuple(int(d) for d in dims)
    if not 1 <= mode <= len(dims):
        raise ValueError(f"mode {mode} out of range for dims {dims}")
    rest = dims[: mode - 1] + dims[mode:]
    return np.moveaxis(np.asarray(matrix).reshape((dims[mode - 1],) + rest), 0, mode - 1)
