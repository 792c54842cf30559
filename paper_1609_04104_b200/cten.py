"""CTEN container I/O — the reference's interchange format for truth tensors and
reconstructions (`cten.py:1-74`; read by `experiment.py:700`, written at
`experiment.py:719`, used by the CLI `cli.py:96-121`).

Layout (little-endian): b"CTEN" | u8 version 1 | u8 dtype (0: float32 pairs,
1: float64 pairs) | u8 ndim | ndim x u32 dims | row-major (real, imag) payload.

Parsing, validation and conversion are native (``tt_cten_*`` in the C ABI,
host code); the same malformed inputs the reference rejects raise
:class:`CtenFormatError`. ``read_cten``/``write_cten`` keep the reference's
signatures and complex128 results (bit-exact round trips for matching
dtypes); ``read_cten_tensor`` loads straight into a (pinned) complex64 torch
tensor for the device engines.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np
import torch

from . import _lib as L

__all__ = ["CtenFormatError", "write_cten", "read_cten", "read_cten_tensor", "cten_info"]


class CtenFormatError(ValueError):
    """Raised for malformed CTEN payloads or headers (cten.py:27-28)."""


def _call(rc: int, what: str) -> None:
    if rc == L.TT_OK:
        return
    msg = L.lib().tt_last_error()
    msg = msg.decode() if isinstance(msg, bytes) else str(msg)
    if rc == L.TT_EINVAL:
        raise CtenFormatError(msg)
    L.check(rc, what)


def _path(path) -> bytes:
    p = os.fspath(path)
    if not os.path.exists(p):
        raise FileNotFoundError(p)
    return p.encode()


def cten_info(path) -> tuple[int, tuple[int, ...]]:
    """(dtype_code, dims) of a CTEN file."""
    code, nd = C.c_int(), C.c_int()
    dims = (C.c_uint32 * 32)()
    _call(L.lib().tt_cten_info(_path(path), C.byref(code), C.byref(nd), C.cast(dims, C.c_void_p), 32), "cten_info")
    return code.value, tuple(int(dims[i]) for i in range(nd.value))


def write_cten(path, array, dtype_code: int = 1) -> None:
    """cten.py:33-46: complex data stored as float32 (0) or float64 (1) pairs."""
    if dtype_code not in (0, 1):
        raise CtenFormatError(f"unknown dtype code {dtype_code}")
    a = np.ascontiguousarray(np.asarray(array, dtype=np.complex128))
    if a.ndim < 1:
        a = a.reshape(1)
    dims = (C.c_uint32 * max(1, a.ndim))(*a.shape)
    _call(L.lib().tt_cten_write(os.fspath(path).encode(), a.ctypes.data if a.size else None, 1, int(dtype_code),
                                a.ndim, C.cast(dims, C.c_void_p)), "write_cten")


def read_cten(path) -> np.ndarray:
    """cten.py:49-74: complex128 array with the stored dims."""
    _, dims = cten_info(path)
    out = np.empty(dims, dtype=np.complex128)
    _call(L.lib().tt_cten_read(_path(path), out.ctypes.data if out.size else None, out.size, 1), "read_cten")
    # the reference assembles real + 1j * imag (cten.py:72-73): a non-finite imaginary part makes the real
    # part NaN (0 * inf); kept for drop-in parity
    bad = ~np.isfinite(out.imag)
    if bad.any():  # same arithmetic as the reference, so even the NaN bits agree
        fix = out.real[bad].astype(np.complex128)
        with np.errstate(invalid="ignore"):
            fix += 1j * out.imag[bad]
        out[bad] = fix
    return out


def read_cten_tensor(path, pin: bool = True) -> torch.Tensor:
    """The payload as a complex64 CPU tensor (pinned by default, ready for asynchronous upload)."""
    _, dims = cten_info(path)
    out = torch.empty(dims, dtype=torch.complex64, pin_memory=pin and torch.cuda.is_available())
    _call(L.lib().tt_cten_read(_path(path), out.data_ptr() if out.numel() else None, out.numel(), 0), "read_cten")
    return out
