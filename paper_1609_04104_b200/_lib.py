"""ctypes binding of ``libtensortrack_b200.so`` (the C ABI in
``include/tensortrack_b200.h``).

The product path has no CPU fallback: if the library is missing or CUDA is
unavailable, every entry point raises. Status codes map 1:1 onto the
reference's exceptions: 1 -> ValueError, 2 -> TypeError,
3 -> NumericalError, 4 -> RuntimeError.
"""

from __future__ import annotations

import ctypes as C
import os

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libtensortrack_b200.so")

TT_OK, TT_EINVAL, TT_EUNSUPPORTED, TT_ENONFINITE, TT_ECUDA = 0, 1, 2, 3, 4
TT_ST_BADROW, TT_ST_DUPROW, TT_ST_NONFINITE, TT_ST_ZEROCOL, TT_ST_OVERFLOW = 1, 2, 4, 8, 16
TT_POLICY_STATIC, TT_POLICY_INFORMATIVE = 0, 1
TT_Y_GATHER, TT_Y_PACKED = 0, 1
TT_STEP_FIXED, TT_STEP_HESSIAN = 0, 1


class NumericalError(RuntimeError):
    """Non-finite result (experiment.py:66-67)."""


_p = C.c_void_p
_i32 = C.c_int32
_i64 = C.c_int64
_u64 = C.c_uint64
_f64 = C.c_double


class RowsArgs(C.Structure):
    _fields_ = [
        ("nslices", _i32), ("nx", _i32), ("ny", _i32), ("rank", _i32), ("frames", _i32), ("max_rows", _i32),
        ("cluster", _i32), ("t0", _i64),
        ("ah_in", _p), ("bh_in", _p), ("ah_out", _p), ("bh_out", _p), ("alpha_bar", _p),
        ("policy", _i32), ("rows_tab", _p), ("rows_cnt", _p), ("k_draws", _i32), ("forced", _p),
        ("nforced", _i32), ("beta", _f64), ("key0", _u64), ("key1", _u64), ("philox_pos", _p),
        ("y_mode", _i32), ("ysrc", _p), ("y_frame_stride", _i64), ("y_slice_stride", _i64),
        ("lam", _f64), ("step_mode", _i32), ("mu", _f64), ("c_floor", _f64), ("c_cap", _f64),
        ("gamma_out", _p), ("cost_out", _p), ("mu_out", _p), ("alpha_out", _p), ("rows_out", _p),
        ("cnt_out", _p), ("resid_out", _p), ("ah_hist", _p), ("bh_hist", _p), ("status", _p), ("scratch", _p),
        ("phase_clock", _p), ("shard_rank", _i32), ("shard_world", _i32), ("shard_phase", _i32), ("xw", _p),
        ("xg", _p), ("shard_local", _i32), ("shard_fused", _i32), ("grid_sync", _p),
        ("draw_wor", _i32), ("norm_cap", _f64), ("norm_out", _p), ("sraw_in", _p), ("y_host", _i32),
    ]


class EntriesArgs(C.Structure):
    _fields_ = [
        ("nx", _i32), ("ny", _i32), ("rank", _i32), ("nmeas", _i32), ("t", _i64),
        ("ah_in", _p), ("bh_in", _p), ("ah_out", _p), ("bh_out", _p), ("alpha_bar", _p),
        ("idx", _p), ("y", _p), ("lam", _f64), ("step_mode", _i32), ("mu", _f64), ("c_floor", _f64),
        ("c_cap", _f64), ("gamma_out", _p), ("cost_out", _p), ("mu_out", _p), ("alpha_out", _p),
        ("resid_out", _p), ("status", _p), ("scratch", _p), ("nmeas_dev", _p), ("omega", _p), ("frame", _p),
    ]


class PatchesArgs(C.Structure):
    _fields_ = [
        ("nx", _i32), ("ny", _i32), ("pn1", _i32), ("pn2", _i32), ("rank", _i32),
        ("patch0", _i32), ("npatch_local", _i32), ("frames", _i32),
        ("pidx", _p), ("py", _p), ("pcnt", _p), ("nsteps", _i32), ("sched", _p),
        ("a", _p), ("b", _p), ("t", _p), ("alpha_bar", _p),
        ("lam", _f64), ("step_mode", _i32), ("mu", _f64), ("c_floor", _f64), ("c_cap", _f64),
        ("project", _i32), ("gamma_out", _p), ("cost_out", _p), ("mu_out", _p), ("resid_out", _p),
        ("recon_out", _p), ("status", _p),
    ]


# (name, restype, argtypes) — every symbol declared in include/tensortrack_b200.h
SIGNATURES = {
    "tt_version": (C.c_char_p, []),
    "tt_last_error": (C.c_char_p, []),
    "tt_fft_cols": (C.c_int, [_p, _p, C.c_int, C.c_int, C.c_int, C.c_int]),
    "tt_fft_rows": (C.c_int, [_p, _p, C.c_longlong, C.c_int, C.c_int]),
    "tt_rows_plan": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int),
                               C.POINTER(C.c_size_t)]),
    "tt_rows_scratch_bytes": (C.c_size_t, [C.c_int] * 6),
    "tt_track_rows": (C.c_int, [_p, C.POINTER(RowsArgs)]),
    "tt_rows_shard_xg_len": (C.c_size_t, [C.c_int]),
    "tt_rows_mirror_fits": (C.c_int, [C.c_int] * 5),
    "tt_rows_plan_info": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _p]),
    "tt_rows_max_clusters": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _p]),
    "tt_rows_shard_reduce": (C.c_int, [_p, C.c_int, C.c_int, C.c_int, _p, _p]),
    "tt_entries_scratch_bytes": (C.c_size_t, [C.c_int] * 4),
    "tt_track_entries": (C.c_int, [_p, C.POINTER(EntriesArgs)]),
    "tt_gather_entries": (C.c_int, [_p, C.c_int, C.c_int, _p, _p, _p, C.c_int, _p, _p]),
    "tt_draw_scratch_bytes": (C.c_size_t, [C.c_int]),
    "tt_cten_info": (C.c_int, [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int), _p, C.c_int]),
    "tt_cten_read": (C.c_int, [C.c_char_p, _p, C.c_size_t, C.c_int]),
    "tt_cten_write": (C.c_int, [C.c_char_p, _p, C.c_int, C.c_int, C.c_int, _p]),
    "tt_draw_with_replacement_large": (C.c_int, [_p, C.c_int, _p, C.c_int, _p, C.c_int, C.c_uint64, C.c_uint64, _p,
                                                 _p, _p, _p]),
    "tt_rows_shard_energy": (C.c_int, [_p, C.c_int, C.c_int, C.c_int, C.c_int, _p, _p]),
    "tt_rows_shard_scores": (C.c_int, [_p, C.c_int, C.c_int, C.c_int, _p, _p, _p]),
    "tt_factor_norms2": (C.c_int, [_p, C.c_int, C.c_size_t, _p, _p]),
    "tt_vd_rows_batch": (C.c_int, [_p, C.c_int, C.c_int, C.c_int, _p, C.c_int, C.c_uint64, C.c_uint64, _p, _p]),
    "tt_terms_scratch_bytes": (C.c_size_t, [C.c_int, C.c_int, C.c_int]),
    "tt_residual": (C.c_int, [_p, C.c_int, C.c_int, C.c_int, C.c_int, _p, _p, _p, _p, _p, _p]),
    "tt_data_terms": (C.c_int, [_p, C.c_int, C.c_int, C.c_int, C.c_int, _p, _p, _p, _p, _p, _p, _p, _p, _p]),
    "tt_row_scores": (C.c_int, [_p, C.c_int, C.c_int, C.c_int, C.c_int, _p, _f64, _p, _p]),
    "tt_entry_scores": (C.c_int, [_p, C.c_int, C.c_int, C.c_int, _p, _p, _f64, _p, _p]),
    "tt_entry_scores_ws_bytes": (C.c_size_t, [C.c_int, C.c_int]),
    "tt_entry_scores_ws": (C.c_int, [_p, C.c_int, C.c_int, C.c_int, _p, _p, _f64, _p, _p, _p]),
    "tt_draw_with_replacement": (C.c_int, [_p, C.c_int, C.c_int, _p, C.c_int, _p, C.c_int, _u64, _u64, _p, _p,
                                           _p]),
    "tt_draw_without_replacement": (C.c_int, [_p, C.c_int, _p, C.c_int, _u64, _u64, _p, _p, _p]),
    "tt_draw_with_replacement_u": (C.c_int, [_p, C.c_int, C.c_int, _p, C.c_int, _p, C.c_int, _p, _p, _p]),
    "tt_draw_with_replacement_large_u": (C.c_int, [_p, C.c_int, _p, C.c_int, _p, C.c_int, _p, _p, _p, _p, _p]),
    "tt_draw_without_replacement_u": (C.c_int, [_p, C.c_int, _p, C.c_int, _p, _p, _p]),
    "tt_reconstruct": (C.c_int, [_p, C.c_int, C.c_int, C.c_int, C.c_int, _p, _p, _p, _p]),
    "tt_nmse": (C.c_int, [_p, C.c_int, C.c_size_t, _p, _p, _p, _p]),
    "tt_nmse_work_doubles": (C.c_size_t, [C.c_int]),
    "tt_rebalance": (C.c_int, [_p, C.c_int, C.c_int, C.c_int, C.c_int, _p, _p, _p]),
    "tt_patches_smem_bytes": (C.c_size_t, [C.c_int, C.c_int, C.c_int]),
    "tt_patch_bin": (C.c_int, [_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _p, _p, _p, _p, _p, _p, _p]),
    "tt_track_patches": (C.c_int, [_p, C.POINTER(PatchesArgs)]),
    "tt_solve_scratch_bytes": (C.c_size_t, [C.c_int, C.c_int]),
    "tt_solve_gamma": (C.c_int, [_p, C.c_int, C.c_int, _p, _p, _f64, _p, _p]),
}

_LIB = None


def load(path: str = LIB_PATH):
    """Load the shared library (no CUDA context needed). Raises if absent."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(path):
        raise RuntimeError(
            f"{path} is missing: build it with `python -m paper_1609_04104_b200._build` "
            "(there is no CPU fallback)")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = lib
    return lib


def lib():
    return load()


def check(rc: int, what: str = "") -> None:
    if rc == TT_OK:
        return
    msg = lib().tt_last_error().decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if rc == TT_EINVAL:
        raise ValueError(text)
    if rc == TT_EUNSUPPORTED:
        raise TypeError(text)
    if rc == TT_ENONFINITE:
        raise NumericalError(text)
    raise RuntimeError(text)


def raise_status(st: int, what: str = "") -> None:
    """Map device status bits to the reference's exceptions."""
    if not st:
        return
    if st & (TT_ST_BADROW | TT_ST_DUPROW | TT_ST_OVERFLOW):
        kinds = []
        if st & TT_ST_BADROW:
            kinds.append("index out of range")
        if st & TT_ST_DUPROW:
            kinds.append("duplicate indices within one descriptor")
        if st & TT_ST_OVERFLOW:
            kinds.append("too many rows")
        raise ValueError(f"{what}: " + ", ".join(kinds))
    if st & TT_ST_ZEROCOL:
        raise ValueError(f"{what}: all-zero column; scores undefined")
    if st & TT_ST_NONFINITE:
        raise NumericalError(f"{what}: non-finite result")


def device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("tensortrack_b200 needs a CUDA device (sm_100a); there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)
_raw_device = getattr(torch._C, "_cuda_getDevice", None)


def stream_ptr() -> int:
    """The current torch stream's cudaStream_t (every launch asks: the raw accessors skip the ~15 us of
    ``torch.cuda.current_stream()``'s device-index plumbing)."""
    if _raw_stream is not None and _raw_device is not None and torch.cuda.is_initialized():
        return _raw_stream(_raw_device())
    return torch.cuda.current_stream().cuda_stream


def ptr(t) -> int | None:
    if t is None:
        return None
    return t.data_ptr()


def f32view(t: torch.Tensor) -> torch.Tensor:
    """complex64 tensor -> the raw buffer it owns (for data_ptr only)."""
    return t
