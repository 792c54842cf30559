"""Thin torch-facing wrappers over the C ABI. Tensors are CUDA tensors;
nothing here computes on the CPU. Used by the reference-mirroring API
modules and by the device-resident engine."""

from __future__ import annotations

import ctypes as C

import numpy as np

import torch

from . import _lib as L

C64 = torch.complex64


def _need(t: torch.Tensor, dtype, name: str):
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")


def fft_cols_(x: torch.Tensor, inverse: bool = False) -> torch.Tensor:
    """In-place ortho DFT down the columns of (..., n, ncols) complex64."""
    _need(x, C64, "x")
    n, ncols = x.shape[-2], x.shape[-1]
    batch = x.numel() // max(1, n * ncols)
    if x.numel() == 0:
        return x
    done = 0
    while done < batch:  # grid.y limit
        nb = min(65535, batch - done)
        view = x.reshape(batch, n, ncols)[done:done + nb]
        L.check(L.lib().tt_fft_cols(L.stream_ptr(), view.data_ptr(), n, ncols, nb, 1 if inverse else 0),
                "fft_cols")
        done += nb
    return x


def fft_cols(x: torch.Tensor, inverse: bool = False) -> torch.Tensor:
    return fft_cols_(x.clone(), inverse)


FFT_ROWS_N = (16, 32, 64, 128, 256, 512, 1024)  # row lengths tt_fft_rows transforms (the register kernel's sizes)


def fft_rows_(x: torch.Tensor, inverse: bool = False) -> torch.Tensor:
    """In-place ortho DFT along the last axis of (..., n) complex64, n in FFT_ROWS_N."""
    _need(x, C64, "x")
    n = x.shape[-1]
    if x.numel() == 0:
        return x
    L.check(L.lib().tt_fft_rows(L.stream_ptr(), x.data_ptr(), x.numel() // n, n, 1 if inverse else 0), "fft_rows")
    return x


def fft2_(x: torch.Tensor, inverse: bool = False) -> torch.Tensor:
    """In-place unshifted ortho 2-D DFT of (..., nx, ny) complex64 frames (observation.py:171-183): a column
    pass and a row pass over the same buffer; row lengths the row kernel does not take go through a
    transposed copy and a second column pass."""
    _need(x, C64, "x")
    fft_cols_(x, inverse)
    if x.shape[-1] in FFT_ROWS_N:
        return fft_rows_(x, inverse)
    xt = fft_cols_(x.transpose(-1, -2).contiguous(), inverse)
    x.copy_(xt.transpose(-1, -2))
    return x


def fft2(x: torch.Tensor, inverse: bool = False) -> torch.Tensor:
    return fft2_(x.clone(), inverse)


_MAX_CLUSTERS: dict = {}  # (device, nx, ny, rank, max_rows, cluster) -> resident clusters (the query takes ~1 ms)


def _max_clusters(nx, ny, rank, max_rows, cluster) -> int:
    key = (torch.cuda.current_device(), nx, ny, rank, max_rows, cluster)
    n = _MAX_CLUSTERS.get(key)
    if n is None:
        out = C.c_int(0)
        L.check(L.lib().tt_rows_max_clusters(nx, ny, rank, max_rows, cluster, C.byref(out)), "rows cluster occupancy")
        n = _MAX_CLUSTERS[key] = out.value
    return n


class RowsScratch:
    """Cached scratch / plan for one (nslices, nx, ny, R, max_rows) shape."""

    def __init__(self, nslices, nx, ny, rank, max_rows, cluster=0, policy=0, dev=None):
        sm = C.c_size_t(0)
        if int(cluster) <= 0:
            # widest cluster that keeps every slice's cluster resident at once: 16 CTAs for one
            # slice (latency), 2 for 64 slices. The device holds fewer than 148 / c clusters of 8
            # or 16 CTAs (8 GPCs of 16-20 SMs: tt_rows_max_clusters asks the occupancy
            # calculator), and a launch with more slices than that runs in two waves.
            cl = None
            for c in (16, 8, 4, 2, 1):
                if c > 1 and nslices * c > 148:
                    continue
                t = C.c_int(c)
                if L.lib().tt_rows_plan(nx, ny, rank, max_rows, policy, C.byref(t), C.byref(sm)) != 0:
                    continue
                if c > 1 and nslices > _max_clusters(nx, ny, rank, max_rows, c):
                    continue
                cl = t
                break
            if cl is None:
                cl = C.c_int(0)
                L.check(L.lib().tt_rows_plan(nx, ny, rank, max_rows, policy, C.byref(cl), C.byref(sm)),
                        "rows plan")
        else:
            cl = C.c_int(int(cluster))
            L.check(L.lib().tt_rows_plan(nx, ny, rank, max_rows, policy, C.byref(cl), C.byref(sm)), "rows plan")
        self.cluster = cl.value
        self.smem = sm.value
        nbytes = L.lib().tt_rows_scratch_bytes(nslices, nx, ny, rank, max_rows, self.cluster)
        self.buf = torch.empty(int(nbytes), dtype=torch.uint8, device=dev or L.device())
        self.key = (nslices, nx, ny, rank, max_rows, self.cluster)


def rows_plan_fits(nx, ny, rank, max_rows) -> bool:
    cl = C.c_int(0)
    sm = C.c_size_t(0)
    return L.lib().tt_rows_plan(nx, ny, rank, max_rows, 0, C.byref(cl), C.byref(sm)) == 0


_scratch_cache: dict = {}


def rows_scratch(nslices, nx, ny, rank, max_rows, cluster=0) -> RowsScratch:
    k = (nslices, nx, ny, rank, max_rows, cluster, torch.cuda.current_device())
    s = _scratch_cache.get(k)
    if s is None:
        s = RowsScratch(nslices, nx, ny, rank, max_rows, cluster)
        _scratch_cache[k] = s
    return s


def track_rows(args: L.RowsArgs) -> None:
    L.check(L.lib().tt_track_rows(L.stream_ptr(), C.byref(args)), "track_rows")


def track_entries(args: L.EntriesArgs) -> None:
    L.check(L.lib().tt_track_entries(L.stream_ptr(), C.byref(args)), "track_entries")


_ent_cache: dict = {}


def entries_scratch(nx, ny, rank) -> torch.Tensor:
    k = (nx, ny, rank, torch.cuda.current_device())
    s = _ent_cache.get(k)
    if s is None:
        s = torch.zeros(int(L.lib().tt_entries_scratch_bytes(nx, ny, rank, 0)), dtype=torch.uint8,
                        device=L.device())  # zero-filled before first use (frame stamps)
        _ent_cache[k] = s
    return s


def row_scores(a: torch.Tensor, ny: int, beta: float, status: torch.Tensor | None = None) -> torch.Tensor:
    """a: (nslices, nx, R) or (nx, R) complex64 -> fp64 (nslices, nx) / (nx,)."""
    _need(a, C64, "factor")
    squeeze = a.dim() == 2
    a3 = a.reshape(-1, a.shape[-2], a.shape[-1])
    ns, nx, R = a3.shape
    out = torch.empty(ns, nx, dtype=torch.float64, device=a.device)
    st = status if status is not None else torch.zeros(ns, dtype=torch.int32, device=a.device)
    L.check(L.lib().tt_row_scores(L.stream_ptr(), ns, nx, ny, R, a3.data_ptr(), float(beta), out.data_ptr(),
                                  st.data_ptr()), "row_scores")
    return out[0] if squeeze else out


def entry_scores(a: torch.Tensor, b: torch.Tensor, beta: float, status: torch.Tensor) -> torch.Tensor:
    _need(a, C64, "a")
    _need(b, C64, "b")
    nx, R = a.shape
    ny = b.shape[0]
    out = torch.empty(nx, ny, dtype=torch.float64, device=a.device)
    L.check(L.lib().tt_entry_scores(L.stream_ptr(), nx, ny, R, a.data_ptr(), b.data_ptr(), float(beta),
                                    out.data_ptr(), status.data_ptr()), "entry_scores")
    return out


def draw_with_replacement(probs: torch.Tensor, k: int, forced: torch.Tensor | None, key: tuple[int, int] | None,
                          pos: torch.Tensor | None, uniforms: torch.Tensor | None = None):
    """probs (nslices, n) fp64; pos (nslices,) uint64-as-int64 in/out (Philox stream ``key``), or
    ``uniforms`` (nslices, k - nforced) fp64: the Generator.random() values the draws consume."""
    _need(probs, torch.float64, "probs")
    ns, n = probs.shape
    omega = torch.empty(ns, k, dtype=torch.int32, device=probs.device)
    cnt = torch.empty(ns, dtype=torch.int32, device=probs.device)
    nf = 0 if forced is None else int(forced.numel())
    if uniforms is not None:
        _need(uniforms, torch.float64, "uniforms")
        if uniforms.numel() != ns * (k - nf):
            raise ValueError("uniforms: one value per draw and slice")
    fp = None if nf == 0 else forced.data_ptr()
    up = None if uniforms is None or uniforms.numel() == 0 else uniforms.data_ptr()
    if 24 * n + 512 > 220 * 1024:  # domain beyond one CTA's shared memory (entry sampling): global-memory path
        scr = torch.zeros(int(L.lib().tt_draw_scratch_bytes(n)), dtype=torch.uint8, device=probs.device)
        for s in range(ns):
            if uniforms is not None:
                p1 = torch.zeros(1, dtype=torch.int64, device=probs.device)
                L.check(L.lib().tt_draw_with_replacement_large_u(
                    L.stream_ptr(), n, probs[s].data_ptr(), int(k), fp, nf,
                    None if up is None else up + 8 * s * (k - nf), p1.data_ptr(), omega[s].data_ptr(),
                    cnt[s:s + 1].data_ptr(), scr.data_ptr()), "draw_samples")
                continue
            L.check(L.lib().tt_draw_with_replacement_large(
                L.stream_ptr(), n, probs[s].data_ptr(), int(k), fp, nf,
                int(key[0]), int(key[1]) + s, pos[s:s + 1].data_ptr(), omega[s].data_ptr(), cnt[s:s + 1].data_ptr(),
                scr.data_ptr()), "draw_samples")
        return omega, cnt
    if uniforms is not None:
        L.check(L.lib().tt_draw_with_replacement_u(L.stream_ptr(), ns, n, probs.data_ptr(), int(k), fp, nf, up,
                                                   omega.data_ptr(), cnt.data_ptr()), "draw_samples")
        return omega, cnt
    L.check(L.lib().tt_draw_with_replacement(L.stream_ptr(), ns, n, probs.data_ptr(), int(k), fp, nf, int(key[0]),
                                             int(key[1]), pos.data_ptr(), omega.data_ptr(), cnt.data_ptr()),
            "draw_samples")
    return omega, cnt


def draw_without_replacement(weights: torch.Tensor, k: int, key: tuple[int, int] | None, pos: torch.Tensor | None,
                             status: torch.Tensor, uniforms: torch.Tensor | None = None) -> torch.Tensor:
    """k sequential draws from the Philox stream ``key`` at ``pos``, or from ``uniforms`` (k fp64)."""
    _need(weights, torch.float64, "weights")
    out = torch.empty(max(k, 1), dtype=torch.int32, device=weights.device)
    if uniforms is not None:
        _need(uniforms, torch.float64, "uniforms")
        if uniforms.numel() != k:
            raise ValueError("uniforms: one value per draw")
        L.check(L.lib().tt_draw_without_replacement_u(L.stream_ptr(), weights.numel(), weights.data_ptr(), int(k),
                                                      uniforms.data_ptr() if k else None, out.data_ptr(),
                                                      status.data_ptr()), "weighted_draw_without_replacement")
        return out[:k]
    L.check(L.lib().tt_draw_without_replacement(L.stream_ptr(), weights.numel(), weights.data_ptr(), int(k),
                                                int(key[0]), int(key[1]), pos.data_ptr(), out.data_ptr(),
                                                status.data_ptr()), "weighted_draw_without_replacement")
    return out[:k]


def vd_rows_batch(frames: int, nslices: int, n: int, alpha: float, n_rows: int, key: tuple[int, int],
                  pos0: torch.Tensor | None, out: torch.Tensor | None = None) -> torch.Tensor:
    """variable_density_rows for ``frames`` x ``nslices`` (frame f of slice s from the Philox stream
    (key0, key1 + s) at pos0[s] + f (n_rows - 1)) -> (frames, nslices, n_rows) int32, draw order."""
    from .observation import row_distances

    dist = row_distances(n)
    w = np.zeros(n)
    nz = dist > 0
    w[nz] = dist[nz].astype(float) ** alpha / 2.0  # observation.py:317-318, on the host exactly as numpy
    if n_rows - 1 > int(np.count_nonzero(w)):
        raise ValueError("cannot draw more items than have positive weight")
    dev = L.device()
    wt = torch.from_numpy(w).to(dev)
    if out is None:
        out = torch.empty(frames, nslices, n_rows, dtype=torch.int32, device=dev)
    if pos0 is not None:
        _need(pos0, torch.int64, "pos0")
    L.check(L.lib().tt_vd_rows_batch(L.stream_ptr(), int(frames), int(nslices), int(n), wt.data_ptr(), int(n_rows),
                                     int(key[0]), int(key[1]), pos0.data_ptr() if pos0 is not None else None,
                                     out.data_ptr()), "variable_density_rows")
    return out


def reconstruct(a: torch.Tensor, b: torch.Tensor, gamma: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """a (F, nx, R), b (F, ny, R), gamma (F, R) complex64 -> (F, nx, ny) (into ``out`` when given)."""
    for t, n in ((a, "a"), (b, "b"), (gamma, "gamma")):
        _need(t, C64, n)
    F, nx, R = a.shape
    ny = b.shape[1]
    if out is None:
        out = torch.empty(F, nx, ny, dtype=C64, device=a.device)
    elif out.dtype != C64 or not out.is_contiguous() or out.numel() != F * nx * ny:
        raise ValueError("reconstruct: out must be a contiguous complex64 tensor of F*nx*ny elements")
    done = 0
    while done < F:
        nf = min(65535, F - done)
        L.check(L.lib().tt_reconstruct(L.stream_ptr(), nf, nx, ny, R, a[done].data_ptr(), b[done].data_ptr(),
                                       gamma[done].data_ptr(), out[done].data_ptr()), "reconstruct")
        done += nf
    return out


def rebalance_(a: torch.Tensor, b: torch.Tensor, status: torch.Tensor) -> None:
    _need(a, C64, "a")
    _need(b, C64, "b")
    a3 = a.reshape(-1, a.shape[-2], a.shape[-1])
    b3 = b.reshape(-1, b.shape[-2], b.shape[-1])
    L.check(L.lib().tt_rebalance(L.stream_ptr(), a3.shape[0], a3.shape[1], b3.shape[1], a3.shape[2],
                                 a3.data_ptr(), b3.data_ptr(), status.data_ptr()), "rebalance")


def solve_gamma(phi: torch.Tensor, y: torch.Tensor, lam: float) -> torch.Tensor:
    _need(phi, torch.complex128, "phi")
    _need(y, torch.complex128, "y")
    Lr, R = phi.shape
    out = torch.empty(R, dtype=torch.complex128, device=phi.device)
    L.check(L.lib().tt_solve_gamma(L.stream_ptr(), Lr, R, phi.data_ptr() if Lr else None,
                                   y.data_ptr() if Lr else None, float(lam), out.data_ptr(), None),
            "solve_gamma")
    return out
