"""Device-resident online reconstruction loop (the B200 form of the
per-frame body of ``experiment.run_adaptive``, experiment.py:482-530, and of
``run_tracking``'s streaming pass, :284-296).

One ``tt_track_rows`` launch runs a whole block of frames for a batch of
independent slices: per frame [informative row draw from the current
k-space factor | static row table] -> gather y from the resident truth
k-space -> ridge gamma -> k-space factor update, with the state resident in
shared memory. The post-update factors of every frame are written to a
history buffer; ``reconstruct`` then turns them into image frames
X_t = A_t diag(gamma_t) B_t^T with the inverse column FFT and outer-product
kernels (the online reconstruction with post-update factors and the same
frame's gamma, experiment.py:525).

Semantics kept from the reference loop:
  * t starts at ``t0`` and advances by one per frame (tracker.py:411);
  * informative draws: k trials with replacement from row_scores of the
    pre-step k-space factor, forced lines count toward k, result sorted
    unique (sampler.py:146-162; experiment.py:499-505), Philox stream
    ``(key0, key1 + slice)`` shared across frames;
  * static masks keep the given (draw) order (experiment.py:166-167).
"""

from __future__ import annotations

from collections.abc import Sequence
from dataclasses import dataclass
import ctypes as C

import numpy as np
import torch

from .metrics import nmse_frames
from . import _lib as L
from . import _ops as K
from .tracker import Fixed, HessianBound

__all__ = ["StaticRows", "Informative", "AdaptiveSchedule", "OnlineEngine", "run_online", "OnlineResult", "warm_up", "RowShardedEngine",
           "InformativeEntries", "StaticEntries", "EntryEngine", "run_batch", "BatchResult", "LocalShardedEngine",
           "RowShardLoop", "history_norm_flags"]


@dataclass(frozen=True)
class StaticRows:
    """Pre-drawn row masks: ``rows[f, s, :cnt[f, s]]`` for frame f, slice s."""

    rows: np.ndarray  # (T, nslices, Smax) int
    counts: np.ndarray  # (T, nslices) int


@dataclass(frozen=True)
class Informative:
    """Subspace-driven row sampling (sampler.row_scores + draw_samples): ``k`` trials from the Philox
    stream (key0, key1 + slice) starting at word ``pos0``, with replacement (the deduplicated draws) or
    without (``replacement=False``: k distinct rows by sequential renormalised draws, sampler.py:163-169);
    the forced rows count toward k."""

    k: int
    forced: tuple = (0,)
    beta: float = 0.1
    key0: int = 0
    key1: int = 0
    replacement: bool = True
    pos0: int = 0


@dataclass(frozen=True)
class AdaptiveSchedule:
    """run_adaptive's acquisition schedule (experiment.py:462-497): variable-density rows
    (variable_density_rows, observation.py:300-323, with ``alpha`` and ``fraction``; DC first, draw order)
    for the frames before ``switch_frame``, then ``informative`` draws. ``switch_frame`` counts frames from
    the start of the sequence, warm-up frames included, as the reference's loop index does (None: right
    after the warm-up, the reference default). Both phases draw from one Philox stream per slice,
    (informative.key0, informative.key1 + slice) from word informative.pos0, as the reference's single
    ``rng`` does."""

    informative: Informative
    switch_frame: int | None = None
    alpha: float = -1.0
    fraction: float = 0.25

    def n_rows(self, nx: int) -> int:
        if not 0.0 < self.fraction <= 1.0:
            raise ValueError(f"fraction must be in (0, 1], got {self.fraction}")
        return int(np.ceil(self.fraction * nx))


class _Project:
    """Internal step marker: solve gamma only (mu = 0, the factors stay fixed)."""


def _step_params(step):
    if isinstance(step, _Project):
        return L.TT_STEP_FIXED, 0.0, 0.0, 0.0
    if isinstance(step, HessianBound):
        return L.TT_STEP_HESSIAN, 0.0, float(step.c_floor), float(step.c_cap)
    if isinstance(step, Fixed):
        return L.TT_STEP_FIXED, float(step.mu), 0.0, 0.0
    raise TypeError("step must be Fixed or HessianBound")


class OnlineEngine:
    """``norm_cap`` (StepConfig.norm_cap, tracker.py:406-408): when set, every frame reports whether its
    post-update factors exceed the cap in Frobenius norm (``out["norm"]``, StepReport.norm_exceeded)."""

    def __init__(self, nx, ny, rank, nslices=1, lam=0.1, step=Fixed(0.01), policy=None, cluster=0, t0=1,
                 norm_cap=None):
        if policy is None:
            raise ValueError("policy is required (StaticRows or Informative)")
        self.nx, self.ny, self.rank, self.nslices = int(nx), int(ny), int(rank), int(nslices)
        self.lam = float(lam)
        self.step = step
        self.policy = policy
        self.norm_cap = None if norm_cap is None else float(norm_cap)
        self.dev = L.device()
        if isinstance(policy, Informative):
            if not 1 <= policy.k <= nx:
                raise ValueError("informative k must be in [1, nx]")
            if policy.pos0 < 0:
                raise ValueError("Philox start position must be nonnegative")
            forced = np.unique(np.asarray(policy.forced, dtype=np.int64))
            if forced.size and (forced.min() < 0 or forced.max() >= nx):
                raise ValueError("forced index out of range")
            if forced.size > policy.k:
                raise ValueError("more forced indices than trials")
            self.max_rows = int(policy.k)
            self.forced = torch.from_numpy(forced.astype(np.int32)).to(self.dev)
            self.rows_tab = self.rows_cnt = None
        elif isinstance(policy, StaticRows):
            if isinstance(policy.rows, torch.Tensor) and policy.rows.is_cuda:  # device table (drawn on device)
                rows = policy.rows if policy.rows.dim() == 3 else policy.rows[:, None, :]
                cnt = torch.as_tensor(policy.counts).reshape(rows.shape[0], -1)
                if rows.shape[1] != nslices or tuple(cnt.shape) != tuple(rows.shape[:2]):
                    raise ValueError("static row table must be (T, nslices, Smax) with counts (T, nslices)")
                self.max_rows = int(rows.shape[2])
                self.rows_tab = rows.to(torch.int32).contiguous()
                self.rows_cnt = cnt.to(self.dev, torch.int32).contiguous()
            else:
                rows = np.asarray(policy.rows)
                if rows.ndim == 2:
                    rows = rows[:, None, :]
                cnt = np.asarray(policy.counts).reshape(rows.shape[0], -1)
                if rows.shape[1] != nslices or cnt.shape != rows.shape[:2]:
                    raise ValueError("static row table must be (T, nslices, Smax) with counts (T, nslices)")
                self.max_rows = int(rows.shape[2])
                self.rows_tab = torch.from_numpy(np.ascontiguousarray(rows, dtype=np.int32)).to(self.dev)
                self.rows_cnt = torch.from_numpy(np.ascontiguousarray(cnt, dtype=np.int32)).to(self.dev)
            self.forced = None
        else:
            raise TypeError("policy must be StaticRows or Informative")
        self.scr = K.RowsScratch(nslices, nx, ny, rank, self.max_rows, cluster)
        self.cluster = self.scr.cluster
        z = lambda *s: torch.zeros(*s, dtype=torch.complex64, device=self.dev)  # noqa: E731
        self.ah = z(nslices, nx, rank)
        self.bh = z(nslices, ny, rank)
        self.alpha_bar = torch.zeros(nslices, dtype=torch.float64, device=self.dev)
        self.philox_pos = torch.zeros(nslices, dtype=torch.int64, device=self.dev)
        if isinstance(policy, Informative) and policy.pos0:
            self.philox_pos.fill_(int(policy.pos0))
        self.status = torch.zeros(nslices, dtype=torch.int32, device=self.dev)
        self.t = int(t0)
        self.frame = 0

    # ------------------------------------------------------------------ state
    def set_image_factors(self, A, B):
        """Image-domain factors (nslices, N, R) -> resident k-space factors."""
        na, nb = self.nslices * self.nx * self.rank, self.nslices * self.ny * self.rank
        if isinstance(A, torch.Tensor) or isinstance(B, torch.Tensor):
            a = torch.as_tensor(A).to(self.dev, torch.complex64).reshape(self.nslices, self.nx, self.rank)
            b = torch.as_tensor(B).to(self.dev, torch.complex64).reshape(self.nslices, self.ny, self.rank)
            self.ah = K.fft_cols_(a.contiguous())
            self.bh = K.fft_cols_(b.contiguous())
            return
        # host arrays: one complex64 staging buffer, one upload, two in-place column FFTs
        a, b = np.asarray(A), np.asarray(B)
        if a.size != na or b.size != nb:
            raise ValueError("factor shapes do not match (nslices, nx, R) / (nslices, ny, R)")
        host = np.empty(na + nb, np.complex64)
        host[:na] = a.reshape(-1)
        host[na:] = b.reshape(-1)
        d = torch.from_numpy(host).to(self.dev)
        self.ah = K.fft_cols_(d[:na].view(self.nslices, self.nx, self.rank))
        self.bh = K.fft_cols_(d[na:].view(self.nslices, self.ny, self.rank))

    def reset(self, t0: int = 1) -> None:
        """Back to frame 0 at time ``t0``: step accumulator, Philox position and status cleared."""
        self.t = int(t0)
        self.frame = 0
        self.alpha_bar.zero_()
        self.philox_pos.fill_(int(self.policy.pos0) if isinstance(self.policy, Informative) else 0)
        self.status.zero_()

    def image_factors(self):
        return K.fft_cols(self.ah, inverse=True), K.fft_cols(self.bh, inverse=True)

    # ------------------------------------------------------------------ frames
    def make_outputs(self, frames: int, history: bool = True):
        d, ns, R = self.dev, self.nslices, self.rank
        out = dict(
            gamma=torch.empty(frames, ns, R, dtype=torch.complex64, device=d),
            cost=torch.empty(frames, ns, dtype=torch.float64, device=d),
            mu=torch.empty(frames, ns, dtype=torch.float64, device=d),
            alpha=torch.empty(frames, ns, dtype=torch.float64, device=d),
            rows=torch.empty(frames, ns, self.max_rows, dtype=torch.int32, device=d),
            cnt=torch.empty(frames, ns, dtype=torch.int32, device=d),
        )
        if history:
            out["ah"] = torch.empty(frames, ns, self.nx, R, dtype=torch.complex64, device=d)
            out["bh"] = torch.empty(frames, ns, self.ny, R, dtype=torch.complex64, device=d)
        if self.norm_cap is not None:
            out["norm"] = torch.empty(frames, ns, dtype=torch.int32, device=d)
        return out

    def args(self, kspace: torch.Tensor, frames: int, out: dict, ah_in=None, bh_in=None, ah_out=None,
             bh_out=None, frame0=None, t0=None) -> L.RowsArgs:
        """Build the C argument block. ``kspace`` is the truth, (T, nslices, nx, ny) complex64: a CUDA
        tensor, or a page-locked host tensor read in place (only the sampled rows cross the host link);
        frames [frame0, frame0+frames)."""
        host = not kspace.is_cuda
        if kspace.dtype != torch.complex64 or not kspace.is_contiguous() or (host and not kspace.is_pinned()):
            raise TypeError("kspace must be a contiguous complex64 CUDA or page-locked host tensor (T, nslices, nx, ny)")
        f0 = self.frame if frame0 is None else int(frame0)
        ks = kspace.reshape(kspace.shape[0], self.nslices, self.nx, self.ny)
        if f0 + frames > ks.shape[0]:
            raise ValueError("not enough truth frames")
        mode, mu, cf, cc = _step_params(self.step)
        a = L.RowsArgs()
        a.nslices, a.nx, a.ny, a.rank, a.frames = self.nslices, self.nx, self.ny, self.rank, int(frames)
        a.max_rows, a.cluster = self.max_rows, self.cluster
        a.t0 = self.t if t0 is None else int(t0)
        a.ah_in = (self.ah if ah_in is None else ah_in).data_ptr()
        a.bh_in = (self.bh if bh_in is None else bh_in).data_ptr()
        a.ah_out = (self.ah if ah_out is None else ah_out).data_ptr()
        a.bh_out = (self.bh if bh_out is None else bh_out).data_ptr()
        a.alpha_bar = self.alpha_bar.data_ptr()
        if isinstance(self.policy, Informative):
            a.policy = L.TT_POLICY_INFORMATIVE
            a.k_draws = int(self.policy.k)
            a.forced = self.forced.data_ptr() if self.forced.numel() else None
            a.nforced = int(self.forced.numel())
            a.beta = float(self.policy.beta)
            a.key0, a.key1 = int(self.policy.key0), int(self.policy.key1)
            a.philox_pos = self.philox_pos.data_ptr()
            a.draw_wor = 0 if self.policy.replacement else 1
        else:
            a.policy = L.TT_POLICY_STATIC
            rs = self.nslices * self.max_rows
            a.rows_tab = self.rows_tab.data_ptr() + 4 * f0 * rs
            a.rows_cnt = self.rows_cnt.data_ptr() + 4 * f0 * self.nslices
        a.y_mode = L.TT_Y_GATHER
        a.ysrc = ks[f0].data_ptr()
        a.y_host = 1 if host else 0
        a.y_frame_stride = self.nslices * self.nx * self.ny
        a.y_slice_stride = self.nx * self.ny
        a.lam, a.step_mode, a.mu, a.c_floor, a.c_cap = self.lam, mode, mu, cf, cc
        a.gamma_out = out["gamma"].data_ptr()
        a.cost_out = out["cost"].data_ptr()
        a.mu_out = out["mu"].data_ptr()
        a.alpha_out = out["alpha"].data_ptr()
        a.rows_out = out["rows"].data_ptr()
        a.cnt_out = out["cnt"].data_ptr()
        a.ah_hist = out["ah"].data_ptr() if "ah" in out else None
        a.bh_hist = out["bh"].data_ptr() if "bh" in out else None
        a.status = self.status.data_ptr()
        a.scratch = self.scr.buf.data_ptr()
        if self.norm_cap is not None and "norm" in out:
            a.norm_cap = self.norm_cap
            a.norm_out = out["norm"].data_ptr()
        return a

    def run(self, kspace: torch.Tensor, frames: int, history: bool = True, out: dict | None = None) -> dict:
        """Advance ``frames`` frames from the current frame index."""
        if out is None:
            out = self.make_outputs(frames, history)
        K.track_rows(self.args(kspace, frames, out))
        self.frame += frames
        self.t += frames
        return out

    def check_status(self):
        L.raise_status(int(self.status.max().item()), "online engine")

    def reconstruct(self, out: dict, into: torch.Tensor | None = None, in_place: bool = False,
                    domain: str = "image") -> torch.Tensor:
        """Frames (F, nslices, nx, ny) from the recorded k-space factor history. ``domain="image"``:
        inverse column FFT of each frame's factors, then the gamma-weighted outer product (``in_place``
        transforms the history itself, no copies). ``domain="kspace"``: the outer product of the k-space
        factors themselves, Ah diag(gamma) Bh^T = F_x X F_y^T — what run_adaptive records for k-space data
        (reconstruct_frame(...).kspace, experiment.py:242-245, :525), no FFT. ``into`` receives the frames."""
        F, ns = out["gamma"].shape[:2]
        if domain == "kspace":
            X = K.reconstruct(out["ah"].reshape(F * ns, self.nx, self.rank), out["bh"].reshape(F * ns, self.ny, self.rank),
                              out["gamma"].reshape(F * ns, self.rank), out=into)
            return X.reshape(F, ns, self.nx, self.ny)
        if domain != "image":
            raise ValueError("domain must be 'image' or 'kspace'")
        if in_place:
            A = K.fft_cols_(out["ah"], inverse=True).reshape(F * ns, self.nx, self.rank)
            B = K.fft_cols_(out["bh"], inverse=True).reshape(F * ns, self.ny, self.rank)
        else:
            A = K.fft_cols(out["ah"], inverse=True).reshape(F * ns, self.nx, self.rank)
            B = K.fft_cols(out["bh"], inverse=True).reshape(F * ns, self.ny, self.rank)
        X = K.reconstruct(A, B, out["gamma"].reshape(F * ns, self.rank), out=into)
        return X.reshape(F, ns, self.nx, self.ny)


class FrameRows(Sequence):
    """The sampled rows of a run as a read-only sequence: ``rows[f][s]`` is the int64 row array of
    frame f and slice s (the kernel's order: sorted and unique for draws with replacement, draw order
    without). Backed by the run's (frames, nslices, Smax) row tables and counts; the per-frame lists
    are built on access (a C3 run has 6400 of them), not inside the timed call."""

    def __init__(self, segments):
        self._seg = [(np.asarray(r), np.asarray(c)) for r, c in segments]  # (rows table, counts) per run segment
        self._off = np.cumsum([0] + [c.shape[0] for _, c in self._seg])

    def __len__(self):
        return int(self._off[-1])

    def __getitem__(self, f):
        if isinstance(f, slice):
            return [self[i] for i in range(*f.indices(len(self)))]
        f = int(f)
        if f < 0:
            f += len(self)
        if not 0 <= f < len(self):
            raise IndexError("frame index out of range")
        k = int(np.searchsorted(self._off, f, side="right")) - 1
        rows, cnt = self._seg[k]
        g = f - int(self._off[k])
        return [rows[g, s, :cnt[g, s]].astype(np.int64) for s in range(cnt.shape[1])]

    def total(self) -> int:
        """Number of sampled rows over all frames and slices."""
        return int(sum(int(c.sum()) for _, c in self._seg))


@dataclass
class OnlineResult:
    recon: np.ndarray     # (T, nslices, nx, ny) complex64 image frames
    gamma: np.ndarray     # (T, nslices, R)
    cost: np.ndarray      # (T, nslices)
    mu: np.ndarray
    rows: Sequence        # rows[f][s]: row array of frame f, slice s (FrameRows, or a list of lists)
    nmse: np.ndarray | None
    final_A: np.ndarray
    final_B: np.ndarray
    factor_history: object = None  # (T, nx, R) k-space Ah after each frame (slice 0), device; keep_history=True
    norm_exceeded: np.ndarray | None = None  # (T, nslices) bool, StepReport.norm_exceeded (norm_cap set)


def warm_up(engine: "OnlineEngine", kspace_warm: torch.Tensor, epochs: int) -> None:
    """experiment._warm_up (experiment.py:219-239) on device: the fully sampled
    leading frames tracked for `epochs` passes with `rebalance` between passes
    (core.py:138-166); t keeps growing. Leaves the engine's resident factors,
    t and alpha_bar as the streaming phase's starting state."""
    W = int(kspace_warm.shape[0])
    ns, nx = engine.nslices, engine.nx
    full = np.broadcast_to(np.arange(nx, dtype=np.int32), (W, ns, nx)).copy()
    weng = OnlineEngine(nx, engine.ny, engine.rank, ns, engine.lam, engine.step, StaticRows(full, np.full((W, ns), nx)),
                        0, engine.t)
    weng.ah, weng.bh, weng.alpha_bar = engine.ah, engine.bh, engine.alpha_bar
    st = torch.zeros(ns, dtype=torch.int32, device=engine.dev)
    for epoch in range(int(epochs)):
        if epoch > 0:
            K.rebalance_(weng.ah, weng.bh, st)
        weng.frame = 0
        weng.run(kspace_warm, W, history=False)
    L.raise_status(int(st.max().item()) & L.TT_ST_ZEROCOL, "warm-up rebalance")
    engine.ah, engine.bh, engine.alpha_bar, engine.t = weng.ah, weng.bh, weng.alpha_bar, weng.t


@dataclass(frozen=True)
class InformativeEntries:
    """adaptive_step(domain="entries") per frame (sampler.py:190-238; experiment.run_adaptive's
    entries mode): entry_scores of the k-space factors (sampler.py:95-112), ``k`` trials with
    replacement over the nx*ny entries (flat index i*ny + j) including the forced ones, EntryMask step."""
    k: int
    forced: tuple = ()
    beta: float = 0.1
    key0: int = 0
    key1: int = 0


@dataclass(frozen=True)
class StaticEntries:
    """Fixed entry lists per frame: ``entries`` (T, Smax) flat indices i*ny + j (-1 padded, any order
    without duplicates), ``counts`` (T,)."""
    entries: np.ndarray
    counts: np.ndarray


class EntryEngine:
    """Device-resident online loop for entry masks on k-space factors (the EntryMask /
    k-space interpolation path; EntryMask on (F_x A, F_y B) is the FourierMask iteration,
    test_mri.py:258-286). Per frame, on the device: [entry scores -> large-domain Philox draw] or the
    static list -> the generic index-list step reading y at the flat entries of the resident truth
    (tt_track_entries with a device-side count) -> per-frame outputs and factor history. The T-frame
    chain is captured once in a CUDA graph and replayed (no host round trip per frame). One slice."""

    def __init__(self, nx, ny, rank, lam=0.1, step=Fixed(0.01), policy=None, t0=1):
        self.nx, self.ny, self.rank = int(nx), int(ny), int(rank)
        self.lam, self.step, self.policy = float(lam), step, policy
        self.dev = L.device()
        n = self.nx * self.ny
        i32 = dict(dtype=torch.int32, device=self.dev)
        if isinstance(policy, InformativeEntries):
            if not 1 <= policy.k <= n:
                raise ValueError("informative k must be in [1, nx*ny]")
            forced = np.unique(np.asarray(policy.forced, dtype=np.int64))
            if forced.size and (forced.min() < 0 or forced.max() >= n):
                raise ValueError("forced index out of range")
            if forced.size > policy.k:
                raise ValueError("more forced indices than trials")
            self.cap = int(policy.k)
            self.forced = torch.from_numpy(forced.astype(np.int32)).to(self.dev)
            self.probs = torch.empty(n, dtype=torch.float64, device=self.dev)
            self.sws = torch.empty(int(L.lib().tt_entry_scores_ws_bytes(self.nx, self.ny)), dtype=torch.uint8,
                                   device=self.dev)
            self.dscr = torch.zeros(int(L.lib().tt_draw_scratch_bytes(n)), dtype=torch.uint8, device=self.dev)
            self.omega = torch.empty(self.cap, **i32)
            self.count = torch.zeros(1, **i32)
        elif isinstance(policy, StaticEntries):
            ent = np.asarray(policy.entries)
            cnt = np.asarray(policy.counts).reshape(-1)
            if ent.ndim != 2 or cnt.shape[0] != ent.shape[0]:
                raise ValueError("static entries must be (T, Smax) with counts (T,)")
            for f in range(ent.shape[0]):
                e = ent[f, :cnt[f]]
                if cnt[f] < 0 or cnt[f] > ent.shape[1] or (e.size and (e.min() < 0 or e.max() >= n)):
                    raise ValueError(f"frame {f}: entry index out of range")
                if np.unique(e).size != e.size:
                    raise ValueError(f"frame {f}: duplicate entries")  # observation.py:41-55
            self.cap = int(max(1, ent.shape[1]))
            self.tab = torch.from_numpy(np.ascontiguousarray(ent, dtype=np.int32)).to(self.dev)
            self.tab_cnt = torch.from_numpy(np.ascontiguousarray(cnt, dtype=np.int32)).to(self.dev)
        else:
            raise TypeError("policy must be InformativeEntries or StaticEntries")
        self.scr = torch.zeros(int(L.lib().tt_entries_scratch_bytes(self.nx, self.ny, self.rank, self.cap)),
                               dtype=torch.uint8, device=self.dev)  # zero-filled before first use (frame stamps)
        self.ah = torch.zeros(self.nx, self.rank, dtype=torch.complex64, device=self.dev)
        self.bh = torch.zeros(self.ny, self.rank, dtype=torch.complex64, device=self.dev)
        self.alpha_bar = torch.zeros(1, dtype=torch.float64, device=self.dev)
        self.pos = torch.zeros(1, dtype=torch.int64, device=self.dev)
        self.status = torch.zeros(1, **i32)
        self.t = int(t0)
        self._t0 = int(t0)
        self.frame = 0

    def set_image_factors(self, A, B):
        a = torch.as_tensor(np.asarray(A) if not isinstance(A, torch.Tensor) else A)
        b = torch.as_tensor(np.asarray(B) if not isinstance(B, torch.Tensor) else B)
        self.ah = K.fft_cols_(a.to(self.dev, torch.complex64).reshape(self.nx, self.rank).contiguous())
        self.bh = K.fft_cols_(b.to(self.dev, torch.complex64).reshape(self.ny, self.rank).contiguous())

    def rerun(self, A, B, gate=None, done=None) -> dict:
        """Restart from image factors (A, B) and replay the sequence captured by the last
        ``run(graph=True)`` over the same resident truth buffer (whose contents may have changed):
        state reset, frame 0 eagerly, the captured blocks replayed. ``gate(f)`` is called before the
        work that first reads truth frame f is enqueued (a pipelined caller makes the stream wait
        for that frame's upload); ``done(b)`` after the frames before b are enqueued. Returns that
        run's outputs."""
        if getattr(self, "_graph", None) is None:
            raise RuntimeError("rerun needs a previous run(graph=True)")
        gs, keep, ks, frames, out = self._graph
        self.set_image_factors(A, B)
        self.alpha_bar.zero_()
        self.pos.zero_()
        self.status.zero_()
        self.t, self.frame = self._t0, 0
        P = self._P
        P["ah0"], P["bh0"] = self.ah.data_ptr(), self.bh.data_ptr()
        if gate:
            gate(0)
        self._frame(ks.data_ptr(), 0, P, [])
        if done and gs[0][1] > 1:
            done(1)
        for g, a, b in gs:
            if gate:
                gate(b - 1)
            g.replay()
            if done:
                done(b)
        self.t += frames - 1
        self.ah = out["ah"][frames - 1, 0].clone()
        self.bh = out["bh"][frames - 1, 0].clone()
        self.frame = frames
        return out

    def make_outputs(self, frames: int) -> dict:
        d, R = self.dev, self.rank
        return dict(gamma=torch.empty(frames, 1, R, dtype=torch.complex64, device=d),
                    cost=torch.empty(frames, 1, dtype=torch.float64, device=d),
                    mu=torch.empty(frames, 1, dtype=torch.float64, device=d),
                    alpha=torch.empty(frames, 1, dtype=torch.float64, device=d),
                    rows=torch.full((frames, 1, self.cap), -1, dtype=torch.int32, device=d),
                    cnt=torch.empty(frames, 1, dtype=torch.int32, device=d),
                    ah=torch.empty(frames, 1, self.nx, R, dtype=torch.complex64, device=d),
                    bh=torch.empty(frames, 1, self.ny, R, dtype=torch.complex64, device=d))

    def _frame(self, ks_ptr: int, fo: int, P: dict, keep: list) -> None:
        """One frame. The step ping-pongs through the factor history (frame fo reads slot fo-1, writes
        slot fo), the draw writes its entry list and count straight into the outputs, and the step
        reads the drawn entries' values from the resident frame (no gather pass), so a frame is three
        C calls and no copies. ``P`` holds the output base pointers and strides."""
        lib, st = L.lib(), L.stream_ptr()
        nx, ny, R = self.nx, self.ny, self.rank
        ah_in = P["ah0"] if fo == 0 else P["ah"] + (fo - 1) * P["sah"]
        bh_in = P["bh0"] if fo == 0 else P["bh"] + (fo - 1) * P["sbh"]
        if isinstance(self.policy, InformativeEntries):
            pol = self.policy
            omega, count = P["rows"] + fo * P["srows"], P["cnt"] + 4 * fo
            L.check(lib.tt_entry_scores_ws(st, nx, ny, R, ah_in, bh_in, float(pol.beta), self.probs.data_ptr(),
                                           self.status.data_ptr(), self.sws.data_ptr()), "entry_scores")
            L.check(lib.tt_draw_with_replacement_large(
                st, nx * ny, self.probs.data_ptr(), int(pol.k), self.forced.data_ptr() if self.forced.numel() else None,
                int(self.forced.numel()), int(pol.key0), int(pol.key1), self.pos.data_ptr(), omega, count,
                self.dscr.data_ptr()), "draw (entries)")
        else:
            f = self.frame + fo
            omega, count = P["tab"] + f * P["stab"], P["tcnt"] + 4 * f
        mode, mu, cf, cc = _step_params(self.step)
        a = L.EntriesArgs()
        a.nx, a.ny, a.rank, a.nmeas, a.t = nx, ny, R, self.cap, self.t
        a.ah_in, a.ah_out = ah_in, P["ah"] + fo * P["sah"]
        a.bh_in, a.bh_out = bh_in, P["bh"] + fo * P["sbh"]
        a.alpha_bar = self.alpha_bar.data_ptr()
        a.omega, a.frame = omega, ks_ptr  # the step reads the drawn entries from the resident frame
        a.lam, a.step_mode, a.mu, a.c_floor, a.c_cap = self.lam, mode, mu, cf, cc
        a.gamma_out = P["gamma"] + fo * 8 * R
        a.cost_out, a.mu_out, a.alpha_out = P["cost"] + 8 * fo, P["mu"] + 8 * fo, P["alpha"] + 8 * fo
        a.status = self.status.data_ptr()
        a.scratch = self.scr.data_ptr()
        a.nmeas_dev = count
        keep.append(a)
        L.check(lib.tt_track_entries(st, C.byref(a)), "track_entries")
        self.t += 1

    def run(self, kspace: torch.Tensor, frames: int, out: dict | None = None, graph: bool = True,
            blocks: list | None = None) -> dict:
        """Advance ``frames`` frames; ``kspace`` (T, nx, ny) complex64 resident truth, frames from the
        current index. With ``graph`` the chain after the first frame is captured once and replayed;
        ``blocks`` (frame ranges [a, b) covering [1, frames)) captures one graph per range, so a
        pipelined caller can start each block once its truth has arrived (``rerun(..., gate=...)``)."""
        ks = kspace.reshape(kspace.shape[0], self.nx, self.ny)
        if ks.dtype != torch.complex64 or not ks.is_cuda or not ks.is_contiguous():
            raise TypeError("kspace must be a contiguous complex64 CUDA tensor (T, nx, ny)")
        if self.frame + frames > ks.shape[0]:
            raise ValueError("not enough truth frames")
        if out is None:
            out = self.make_outputs(frames)
        if frames == 0:
            return out
        P = dict(ah0=self.ah.data_ptr(), bh0=self.bh.data_ptr(), ah=out["ah"].data_ptr(), bh=out["bh"].data_ptr(),
                 sah=8 * self.nx * self.rank, sbh=8 * self.ny * self.rank, gamma=out["gamma"].data_ptr(),
                 cost=out["cost"].data_ptr(), mu=out["mu"].data_ptr(), alpha=out["alpha"].data_ptr(),
                 rows=out["rows"].data_ptr(), srows=4 * self.cap, cnt=out["cnt"].data_ptr())
        if isinstance(self.policy, StaticEntries):
            P.update(tab=self.tab.data_ptr(), stab=4 * self.tab.shape[1], tcnt=self.tab_cnt.data_ptr())
        keep: list = [self.ah, self.bh]
        f0 = self.frame
        kbase, kstride = ks.data_ptr(), 8 * self.nx * self.ny
        first = min(frames, 1)
        for fo in range(first):  # eager: one-time attribute setup happens outside any capture
            self._frame(kbase + (f0 + fo) * kstride, fo, P, keep)
        rest = frames - first
        if rest > 0 and graph:
            ranges = blocks if blocks else [(first, frames)]
            if ranges[0][0] != first or ranges[-1][1] != frames or any(
                    x[1] != y[0] for x, y in zip(ranges, ranges[1:])):
                raise ValueError("graph blocks must cover frames [1, frames) in order")
            t_save = self.t
            gs = []
            for (a, b) in ranges:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    for fo in range(a, b):
                        self._frame(kbase + (f0 + fo) * kstride, fo, P, keep)
                gs.append((g, a, b))
            self._graph = (gs, keep, ks, frames, out)  # the captured argument blocks must outlive the replay
            self._P = P
            for g, _, _ in gs:
                g.replay()
            assert self.t == t_save + rest
        else:
            for fo in range(first, frames):
                self._frame(kbase + (f0 + fo) * kstride, fo, P, keep)
            self._keep = keep
        if isinstance(self.policy, StaticEntries):
            out["cnt"][:, 0].copy_(self.tab_cnt[f0:f0 + frames])
            out["rows"][:, 0, :self.tab.shape[1]].copy_(self.tab[f0:f0 + frames])
        # the state is the last history slot (copied: the outputs may be reused by the caller)
        self.ah = out["ah"][frames - 1, 0].clone()
        self.bh = out["bh"][frames - 1, 0].clone()
        self.frame += frames
        return out

    def check_status(self):
        L.raise_status(int(self.status.max().item()), "entry engine")

    def reconstruct(self, out: dict) -> torch.Tensor:
        F = out["gamma"].shape[0]
        A = K.fft_cols(out["ah"], inverse=True).reshape(F, self.nx, self.rank)
        B = K.fft_cols(out["bh"], inverse=True).reshape(F, self.ny, self.rank)
        return K.reconstruct(A, B, out["gamma"].reshape(F, self.rank)).reshape(F, 1, self.nx, self.ny)

    def image_factors(self):
        return K.fft_cols(self.ah, inverse=True)[None], K.fft_cols(self.bh, inverse=True)[None]


def _host_source(kspace):
    """(T, nslices, nx, ny) complex64 CPU tensor over the caller's host buffer (no copy when it
    already is one; pinned buffers make the chunked uploads asynchronous)."""
    if isinstance(kspace, torch.Tensor):
        t = kspace
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(kspace), dtype=np.complex64))
    if t.dim() == 3:
        t = t[:, None]
    return t.to(torch.complex64).contiguous()


EDGE_BLOCK = 8  # frames in the first and last pipeline blocks
_STREAMS: dict = {}  # device index -> (upload, reconstruction, download) streams of run_online
_ENGINES: dict = {}  # run_online's informative-policy engines, reused across calls of the same configuration


def _take_engine(nx, ny, R, ns, lam, step, policy, cluster, t0, norm_cap=None):
    """An OnlineEngine for run_online: a cached one (reset) when the configuration repeats, else new.
    The engine is taken out of the cache for the duration of the call (concurrent calls never share)."""
    key = None
    if isinstance(policy, Informative):
        try:
            key = (torch.cuda.current_device(), nx, ny, R, ns, float(lam), repr(step), policy, int(cluster), norm_cap)
            hash(key)
        except TypeError:
            key = None
    eng = _ENGINES.pop(key, None) if key is not None else None
    if eng is None:
        eng = OnlineEngine(nx, ny, R, ns, lam, step, policy, cluster, t0, norm_cap)
    else:
        eng.reset(t0)
    return eng, key


def _give_engine(key, eng):
    if key is not None:
        while len(_ENGINES) >= 4:
            _ENGINES.pop(next(iter(_ENGINES)))
        _ENGINES[key] = eng


def _pipeline_streams(dev):
    key = dev.index if dev.index is not None else torch.cuda.current_device()
    if key not in _STREAMS:
        _STREAMS[key] = tuple(torch.cuda.Stream(dev) for _ in range(3))
    return _STREAMS[key]


def _blocks(f0, f1, C):
    """Frame blocks [a, b) covering [f0, f1): short first and last blocks (the pipeline's fill and
    drain are one upload / one download of a block), ``C`` frames in between."""
    n = f1 - f0
    if n <= 0:
        return []
    e = max(1, min(C, EDGE_BLOCK))
    if n <= 2 * e + C:
        sizes = [n] if n <= C else [e, n - e]
    else:
        mid = n - 2 * e
        sizes = [e] + [C] * (mid // C) + ([mid % C] if mid % C else []) + [e]
    out, f = [], f0
    for sz in sizes:
        out.append((f, f + sz))
        f += sz
    return out


BLOCK_BYTES = 128 << 20  # run_online's default pipeline block: ~128 MB of truth per upload
ZERO_COPY_BYTES = 512 << 20  # run_online(truth_transfer="auto"): page-locked truths this large are read in place


def run_online(kspace, A0, B0, lam, step, policy, clean=None, cluster=0, t0=1, warm_frames=0,
               warm_epochs=20, chunk=None, keep_history=False, norm_cap=None, recon_domain="image",
               truth_transfer="auto") -> OnlineResult:
    """Public end-to-end call (host in, host out): the online loop over the
    frames of ``kspace`` (T, [nslices,] nx, ny) from image-domain initial
    factors, returning reconstructions and per-frame reports. The analogue of
    ``experiment.run_adaptive`` for pre-noised truth: with ``warm_frames`` > 0
    the leading frames are fully sampled and tracked for ``warm_epochs`` passes
    first (experiment.py:219-239, default 5 x 20 in the reference config) and
    the results cover the streaming frames only; the policy applies to those. ``recon_domain``:
    "image" (default) returns image frames; "kspace" the k-space estimates Ah diag(gamma) Bh^T, which is what
    run_adaptive records for k-space data (no inverse FFTs); ``clean`` is an image sequence either way.
    ``truth_transfer``: "upload" copies the truth to the device block by block; "zero-copy" has the row
    kernels read a page-locked host truth in place, only each frame's sampled rows crossing the host link;
    "auto" takes zero-copy for page-locked truths of at least ZERO_COPY_BYTES (there the full upload
    dominates the call; below it the per-frame host-link latency costs more than the copy saves).
    ``policy`` is StaticRows, Informative, AdaptiveSchedule (variable-density rows until the switch
    frame, then informative draws, experiment.py:462-497) or an entries policy. ``norm_cap`` flags
    the frames whose post-update factors exceed it (``norm_exceeded``, tracker.py:406-408).

    Pipelined in blocks of ``chunk`` frames (default: ~BLOCK_BYTES of truth per block, at most 40
    frames — 40 frames at 256^2 x 1 slice, 4 at config 3's 64 slices, so that the uploads and the
    downloads overlap on the two copy engines): the truth uploads on one copy
    stream, tracking + reconstruction of block c on the compute stream once
    its upload landed, and the reconstructions download into pinned host
    memory on a second copy stream while later blocks compute. Results do not
    depend on ``chunk`` (the resident state and the Philox stream position
    carry across launches)."""
    on_dev = isinstance(kspace, torch.Tensor) and kspace.is_cuda
    src = kspace.to(torch.complex64) if on_dev else _host_source(kspace)
    if src.dim() == 3:
        src = src[:, None]
    T, ns, nx, ny = src.shape
    # a page-locked host truth is read in place by the row kernels (zero-copy: only each frame's sampled rows
    # cross the host link, as run_adaptive's StreamingProvider consults the truth at the sampled indices);
    # pageable inputs are uploaded block by block
    if truth_transfer not in ("auto", "upload", "zero-copy"):
        raise ValueError("truth_transfer must be 'auto', 'upload' or 'zero-copy'")
    rows_policy = not isinstance(policy, (InformativeEntries, StaticEntries))
    if truth_transfer == "zero-copy" and not (rows_policy and not on_dev and src.is_pinned()):
        raise ValueError("zero-copy needs a page-locked host truth and a row policy")
    zero_copy = rows_policy and not on_dev and src.is_pinned() and (
        truth_transfer == "zero-copy" or (truth_transfer == "auto" and src.numel() * 8 >= ZERO_COPY_BYTES))
    A0 = np.asarray(A0).reshape(ns, nx, -1)
    R = A0.shape[-1]
    if isinstance(policy, (InformativeEntries, StaticEntries)):
        return _run_online_entries(src, on_dev, A0, B0, lam, step, policy, clean, t0, warm_frames, norm_cap)
    sched = policy if isinstance(policy, AdaptiveSchedule) else None
    dev = L.device()
    comp = torch.cuda.current_stream(dev)
    s_in, s_rec, s_out = _pipeline_streams(dev)
    # the engine (cached for repeated informative configurations) and its initial factors first: their
    # small upload must not queue behind the truth uploads on the copy engine
    eng, ekey = _take_engine(nx, ny, R, ns, lam, step, sched.informative if sched else policy, cluster, t0, norm_cap)
    eng.set_image_factors(A0, np.asarray(B0).reshape(ns, ny, R))
    kd = src.contiguous() if (on_dev or zero_copy) else torch.empty(T, ns, nx, ny, dtype=torch.complex64, device=dev)
    W = int(warm_frames)
    if W < 0 or W > T:
        raise ValueError("warm_frames must be in [0, T]")
    # AdaptiveSchedule: the variable-density frames [W, W + nvd) first (experiment.py:484-497)
    nvd = 0
    if sched is not None:
        sw = W if sched.switch_frame is None else int(sched.switch_frame)
        nvd = min(max(sw - W, 0), T - W)
    if chunk is None:
        chunk = min(40, max(1, BLOCK_BYTES // max(1, ns * nx * ny * 8)))
    C = max(1, int(chunk))
    # upload blocks: the warm-up frames as one block, then the streaming frames in blocks of C (a block
    # never straddles the switch frame)
    bounds = ([(0, W)] if W else []) + _blocks(W, W + nvd, C) + _blocks(W + nvd, T, C)
    s_in.wait_stream(comp)
    ev_in = []
    with torch.cuda.stream(s_in):
        for f0, f1 in bounds:
            if not (on_dev or zero_copy):
                kd[f0:f1].copy_(src[f0:f1], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(s_in)
            ev_in.append(ev)
    blocks = list(zip(bounds, ev_in))
    if W:
        comp.wait_event(blocks[0][1])
        # the warm-up revisits its full frames warm_epochs times: resident on the device even in zero-copy mode
        warm_up(eng, kd[:W].to(dev, non_blocking=True) if zero_copy else kd[:W], warm_epochs)
        blocks = blocks[1:]
        if clean is not None:
            clean = np.asarray(clean).reshape(T, ns, nx, ny)[W:]
    Ts = T - W
    ks_stream = kd[W:]
    # segments of the streaming frames: (engine, outputs, first frame); the VD engine shares the state
    segs = []
    if nvd:
        inf = sched.informative
        nr = sched.n_rows(nx)
        tab = K.vd_rows_batch(nvd, ns, nx, float(sched.alpha), nr, (int(inf.key0), int(inf.key1)), eng.philox_pos)
        veng = OnlineEngine(nx, ny, R, ns, lam, step,
                            StaticRows(tab, torch.full((nvd, ns), nr, dtype=torch.int32, device=dev)), cluster,
                            eng.t, norm_cap)
        veng.ah, veng.bh, veng.alpha_bar, veng.status = eng.ah, eng.bh, eng.alpha_bar, eng.status
        eng.philox_pos += nvd * (nr - 1)  # the informative draws continue the stream
        segs.append((veng, veng.make_outputs(nvd), 0))
    if Ts - nvd > 0 or not segs:
        segs.append((eng, eng.make_outputs(Ts - nvd), nvd))
    recon = Xd = None
    hist = torch.empty(Ts, nx, R, dtype=torch.complex64, device=dev) if keep_history else None
    # tracking blocks run back to back on the compute stream; each block's reconstruction runs on its
    # own stream once the block's tracking is done, and its download follows on the copy stream
    for (f0, f1), ev in blocks:
        a, b = f0 - W, f1 - W
        e, out, base = segs[-1] if a >= segs[-1][2] else segs[0]
        if e is eng and nvd and e.frame < nvd:  # hand over from the VD phase: same state, next frame, t
            e.frame, e.t = nvd, segs[0][0].t
        comp.wait_event(ev)
        part = {k: v[a - base:b - base] for k, v in out.items()}
        e.run(ks_stream, b - a, out=part)
        if recon is None:  # the result buffers are set up while the first block tracks
            recon = torch.empty(Ts, ns, nx, ny, dtype=torch.complex64, pin_memory=True)
            Xd = torch.empty(Ts, ns, nx, ny, dtype=torch.complex64, device=dev)
            s_rec.wait_stream(comp)
            s_out.wait_stream(comp)
        tracked = torch.cuda.Event()
        tracked.record(comp)
        s_rec.wait_event(tracked)
        with torch.cuda.stream(s_rec):
            if keep_history:
                hist[a:b].copy_(part["ah"][:, 0])
            e.reconstruct(part, into=Xd[a:b], in_place=True, domain=recon_domain)  # history not needed after
            done = torch.cuda.Event()
            done.record(s_rec)
        s_out.wait_event(done)
        with torch.cuda.stream(s_out):
            recon[a:b].copy_(Xd[a:b], non_blocking=True)
    if recon is None:  # no streaming frames
        recon = torch.empty(Ts, ns, nx, ny, dtype=torch.complex64, pin_memory=True)
        Xd = torch.empty(Ts, ns, nx, ny, dtype=torch.complex64, device=dev)
    comp.wait_stream(s_rec)
    # small results, final factors and the status word: asynchronous copies into pinned memory, one sync
    pinned = lambda t: torch.empty(t.shape, dtype=t.dtype, pin_memory=True)  # noqa: E731
    keys = ("gamma", "cost", "mu", "cnt", "rows") + (("norm",) if norm_cap is not None else ())
    small = []
    for _, out, _ in segs:
        sm = {k: pinned(out[k]) for k in keys}
        for k, v in sm.items():
            v.copy_(out[k], non_blocking=True)
        small.append(sm)
    Ad, Bd = eng.image_factors()
    A, B, st = pinned(Ad), pinned(Bd), pinned(eng.status)
    A.copy_(Ad, non_blocking=True)
    B.copy_(Bd, non_blocking=True)
    st.copy_(eng.status, non_blocking=True)
    nm = None
    if clean is not None:
        cl = torch.as_tensor(np.asarray(clean, dtype=np.complex64)).to(dev).reshape(Ts * ns, nx, ny)
        if recon_domain == "kspace":  # F_x X F_y^T of the clean images (unitary: the same NMSE)
            cl = K.fft2_(cl.contiguous())
        nm = nmse_frames(cl.reshape(Ts * ns, nx * ny).contiguous(),
                         Xd.reshape(Ts * ns, nx * ny)).reshape(Ts, ns).cpu().numpy()  # metrics.py:53-62
    comp.synchronize()
    s_out.synchronize()
    L.raise_status(int(st.max().item()), "online engine")
    _give_engine(ekey, eng)
    cat = lambda k: np.concatenate([sm[k].numpy() for sm in small], axis=0)  # noqa: E731
    rows = FrameRows([(sm["rows"].numpy(), sm["cnt"].numpy()) for sm in small])
    return OnlineResult(recon=recon.numpy(), gamma=cat("gamma"), cost=cat("cost"), mu=cat("mu"), rows=rows, nmse=nm,
                        final_A=A.numpy(), final_B=B.numpy(), factor_history=hist,
                        norm_exceeded=cat("norm").astype(bool) if norm_cap is not None else None)


class LocalShardedEngine:
    """The row-sharded step (BASELINE config 4) on one GPU: ``ranks`` thread-block clusters
    each own a block of k-space rows of Ah (as a GPU of the multi-GPU sharding would); per frame one
    phase-1 launch holds all ranks (partials of W, GA, ||Y||^2, ||Ah||^2 into one payload slot per
    rank), a device kernel sums the slots in fixed order (the all-reduce of the multi-GPU path), and
    one phase-2 launch solves redundantly and updates every rank's rows and the replicated Bh. Uses
    ranks x 16 SMs instead of 16 for a single large slice; static row masks, one slice. The T-frame
    chain of 3 launches per frame is replayed as one CUDA graph.

    The replicated Bh is double-buffered across phase 2 (read one, rank 0 writes the other): when
    the ranks' clusters do not fit the GPU at once they run in waves, and a later wave must still
    read the frame's pre-update Bh.

    ``fused`` (default): one cooperative cluster launch runs every frame of a ``run`` call, both phases
    per frame, the payload summed inside the kernel between two inter-cluster barriers (same fixed
    order as ``tt_rows_shard_reduce``); the factors and the frame's row table stay in shared memory
    across the phases and frames, and the replicated Bh's GB Gram is split across the ranks (rank q
    takes every world-th column) and summed with the payload, so GB rounds differently from the
    3-launch path (~1e-16 relative). It needs all ranks' clusters resident at once (up to 7 clusters of
    16 CTAs on a B200); when they do not fit, ``run`` falls back to the 3-launch frames."""

    def __init__(self, nx, ny, rank, lam, step, rows, counts, ranks, cluster=0, t0=1, fused=True):
        self.nx, self.ny, self.R = int(nx), int(ny), int(rank)
        self.ranks = int(ranks)
        if self.ranks < 1 or self.ranks > self.nx:
            raise ValueError("ranks must be in [1, nx]")
        self.lam, self.step = float(lam), step
        self.dev = L.device()
        rows = np.asarray(rows).reshape(np.asarray(rows).shape[0], -1)
        self.max_rows = int(rows.shape[1])
        self.rows_tab = torch.from_numpy(np.ascontiguousarray(rows, dtype=np.int32)).to(self.dev)
        self.rows_cnt = torch.from_numpy(np.ascontiguousarray(np.asarray(counts).reshape(-1), dtype=np.int32)).to(self.dev)
        self.scr = K.RowsScratch(self.ranks, self.nx, self.ny, self.R, self.max_rows, cluster)  # one scratch per rank
        self.cluster = self.scr.cluster
        self.ah = torch.zeros(self.nx, self.R, dtype=torch.complex64, device=self.dev)
        self._bhs = [torch.zeros(self.ny, self.R, dtype=torch.complex64, device=self.dev) for _ in range(2)]
        self._cur = 0  # index of the buffer holding the current Bh
        self.xg_len = int(L.lib().tt_rows_shard_xg_len(self.R))
        self.fused = bool(fused)
        sets = 2 if self.fused else 1  # the fused launch double-buffers the payload by frame parity
        self.xw = torch.zeros(sets * self.ranks, self.ny, self.R, dtype=torch.complex128, device=self.dev)
        # fused slots also carry the ranks' GB partials: [GA packed][||Y||^2, ||Ah||^2][GB packed]
        slot = 2 * self.xg_len - 2 if self.fused else self.xg_len
        self.xg = torch.zeros(sets * self.ranks, slot, dtype=torch.float64, device=self.dev)
        self.grid_sync = torch.zeros(1, dtype=torch.int32, device=self.dev)
        self.alpha_bar = torch.zeros(1, dtype=torch.float64, device=self.dev)
        self.status = torch.zeros(1, dtype=torch.int32, device=self.dev)
        self.t = int(t0)
        self.frame = 0

    def set_image_factors(self, A, B):
        a = torch.as_tensor(np.asarray(A) if not isinstance(A, torch.Tensor) else A).to(self.dev, torch.complex64)
        b = torch.as_tensor(np.asarray(B) if not isinstance(B, torch.Tensor) else B).to(self.dev, torch.complex64)
        self.ah = K.fft_cols_(a.reshape(self.nx, self.R).contiguous())
        self._bhs = [K.fft_cols_(b.reshape(self.ny, self.R).contiguous()), torch.empty(self.ny, self.R,
                                                                                      dtype=torch.complex64,
                                                                                      device=self.dev)]
        self._cur = 0

    @property
    def bh(self) -> torch.Tensor:
        return self._bhs[self._cur]

    def image_factors(self):
        return K.fft_cols(self.ah, inverse=True), K.fft_cols(self.bh, inverse=True)

    def make_outputs(self, frames):
        d = self.dev
        return dict(gamma=torch.empty(frames, self.R, dtype=torch.complex64, device=d),
                    cost=torch.empty(frames, dtype=torch.float64, device=d),
                    mu=torch.empty(frames, dtype=torch.float64, device=d),
                    ah=torch.empty(frames, self.nx, self.R, dtype=torch.complex64, device=d),
                    bh=torch.empty(frames, self.ny, self.R, dtype=torch.complex64, device=d))

    def _args(self, kspace, f, out, fo, phase, bh_cur, bh_nxt, frames=1):
        mode, mu, cf, cc = _step_params(self.step)
        a = L.RowsArgs()
        a.nslices, a.nx, a.ny, a.rank, a.frames = 1, self.nx, self.ny, self.R, int(frames)
        a.max_rows, a.cluster, a.t0 = self.max_rows, self.cluster, self.t
        a.ah_in = a.ah_out = self.ah.data_ptr()
        a.bh_in = bh_cur.data_ptr()
        a.bh_out = (bh_nxt if phase == 2 else bh_cur).data_ptr()
        a.alpha_bar = self.alpha_bar.data_ptr()
        a.policy = L.TT_POLICY_STATIC
        a.rows_tab = self.rows_tab.data_ptr() + 4 * f * self.max_rows
        a.rows_cnt = self.rows_cnt.data_ptr() + 4 * f
        a.y_mode = L.TT_Y_GATHER
        a.ysrc = kspace[f].data_ptr()
        a.y_frame_stride, a.y_slice_stride = self.nx * self.ny, self.nx * self.ny
        a.lam, a.step_mode, a.mu, a.c_floor, a.c_cap = self.lam, mode, mu, cf, cc
        if phase in (0, 2) and out is not None:  # phase 2 of a frame, or a fused launch (phase 0 here)
            a.gamma_out = out["gamma"][fo].data_ptr()
            a.cost_out = out["cost"][fo:].data_ptr()
            a.mu_out = out["mu"][fo:].data_ptr()
            a.ah_hist = out["ah"][fo].data_ptr()
            a.bh_hist = out["bh"][fo].data_ptr()
        a.status = self.status.data_ptr()
        a.scratch = self.scr.buf.data_ptr()
        a.shard_rank, a.shard_world, a.shard_phase, a.shard_local = 0, self.ranks, phase, 1
        a.xw, a.xg = self.xw.data_ptr(), self.xg.data_ptr()
        if phase == 0:  # fused launch: both phases of every frame
            a.shard_phase, a.shard_fused, a.grid_sync = 1, 1, self.grid_sync.data_ptr()
        return a

    def _run_fused(self, kspace, frames, out):
        cur, nxt = self._bhs[self._cur], self._bhs[1 - self._cur]
        a = self._args(kspace, self.frame, out, 0, 0, cur, nxt, frames=frames)
        self.grid_sync.zero_()
        K.track_rows(a)  # Bh in place: every rank loads it at the start, rank 0 writes it back at the end
        self.t += frames

    def _frame(self, kspace, f, out, fo, keep):
        cur, nxt = self._bhs[self._cur], self._bhs[1 - self._cur]
        a1 = self._args(kspace, f, None, fo, 1, cur, nxt)
        a2 = self._args(kspace, f, out, fo, 2, cur, nxt)
        keep += [a1, a2]
        K.track_rows(a1)
        L.check(L.lib().tt_rows_shard_reduce(L.stream_ptr(), self.ranks, self.ny, self.R, self.xw.data_ptr(),
                                             self.xg.data_ptr()), "shard_reduce")
        K.track_rows(a2)
        self.t += 1
        self._cur = 1 - self._cur

    def run(self, kspace, frames, out=None, graph=True):
        """kspace: (T, nx, ny) complex64 CUDA; frames from the current index."""
        if out is None:
            out = self.make_outputs(frames)
        if self.fused and frames > 0:
            try:
                self._run_fused(kspace, frames, out)
                self.frame += frames
                return out
            except RuntimeError as e:
                if "cooperative" not in str(e).lower():
                    raise
                self.fused = False  # the ranks' clusters do not fit at once: 3-launch frames
        keep: list = []
        f0 = self.frame
        first = min(frames, 1)
        for fo in range(first):  # eager first frame: one-time launch attributes outside any capture
            self._frame(kspace, f0 + fo, out, fo, keep)
        if frames > first and graph:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for fo in range(first, frames):
                    self._frame(kspace, f0 + fo, out, fo, keep)
            self._graph = (g, keep)
            g.replay()
        else:
            for fo in range(first, frames):
                self._frame(kspace, f0 + fo, out, fo, keep)
        self.frame += frames
        return out

    def check_status(self):
        L.raise_status(int(self.status.max().item()), "local sharded engine")


_ENTRY_PLANS: dict = {}  # (shape, policy, length) -> (EntryEngine with a captured graph, resident truth)


def history_norm_flags(out: dict, norm_cap: float) -> torch.Tensor:
    """StepReport.norm_exceeded (tracker.py:406-408) per frame of an engine's outputs from its factor history:
    the frame updated (count > 0) and a post-update factor's Frobenius norm exceeds ``norm_cap`` (the DFT is
    unitary, so the k-space history has the image factors' norms). (F, nslices) bool on the device."""
    ah, bh = out["ah"], out["bh"]
    F = ah.shape[0] * ah.shape[1]
    na = torch.empty(F, dtype=torch.float64, device=ah.device)
    nb = torch.empty(F, dtype=torch.float64, device=ah.device)
    L.check(L.lib().tt_factor_norms2(L.stream_ptr(), F, ah.shape[-2] * ah.shape[-1], ah.data_ptr(), na.data_ptr()),
            "factor norms")
    L.check(L.lib().tt_factor_norms2(L.stream_ptr(), F, bh.shape[-2] * bh.shape[-1], bh.data_ptr(), nb.data_ptr()),
            "factor norms")
    cap2 = float(norm_cap) ** 2
    over = (na > cap2) | (nb > cap2)
    return (over.reshape(ah.shape[:2]) & (out["cnt"] > 0))


def _run_online_entries(src, on_dev, A0, B0, lam, step, policy, clean, t0, warm_frames,
                        norm_cap=None) -> OnlineResult:
    """run_online for the entry policies (one slice): upload, the graph-replayed frame chain,
    reconstruction, download. The entry lists are reported in ``rows`` (flat indices i*ny + j)."""
    T, ns, nx, ny = src.shape
    if ns != 1:
        raise ValueError("entry sampling runs one slice per engine")
    if warm_frames:
        raise ValueError("warm-up applies to the row-mask engine")
    R = A0.shape[-1]
    # repeated calls with the same shapes, policy and length reuse the engine, its resident truth buffer
    # and its captured frame graphs (like an FFT plan). The call is pipelined in blocks of frames:
    # uploads on a copy stream, each block's graph replayed once its truth landed, the block's
    # images reconstructed on a second stream and downloaded into pinned memory on a third.
    key = (nx, ny, R, T, float(lam), repr(step), repr(policy), int(t0), torch.cuda.current_device())
    ub = _blocks(0, T, 40)  # upload / reconstruction / download blocks
    dev = L.device()
    pinned = lambda shape, dt: torch.empty(shape, dtype=dt, pin_memory=True)  # noqa: E731
    X = torch.empty(T, 1, nx, ny, dtype=torch.complex64, device=dev)
    Xh = pinned((T, 1, nx, ny), torch.complex64)
    hit = _ENTRY_PLANS.get(key)
    comp = torch.cuda.current_stream()
    if hit is not None:
        eng, kd, streams = hit
        s_in, s_rec, s_out = streams
        ev_up = [torch.cuda.Event() for _ in ub]
        with torch.cuda.stream(s_in):
            s_in.wait_stream(comp)  # the previous call's replays have read the buffer
            for k, (a, b) in enumerate(ub):
                kd[a:b].copy_(src.reshape(T, nx, ny)[a:b], non_blocking=True)
                ev_up[k].record(s_in)
        blk_of = lambda f: next(k for k, (a, b) in enumerate(ub) if a <= f < b)  # noqa: E731
        waited = set()
        pending = list(range(len(ub)))

        def gate(f):
            k = blk_of(f)
            for j in range(k + 1):
                if j not in waited:
                    comp.wait_event(ev_up[j])
                    waited.add(j)

        outs = {}

        def done(fend):  # frames [0, fend) are enqueued: reconstruct and download finished blocks
            ev = torch.cuda.Event()
            ev.record(comp)
            while pending and ub[pending[0]][1] <= fend:
                k = pending.pop(0)
                a, b = ub[k]
                s_rec.wait_event(ev)
                with torch.cuda.stream(s_rec):
                    o = outs["out"]
                    A = K.fft_cols(o["ah"][a:b], inverse=True).reshape(b - a, nx, R)
                    Bm = K.fft_cols(o["bh"][a:b], inverse=True).reshape(b - a, ny, R)
                    X[a:b] = K.reconstruct(A, Bm, o["gamma"][a:b].reshape(b - a, R)).reshape(b - a, 1, nx, ny)
                    er = torch.cuda.Event()
                    er.record(s_rec)
                s_out.wait_event(er)
                with torch.cuda.stream(s_out):
                    Xh[a:b].copy_(X[a:b], non_blocking=True)

        outs["out"] = eng._graph[4]
        out = eng.rerun(A0.reshape(nx, R), np.asarray(B0).reshape(ny, R), gate=gate, done=done)
        comp.wait_stream(s_out)
        comp.wait_stream(s_rec)
    else:
        eng = EntryEngine(nx, ny, R, lam, step, policy, t0)
        eng.set_image_factors(A0.reshape(nx, R), np.asarray(B0).reshape(ny, R))
        kd = torch.empty(T, nx, ny, dtype=torch.complex64, device=eng.dev)
        kd.copy_(src.reshape(T, nx, ny), non_blocking=True)
        gblocks = [(max(a, 1), b) for a, b in ub if b > 1]
        out = eng.run(kd, T, graph=T > 1, blocks=gblocks if T > 1 else None)
        X.copy_(eng.reconstruct(out))
        Xh.copy_(X, non_blocking=True)
        if T > 1:
            if len(_ENTRY_PLANS) >= 2:
                _ENTRY_PLANS.pop(next(iter(_ENTRY_PLANS)))
            _ENTRY_PLANS[key] = (eng, kd, (torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()))
    nm = None
    if clean is not None:
        cl = torch.as_tensor(np.asarray(clean, dtype=np.complex64)).to(eng.dev).reshape(T, nx * ny)
        nm = nmse_frames(cl, X.reshape(T, nx * ny)).reshape(T, 1).cpu().numpy()  # metrics.py:53-62
    # the small results: asynchronous copies into pinned memory, one synchronisation
    Ad, Bd = eng.image_factors()
    small = (("gamma", out["gamma"]), ("cost", out["cost"]), ("mu", out["mu"]), ("cnt", out["cnt"]),
             ("rows", out["rows"]), ("A", Ad), ("B", Bd), ("st", eng.status))
    if norm_cap is not None:
        small = small + (("norm", history_norm_flags(out, norm_cap).to(torch.int32)),)
    host = {k: pinned(tuple(v.shape), v.dtype) for k, v in small}
    for k, v in small:
        host[k].copy_(v, non_blocking=True)
    comp.synchronize()
    host["recon"] = Xh
    L.raise_status(int(host["st"].max().item()), "entry engine")
    cnt = host["cnt"].numpy()
    rows_np = host["rows"].numpy()
    # entry lists as measured: sorted for informative draws (np.union1d), the given order for static ones
    rows = FrameRows([(rows_np, cnt)])
    return OnlineResult(recon=host["recon"].numpy(), gamma=host["gamma"].numpy(), cost=host["cost"].numpy(),
                        mu=host["mu"].numpy(), rows=rows, nmse=nm, final_A=host["A"].numpy(),
                        final_B=host["B"].numpy(),
                        norm_exceeded=host["norm"].numpy().astype(bool) if norm_cap is not None else None)


@dataclass
class BatchResult:
    recon: np.ndarray     # (T, nx, ny) images at the final subspace
    gamma: np.ndarray     # (T, R) final gammas (re-projected when epochs > 1)
    step_gamma: np.ndarray  # (epochs * T, R) per-step gammas, processing order
    step_cost: np.ndarray
    step_mu: np.ndarray
    orders: list          # frame order per epoch
    final_A: np.ndarray
    final_B: np.ndarray
    t: int
    step_norm_exceeded: np.ndarray | None = None  # (epochs * T,) bool, processing order (norm_cap set)


def run_batch(kspace, A0, B0, lam, step, rows, counts, epochs=1, rng=None, reshuffle=False,
              rebalance_epochs=True, t0=1, cluster=0, norm_cap=None) -> BatchResult:
    """Multi-epoch batch mode on the device (tracker.run tracker.py:456-500,
    experiment.run_tracking experiment.py:284-313): the frames' row-mask data
    (``rows`` (T, Smax) table, ``counts`` (T,)) is revisited for ``epochs`` passes of the rows
    kernel, the factors rebalanced between passes, the order re-drawn with ``rng.permutation`` when
    ``reshuffle`` (the caller's generator, consumed as the reference does), t growing globally.
    With epochs > 1 every frame's gamma is then re-solved against the final subspace (a pass of the
    same kernel with a zero step) and the images synthesised from it. One slice. ``norm_cap`` flags every
    step whose post-update factors exceed it (StepReport.norm_exceeded, tracker.py:406-408)."""
    if epochs < 1:
        raise ValueError("epochs must be at least 1")
    if reshuffle and epochs > 1 and rng is None:
        raise ValueError("rng is required for reshuffling")
    src = kspace.to(torch.complex64) if isinstance(kspace, torch.Tensor) else _host_source(kspace)
    if src.dim() == 4:
        src = src[:, 0]
    T, nx, ny = src.shape
    R = np.asarray(A0).reshape(nx, -1).shape[-1]
    tab = np.asarray(rows).reshape(T, 1, -1)
    cnt = np.asarray(counts).reshape(T, 1)
    dev = L.device()
    kd = src.to(dev).contiguous().reshape(T, 1, nx, ny)
    base = OnlineEngine(nx, ny, R, 1, lam, step, StaticRows(tab, cnt), cluster, t0)
    base.set_image_factors(np.asarray(A0).reshape(1, nx, R), np.asarray(B0).reshape(1, ny, R))
    st = torch.zeros(1, dtype=torch.int32, device=dev)
    g_steps, c_steps, m_steps, n_steps, orders = [], [], [], [], []
    ah, bh, ab, t = base.ah, base.bh, base.alpha_bar, base.t
    for epoch in range(epochs):
        if rebalance_epochs and epoch > 0:
            K.rebalance_(ah, bh, st)
        order = np.arange(T)
        if reshuffle and epoch > 0:
            order = np.asarray(rng.permutation(T))
        orders.append(order)
        eng = OnlineEngine(nx, ny, R, 1, lam, step, StaticRows(tab[order], cnt[order]), base.cluster, t, norm_cap)
        eng.ah, eng.bh, eng.alpha_bar = ah, bh, ab
        sel = torch.from_numpy(order.astype(np.int64)).to(dev)
        out = eng.run(kd.index_select(0, sel).contiguous(), T, history=False)
        g_steps.append(out["gamma"][:, 0])
        c_steps.append(out["cost"][:, 0])
        m_steps.append(out["mu"][:, 0])
        if norm_cap is not None:
            n_steps.append(out["norm"][:, 0])
        ah, bh, ab, t = eng.ah, eng.bh, eng.alpha_bar, eng.t
    L.raise_status(int(st.max().item()) & L.TT_ST_ZEROCOL, "batch rebalance")
    if epochs > 1:  # re-projection onto the final subspace
        proj = OnlineEngine(nx, ny, R, 1, lam, _Project(), StaticRows(tab, cnt), base.cluster, t)
        proj.ah, proj.bh = ah.clone(), bh.clone()
        gam = proj.run(kd, T, history=False)["gamma"][:, 0]
    else:
        gam = g_steps[0]
    A = K.fft_cols(ah, inverse=True).reshape(nx, R)
    B = K.fft_cols(bh, inverse=True).reshape(ny, R)
    X = K.reconstruct(A[None].expand(T, nx, R).contiguous(), B[None].expand(T, ny, R).contiguous(), gam.contiguous())
    # asynchronous downloads into pinned memory, one synchronisation
    dl = {"recon": X, "gamma": gam, "sg": torch.cat(g_steps), "sc": torch.cat(c_steps), "sm": torch.cat(m_steps),
          "A": A, "B": B}
    if norm_cap is not None:
        dl["sn"] = torch.cat(n_steps)
    host = {k: torch.empty(v.shape, dtype=v.dtype, pin_memory=True) for k, v in dl.items()}
    for k, v in dl.items():
        host[k].copy_(v, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    h = {k: v.numpy() for k, v in host.items()}
    return BatchResult(recon=h["recon"], gamma=h["gamma"], step_gamma=h["sg"], step_cost=h["sc"], step_mu=h["sm"],
                       orders=orders, final_A=h["A"], final_B=h["B"], t=t,
                       step_norm_exceeded=h["sn"].astype(bool) if norm_cap is not None else None)


class RowShardLoop:
    """Host orchestration of one rank of the row-sharded online loop (BASELINE config 4),
    independent of where the phases run. Per frame:

    1. informative draws only: the rank's row energies |Ah_ir|^2 into a zeroed full (nx, R) fp64 matrix,
       summed over the ranks (``allreduce``; x + 0 = x, so every rank gets the exact full matrix) and
       turned into raw row scores (``_scores``) — every rank then draws the same rows;
    2. phase 1 (``_phase1``): the rank's partials W, GA, ||Y||^2, ||Ah||^2 into ``payload`` (float64, the
       kernel layout of ``sharding.pack_payload``);
    3. ONE sum all-reduce of ``payload`` across the ranks;
    4. phase 2 (``_phase2``): redundant fp64 solve, update of the owned rows and the replicated Bh.

    ``allreduce(tensor)`` sums in place over the ranks (NCCL over NVLink in ``RowShardedEngine``; gloo
    in the CPU tests). Subclasses provide the buffers and the phases."""

    informative = False

    def _frame(self, kspace, f, out, fo):
        if self.informative:
            self._energy()
            self.allreduce(self.energy)
            self._scores()
        self._phase1(kspace, f)
        self.allreduce(self.payload)  # one sum over the ranks per frame
        self._phase2(kspace, f, out, fo)
        self.t += 1
        self.frame += 1

    def run_frames(self, kspace, frames, out):
        for fo in range(frames):
            self._frame(kspace, self.frame, out, fo)
        return out


class RowShardedEngine(RowShardLoop):
    """One rank (one GPU) of the row-sharded online loop (BASELINE config 4) on the device.

    The rank owns k-space rows [r0, r1) of Ah; Bh is replicated. ``rows``/``counts`` give static row
    tables, or ``rows`` is an :class:`Informative` policy (every rank draws the same rows from the same
    Philox stream and the all-reduced row energies; the drawn set goes from phase 1 to phase 2 on the
    device). ``allreduce`` defaults to ``torch.distributed.all_reduce`` (NCCL). ``run(graph=True)`` captures
    the whole T-frame chain — kernels and NCCL collectives — in one CUDA graph (the first frame runs
    eagerly to settle one-time launch attributes and communicator setup) and replays it.
    """

    def __init__(self, nx, ny, rank, lam, step, rows, counts=None, world=1, rank_id=0, cluster=0, t0=1,
                 allreduce=None):
        from .sharding import payload_doubles, row_partition

        self.nx, self.ny, self.R = int(nx), int(ny), int(rank)
        self.world, self.rank_id = int(world), int(rank_id)
        if not 0 <= self.rank_id < self.world:
            raise ValueError("need 0 <= rank_id < world")
        self.r0, self.r1 = row_partition(self.nx, self.world, self.rank_id)
        self.lam, self.step = float(lam), step
        self.dev = L.device()
        self.policy = rows if isinstance(rows, Informative) else None
        self.informative = self.policy is not None
        if self.informative:
            pol = self.policy
            if not 1 <= pol.k <= self.nx or not pol.replacement:
                raise ValueError("sharded informative draws: 1 <= k <= nx, with replacement")
            forced = np.unique(np.asarray(pol.forced, dtype=np.int64))
            if forced.size > pol.k or (forced.size and (forced.min() < 0 or forced.max() >= self.nx)):
                raise ValueError("bad forced rows")
            self.forced = torch.from_numpy(forced.astype(np.int32)).to(self.dev)
            self.max_rows = int(pol.k)
            self.philox_pos = torch.full((1,), int(pol.pos0), dtype=torch.int64, device=self.dev)
            self.energy = torch.zeros(self.nx, self.R, dtype=torch.float64, device=self.dev)
            self.sraw = torch.zeros(self.nx, dtype=torch.float64, device=self.dev)
            self.rows_tab = None
        else:
            rows = np.asarray(rows).reshape(np.asarray(rows).shape[0], -1)
            self.max_rows = int(rows.shape[1])
            self.rows_tab = torch.from_numpy(np.ascontiguousarray(rows, dtype=np.int32)).to(self.dev)
            self.rows_cnt = torch.from_numpy(np.ascontiguousarray(np.asarray(counts).reshape(-1),
                                                                  dtype=np.int32)).to(self.dev)
        self.scr = K.RowsScratch(1, self.nx, self.ny, self.R, self.max_rows, cluster)
        self.cluster = self.scr.cluster
        self.ah = torch.zeros(self.r1 - self.r0, self.R, dtype=torch.complex64, device=self.dev)
        self.bh = torch.zeros(self.ny, self.R, dtype=torch.complex64, device=self.dev)
        # the frame's payload in one fp64 buffer: W (ny x R complex128) then GA / ||Y||^2 / ||Ah||^2, so one
        # all-reduce per frame carries all of it
        nw = 2 * self.ny * self.R
        self.payload = torch.zeros(payload_doubles(self.ny, self.R), dtype=torch.float64, device=self.dev)
        self.xw = self.payload[:nw].view(torch.complex128).view(self.ny, self.R)
        self.xg = self.payload[nw:]
        self.alpha_bar = torch.zeros(1, dtype=torch.float64, device=self.dev)
        self.status = torch.zeros(1, dtype=torch.int32, device=self.dev)
        self.t = int(t0)
        self.frame = 0
        self._keep = []
        if allreduce is None:
            import torch.distributed as dist

            def allreduce(t):
                dist.all_reduce(t, op=dist.ReduceOp.SUM)
        self.allreduce = allreduce

    def set_image_factors(self, A, B):
        """Full image-domain factors (nx, R), (ny, R) -> this rank's k-space rows and Bh."""
        a = torch.as_tensor(np.asarray(A) if not isinstance(A, torch.Tensor) else A).to(self.dev, torch.complex64)
        b = torch.as_tensor(np.asarray(B) if not isinstance(B, torch.Tensor) else B).to(self.dev, torch.complex64)
        ah = K.fft_cols_(a.reshape(self.nx, self.R).contiguous())
        self.ah = ah[self.r0:self.r1].contiguous()
        self.bh = K.fft_cols_(b.reshape(self.ny, self.R).contiguous())

    def make_outputs(self, frames):
        d = self.dev
        out = dict(gamma=torch.empty(frames, self.R, dtype=torch.complex64, device=d),
                   cost=torch.empty(frames, dtype=torch.float64, device=d),
                   mu=torch.empty(frames, dtype=torch.float64, device=d),
                   ah=torch.empty(frames, self.r1 - self.r0, self.R, dtype=torch.complex64, device=d),
                   bh=torch.empty(frames, self.ny, self.R, dtype=torch.complex64, device=d))
        if self.informative:  # each frame's drawn rows (all ranks'), sorted, -1 padded
            out["rows"] = torch.full((frames, self.max_rows), -1, dtype=torch.int32, device=d)
            out["cnt"] = torch.zeros(frames, dtype=torch.int32, device=d)
        return out

    def _args(self, kspace, f, out, fo, phase):
        mode, mu, cf, cc = _step_params(self.step)
        a = L.RowsArgs()
        a.nslices, a.nx, a.ny, a.rank, a.frames = 1, self.nx, self.ny, self.R, 1
        a.max_rows, a.cluster, a.t0 = self.max_rows, self.cluster, self.t
        a.ah_in = a.ah_out = self.ah.data_ptr()
        a.bh_in = a.bh_out = self.bh.data_ptr()
        a.alpha_bar = self.alpha_bar.data_ptr()
        if self.informative and phase == 1:
            pol = self.policy
            a.policy = L.TT_POLICY_INFORMATIVE
            a.k_draws = int(pol.k)
            a.forced = self.forced.data_ptr() if self.forced.numel() else None
            a.nforced = int(self.forced.numel())
            a.beta = float(pol.beta)
            a.key0, a.key1 = int(pol.key0), int(pol.key1)
            a.philox_pos = self.philox_pos.data_ptr()
            a.sraw_in = self.sraw.data_ptr()
            a.rows_out = out["rows"][fo].data_ptr()  # the drawn set, read back by phase 2
            a.cnt_out = out["cnt"][fo:].data_ptr()
        elif self.informative:
            a.policy = L.TT_POLICY_STATIC
            a.rows_tab = out["rows"][fo].data_ptr()
            a.rows_cnt = out["cnt"][fo:].data_ptr()
        else:
            a.policy = L.TT_POLICY_STATIC
            a.rows_tab = self.rows_tab.data_ptr() + 4 * f * self.max_rows
            a.rows_cnt = self.rows_cnt.data_ptr() + 4 * f
        a.y_mode = L.TT_Y_GATHER
        a.ysrc = kspace[f].data_ptr()
        a.y_frame_stride, a.y_slice_stride = self.nx * self.ny, self.nx * self.ny
        a.lam, a.step_mode, a.mu, a.c_floor, a.c_cap = self.lam, mode, mu, cf, cc
        if phase == 2 and out is not None:
            a.gamma_out = out["gamma"][fo].data_ptr()
            a.cost_out = out["cost"][fo:].data_ptr()
            a.mu_out = out["mu"][fo:].data_ptr()
            a.ah_hist = out["ah"][fo].data_ptr()
            a.bh_hist = out["bh"][fo].data_ptr()
        a.status = self.status.data_ptr()
        a.scratch = self.scr.buf.data_ptr()
        a.shard_rank, a.shard_world, a.shard_phase = self.rank_id, self.world, phase
        a.xw, a.xg = self.xw.data_ptr(), self.xg.data_ptr()
        self._keep.append(a)
        return a

    # ---- the phases on the device
    def _energy(self):
        L.check(L.lib().tt_rows_shard_energy(L.stream_ptr(), self.nx, self.R, self.r0, self.r1 - self.r0,
                                             self.ah.data_ptr(), self.energy.data_ptr()), "shard energy")

    def _scores(self):
        L.check(L.lib().tt_rows_shard_scores(L.stream_ptr(), self.nx, self.ny, self.R, self.energy.data_ptr(),
                                             self.sraw.data_ptr(), self.status.data_ptr()), "shard scores")

    def _phase1(self, kspace, f):
        K.track_rows(self._args(kspace, f, self._out, self._fo, 1))

    def _phase2(self, kspace, f, out, fo):
        K.track_rows(self._args(kspace, f, out, fo, 2))

    def _frame(self, kspace, f, out, fo):
        self._out, self._fo = out, fo
        super()._frame(kspace, f, out, fo)

    # ---- the per-frame API of the emulation tests
    def partial(self, kspace, f, out=None, fo=0):
        if self.informative:
            self._energy()
            self.allreduce(self.energy)
            self._scores()
        self._out, self._fo = out, fo
        self._phase1(kspace, f)

    def finish(self, kspace, f, out, fo):
        self._phase2(kspace, f, out, fo)
        self.t += 1
        self.frame += 1

    def save(self):
        """A copy of the rank's state (factors, step accumulator, Philox position, status, t, frame)."""
        return (self.ah.clone(), self.bh.clone(), self.alpha_bar.clone(),
                self.philox_pos.clone() if self.informative else None, self.status.clone(), self.t, self.frame)

    def restore(self, saved):
        """Back to a :meth:`save`d state, into the same buffers (a captured graph stays valid)."""
        ah, bh, ab, pp, st, t, f = saved
        self.ah.copy_(ah)
        self.bh.copy_(bh)
        self.alpha_bar.copy_(ab)
        if pp is not None:
            self.philox_pos.copy_(pp)
        self.status.copy_(st)
        self.t, self.frame = t, f

    def capture(self, kspace, frames, out):
        """Capture the next ``frames`` frames — energies, scores, both phases and the NCCL collectives —
        into one CUDA graph without running them (``replay`` runs them). One eager frame first, on the
        state that is then restored, settles one-time launch attributes and the communicator."""
        saved = self.save()
        self._keep = []
        self._frame(kspace, self.frame, out, 0)
        self.restore(saved)
        g = torch.cuda.CUDAGraph()
        f0, t0 = self.frame, self.t
        with torch.cuda.graph(g):
            for fo in range(frames):
                self._frame(kspace, f0 + fo, out, fo)
        self.frame, self.t = f0, t0
        self._graph = (g, list(self._keep), int(frames))
        return g

    def replay(self):
        g, _, frames = self._graph
        g.replay()
        self.frame += frames
        self.t += frames

    def run(self, kspace, frames, out=None, graph=False):
        """kspace: (T, nx, ny) complex64 CUDA (full frames). Frames from the current index. ``graph``:
        capture the frames (kernels and collectives) in one CUDA graph and replay it."""
        if out is None:
            out = self.make_outputs(frames)
        if graph and frames > 0:
            self.capture(kspace, frames, out)
            self.replay()
        else:
            self._keep = []
            self.run_frames(kspace, frames, out)
        return out

    def check_status(self):
        L.raise_status(int(self.status.max().item()), "row-sharded engine")
