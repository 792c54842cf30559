"""Per-patch independent trackers on the device (experiment._run_tracking_patched,
`pkg/src/tensortrack/experiment.py:332-441`).

The frame is tiled by a :class:`~.mri.PatchGrid` into k1 x k2 patches, each tracked by its own
rank-rho EntryMask tracker on the entries that fall inside it. Device flow (C ABI
``tt_patch_bin`` / ``tt_track_patches``):

1. the frames' entry lists are split per patch in measurement order (one kernel for all frames);
2. warm-up: ``warm_epochs`` passes over the warm frames, every patch rebalanced (``tt_rebalance``)
   before each pass after the first; each pass is one launch with one CTA per patch;
3. ``epochs`` passes over the remaining frames (rebalanced between passes, order re-drawn with the
   caller's ``rng.permutation`` when ``reshuffle``), one launch each, recording the per-step
   reports;
4. every frame, warm ones included, is re-projected onto each patch's final subspace and the tiles
   are written straight into the assembled frames (one launch).

The reference draws, from one generator and in this order, the per-patch initial subspaces, then
each frame's mask, then the reshuffle permutations. :func:`init_patch_factors` and
:func:`draw_frame_entries` reproduce the first two; pass the same generator as ``rng`` for the
third. Noise is pre-baked into ``frames``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .metrics import nmse_frames
from . import _lib as L
from . import _ops as K
from .mri import PatchGrid
from .observation import rows_to_entries, variable_density_rows
from .tracker import Fixed, HessianBound, random_subspace

__all__ = ["PatchedResult", "init_patch_factors", "draw_frame_entries", "full_entries", "run_tracking_patched"]


def full_entries(shape) -> np.ndarray:
    """All (i, j) of a frame, row-major (experiment.py:139-141)."""
    g = np.meshgrid(*[np.arange(n, dtype=np.int64) for n in shape], indexing="ij")
    return np.stack([x.ravel() for x in g], axis=1)


def init_patch_factors(grid: PatchGrid, rng, init_scale: float = 1.0):
    """The reference's per-patch ``init_state`` draws (experiment.py:347-350): one
    ``random_subspace((n1, n2), rho, rng)`` per patch in row-major order. Returns (A0s, B0s) of
    shapes (npatch, n1, rho), (npatch, n2, rho)."""
    A, B = [], []
    for _ in range(grid.k1 * grid.k2):
        sub = random_subspace((grid.n1, grid.n2), grid.rho, rng, init_scale)
        A.append(sub.factors[0])
        B.append(sub.factors[1])
    return np.stack(A), np.stack(B)


def draw_frame_entries(mode: str, shape, rng, fraction: float = 0.1, alpha: float = -1.0) -> np.ndarray:
    """One frame's static mask (_draw_frame_entries, experiment.py:159-174): ``full``, ``variable_density``
    (rows in draw order, expanded row-major) or ``uniform`` (sorted flat entries without replacement)."""
    if mode == "full":
        return full_entries(shape)
    if mode in ("variable_density", "adaptive"):
        rows = variable_density_rows(shape[0], alpha, fraction, rng)
        return rows_to_entries(rows, shape[1])
    if mode == "uniform":
        total = int(np.prod(shape))
        k = max(1, int(np.ceil(fraction * total)))
        flat = rng.choice(total, size=k, replace=False)
        return np.stack(np.unravel_index(np.sort(flat), shape), axis=1)
    raise ValueError(f"unknown sampling mode {mode!r}")


@dataclass
class PatchedResult:
    """RunResult of a patched run (experiment.py:434-441) plus the per-patch arrays behind it.

    ``step_gamma`` (steps, npatch * rho): each main-epoch step's gammas concatenated over patches;
    ``step_cost`` the per-step cost summed over patches; ``step_mu`` / ``step_t`` patch 0's step
    size and pre-step t (the StepReport fields, experiment.py:398-406); ``step_residual`` the
    concatenated residuals when requested; ``gamma`` (T, npatch, rho) the final re-projection;
    ``recon`` (T, N1, N2) the assembled frames; ``nmse`` per frame against ``clean`` (or the
    frames); ``samples`` per frame."""

    recon: np.ndarray
    gamma: np.ndarray
    step_gamma: np.ndarray
    step_cost: np.ndarray
    step_mu: np.ndarray
    step_t: np.ndarray
    step_residual: list | None
    orders: list
    final_A: np.ndarray
    final_B: np.ndarray
    t: int
    nmse: np.ndarray
    samples: np.ndarray


def _step_params(step):
    if isinstance(step, Fixed):
        return 0, float(step.mu), 0.0, 0.0
    if isinstance(step, HessianBound):
        return 1, 0.0, float(step.c_floor), float(step.c_cap)
    raise TypeError(f"unknown step policy {step!r}")


class _PatchRun:
    """Device state of one patched run: binned data, factors, and the launch helper."""

    def __init__(self, grid: PatchGrid, lam, step, frames_dev, entries=None, offsets=None):
        self.grid = grid
        self.lam = float(lam)
        self.mode, self.mu, self.c_floor, self.c_cap = _step_params(step)
        self.dev = frames_dev.device
        T, N1, N2 = frames_dev.shape
        self.T, self.N1, self.N2 = T, N1, N2
        self.np = grid.k1 * grid.k2
        self.cap = grid.n1 * grid.n2
        self.frames = frames_dev
        self.pidx = torch.empty((T, self.np, self.cap), dtype=torch.int32, device=self.dev)
        self.py = torch.empty((T, self.np, self.cap), dtype=torch.complex64, device=self.dev)
        self.pcnt = torch.zeros((T, self.np), dtype=torch.int32, device=self.dev)
        self.bin_status = torch.zeros(1, dtype=torch.int32, device=self.dev)
        self.status = torch.zeros(self.np, dtype=torch.int32, device=self.dev)
        self._keep = []
        if entries is not None:
            self.bin(torch.from_numpy(entries).to(self.dev), torch.from_numpy(offsets).to(self.dev), 0, T)

    def bin(self, ent_dev, off_dev, f0, f1):
        """Split frames [f0, f1) per patch (``ent_dev`` / ``off_dev``: their compact mask table)."""
        g = self.grid
        fb = 8 * self.N1 * self.N2
        pb = self.np * self.cap
        L.check(L.lib().tt_patch_bin(L.stream_ptr(), self.N1, self.N2, g.n1, g.n2, f1 - f0,
                                     self.frames.data_ptr() + f0 * fb, ent_dev.data_ptr(), off_dev.data_ptr(),
                                     self.pidx.data_ptr() + 4 * f0 * pb, self.py.data_ptr() + 8 * f0 * pb,
                                     self.pcnt.data_ptr() + 4 * f0 * self.np, self.bin_status.data_ptr()),
                "patch binning")
        self._keep.append((ent_dev, off_dev))

    def set_factors(self, A0s, B0s, t0=1):
        g = self.grid
        self.a = torch.from_numpy(np.ascontiguousarray(A0s, dtype=np.complex64).reshape(self.np, g.n1, g.rho)).to(self.dev)
        self.b = torch.from_numpy(np.ascontiguousarray(B0s, dtype=np.complex64).reshape(self.np, g.n2, g.rho)).to(self.dev)
        self.t = torch.full((self.np,), int(t0), dtype=torch.int64, device=self.dev)
        self.ab = torch.zeros(self.np, dtype=torch.float64, device=self.dev)

    def launch(self, sched, project=False, gamma=None, cost=None, mu=None, resid=None, recon=None):
        g = self.grid
        sd = torch.from_numpy(np.asarray(sched, dtype=np.int32)).to(self.dev, non_blocking=True)
        args = L.PatchesArgs(
            nx=self.N1, ny=self.N2, pn1=g.n1, pn2=g.n2, rank=g.rho, patch0=0, npatch_local=self.np, frames=self.T,
            pidx=self.pidx.data_ptr(), py=self.py.data_ptr(), pcnt=self.pcnt.data_ptr(), nsteps=len(sched),
            sched=sd.data_ptr(), a=self.a.data_ptr(), b=self.b.data_ptr(), t=self.t.data_ptr(),
            alpha_bar=self.ab.data_ptr(), lam=self.lam, step_mode=self.mode, mu=self.mu, c_floor=self.c_floor,
            c_cap=self.c_cap, project=int(project), gamma_out=L.ptr(gamma), cost_out=L.ptr(cost),
            mu_out=L.ptr(mu), resid_out=L.ptr(resid), recon_out=L.ptr(recon), status=self.status.data_ptr())
        L.check(L.lib().tt_track_patches(L.stream_ptr(), args), "patch tracking")
        return sd  # keep the schedule alive until the stream passes it

    def rebalance(self):
        K.rebalance_(self.a, self.b, self.status)


def _entry_table(masks, shape, T):
    """Masks -> the compact device layout: concatenated (i, j) int32 pairs and int64 frame offsets."""
    cnt = np.array([len(np.asarray(m).reshape(-1, 2)) for m in masks], dtype=np.int64)
    off = np.zeros(T + 1, dtype=np.int64)
    np.cumsum(cnt, out=off[1:])
    ent = np.empty((max(int(off[-1]), 1), 2), dtype=np.int32)
    for t, m in enumerate(masks):
        ent[off[t]:off[t + 1]] = np.asarray(m, dtype=np.int64).reshape(-1, 2)
    return ent, off


def run_tracking_patched(frames, grid: PatchGrid, lam, step, masks, warm_n=0, warm_epochs=1, epochs=1, rng=None,
                         reshuffle=False, A0s=None, B0s=None, init_scale=1.0, clean=None, keep_residual=False,
                         frames_last=False) -> PatchedResult:
    """_run_tracking_patched (experiment.py:332-441) on the device.

    ``frames`` (T, N1, N2) pre-noised data (or (N1, N2, T), the reference's layout, with
    ``frames_last``); ``masks[t]`` the frame's global (i, j) entries in measurement order (the warm
    frames' are normally the full frame, :func:`full_entries`); ``A0s``/``B0s`` the per-patch initial
    factors (drawn from ``rng`` by :func:`init_patch_factors` when omitted — the reference draws
    them first). Steps, rebalancing, reshuffling and the final re-projection follow the reference
    loop for loop (see the module docstring)."""
    if not isinstance(grid, PatchGrid):
        raise TypeError("grid must be a PatchGrid")
    if epochs < 1 or warm_epochs < 1:
        raise ValueError("epochs must be at least 1")
    src = frames if isinstance(frames, torch.Tensor) else torch.from_numpy(np.asarray(frames))
    if frames_last:
        src = src.permute(2, 0, 1)
    if src.dim() != 3 or tuple(src.shape[1:]) != grid.frame_shape:
        raise ValueError(f"frames {tuple(src.shape)} do not match the grid {grid.frame_shape}")
    T = src.shape[0]
    if len(masks) != T:
        raise ValueError("one mask per frame is required")
    warm_n = min(int(warm_n), T)
    if A0s is None or B0s is None:
        if rng is None:
            raise ValueError("initial factors or a generator are required")
        A0s, B0s = init_patch_factors(grid, rng, init_scale)
    if reshuffle and epochs > 1 and rng is None:
        raise ValueError("rng is required for reshuffling")
    dev = L.device()
    comp = torch.cuda.current_stream()
    # pinned (or device) input uploads asynchronously; a pageable one is copied as is
    fd = src.to(torch.complex64).to(dev, non_blocking=True).contiguous()
    run = _PatchRun(grid, lam, step, fd)
    run.set_factors(A0s, B0s)
    npch, R = run.np, grid.rho

    def upload_bin(f0, f1, stream):
        ent, off = _entry_table(masks[f0:f1], grid.frame_shape, f1 - f0)
        with torch.cuda.stream(stream):  # the driver stages the pageable copy; the compute stream runs on
            ed = torch.from_numpy(ent).to(dev, non_blocking=True)
            od = torch.from_numpy(off).to(dev, non_blocking=True)
        comp.wait_stream(stream)
        run.bin(ed, od, f0, f1)
        return np.diff(off)

    # the warm frames' masks first, so the warm-up starts; the streamed frames' masks are built on the
    # host and uploaded on a copy stream while it runs
    s_copy = torch.cuda.Stream()
    samples = []
    if warm_n:
        samples.append(upload_bin(0, warm_n, s_copy))
    keep = []
    for epoch in range(warm_epochs):
        if warm_n == 0:
            break
        if epoch > 0:
            run.rebalance()
        keep.append(run.launch(list(range(warm_n))))
    if warm_n < T:
        samples.append(upload_bin(warm_n, T, s_copy))
    samples = np.concatenate(samples) if samples else np.zeros(0, np.int64)
    gam_s, cost_s, mu_s, res_s, orders, scheds = [], [], [], [], [], []
    main = T - warm_n
    for epoch in range(epochs):
        if epoch > 0:
            run.rebalance()
        order = list(range(warm_n, T))
        if reshuffle and epoch > 0:
            order = [warm_n + int(i) for i in rng.permutation(main)]
        orders.append(order)
        if not order:
            continue
        n = len(order)
        g = torch.empty((n, npch, R), dtype=torch.complex64, device=dev)
        c = torch.empty((n, npch), dtype=torch.float64, device=dev)
        m = torch.empty((n, npch), dtype=torch.float64, device=dev)
        r = torch.empty((n, npch, run.cap), dtype=torch.complex64, device=dev) if keep_residual else None
        keep.append(run.launch(order, gamma=g, cost=c, mu=m, resid=r))
        gam_s.append(g)
        cost_s.append(c)
        mu_s.append(m)
        res_s.append(r)
        scheds.extend(order)
    # re-projection of every frame onto the final subspaces, tiles assembled in place; in blocks, each
    # downloaded into pinned memory while the next is computed
    gam = torch.empty((T, npch, R), dtype=torch.complex64, device=dev)
    recon = torch.empty((T,) + grid.frame_shape, dtype=torch.complex64, device=dev)
    recon_h = torch.empty((T,) + grid.frame_shape, dtype=torch.complex64, pin_memory=True)
    for a0 in range(0, T, 50):
        a1 = min(T, a0 + 50)
        keep.append(run.launch(list(range(a0, a1)), project=True, gamma=gam[a0:a1], recon=recon))
        s_copy.wait_stream(comp)
        with torch.cuda.stream(s_copy):
            recon_h[a0:a1].copy_(recon[a0:a1], non_blocking=True)
    if clean is None:
        ref = fd
    else:
        ct = clean if isinstance(clean, torch.Tensor) else torch.from_numpy(np.asarray(clean))
        ref = (ct.permute(2, 0, 1) if frames_last else ct).to(dev, torch.complex64)
    err = nmse_frames(ref, recon)  # metrics.py:53-62, per frame
    # the small results: asynchronous downloads into pinned memory, one synchronisation
    pinned = lambda t: torch.empty(t.shape, dtype=t.dtype, pin_memory=True)  # noqa: E731
    dl = {"gamma": gam, "err": err, "pcnt": run.pcnt, "A": run.a, "B": run.b, "t": run.t[:1],
          "st": torch.stack([run.status.max(), run.bin_status[0]])}
    if cost_s:
        dl.update(cost=torch.cat(cost_s), mu=torch.cat(mu_s), sg=torch.cat(gam_s))
    if keep_residual and res_s:
        dl["resid"] = torch.cat([x for x in res_s if x is not None])
    host = {k: pinned(v) for k, v in dl.items()}
    for k, v in dl.items():
        host[k].copy_(v, non_blocking=True)
    comp.wait_stream(s_copy)
    comp.synchronize()
    h = {k: v.numpy() for k, v in host.items()}
    h["recon"] = recon_h.numpy()
    L.raise_status(int(h["st"][0]) | int(h["st"][1]), "patched tracking")

    pcnt = h["pcnt"]
    cost = h["cost"] if cost_s else np.zeros((0, npch))
    mu = h["mu"] if cost_s else np.zeros((0, npch))
    sg = h["sg"].reshape(-1, npch * R) if cost_s else np.zeros((0, npch * R), np.complex64)
    t_first = 1 + warm_epochs * warm_n if warm_n else 1
    step_t = np.arange(t_first, t_first + len(scheds), dtype=np.int64)
    resid = None
    if keep_residual:
        rr = h.get("resid", np.zeros((0, npch, run.cap), np.complex64))
        resid = [np.concatenate([rr[k, p, :pcnt[f, p]] for p in range(npch)]) for k, f in enumerate(scheds)]
    # per-step cost summed over patches left to right, as Python's sum does (experiment.py:402)
    step_cost = np.cumsum(cost, axis=1)[:, -1] if cost.shape[0] and npch else np.zeros(cost.shape[0])
    return PatchedResult(
        recon=h["recon"], gamma=h["gamma"], step_gamma=sg,
        step_cost=step_cost, step_mu=mu[:, 0] if len(mu) else mu.reshape(0),
        step_t=step_t, step_residual=resid, orders=orders, final_A=h["A"], final_B=h["B"],
        t=int(h["t"][0]) if npch else 1, nmse=h["err"], samples=samples)
