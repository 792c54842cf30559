"""Online stochastic MM tracker — drop-in for ``tensortrack.tracker``
(`pkg/src/tensortrack/tracker.py`).

Same names, arguments, defaults, validation and exceptions as the reference
(`Fixed` :51, `HessianBound` :62, `StepConfig` :74, `TrackerState` :99,
`StepReport` :109, `random_subspace` :119, `init_state` :129, `solve_gamma`
:139, `track_step` :367, `run` :456). The arithmetic runs in the CUDA
library: ``track_step`` launches the fused row-mask cluster kernel when the
descriptor is whole phase-encode lines (the BASELINE configs) and the
generic index kernels otherwise. The returned state owns new device buffers
(functional update, tracker.py:411); report fields are read back lazily.
"""

from __future__ import annotations

from dataclasses import dataclass, replace

import numpy as np
import torch

from . import _lib as L
from . import _ops as K
from .core import TensorSubspace, rebalance
from .observation import EntryMask, FourierMask, MeasurementBatch, descriptor_kind

__all__ = [
    "Fixed",
    "HessianBound",
    "StepConfig",
    "TrackerState",
    "StepReport",
    "random_subspace",
    "init_state",
    "solve_gamma",
    "instantaneous_cost",
    "factor_gradient",
    "hessian_bound",
    "track_step",
    "run",
]


@dataclass(frozen=True)
class Fixed:
    """Constant step size (tracker.py:51-59)."""

    mu: float

    def __post_init__(self):
        if self.mu <= 0:
            raise ValueError("fixed step size must be positive")


@dataclass(frozen=True)
class HessianBound:
    """mu_t = 1 / sum_tau alpha_tau with clamped alpha (tracker.py:62-71)."""

    c_floor: float
    c_cap: float

    def __post_init__(self):
        if not 0 < self.c_floor <= self.c_cap:
            raise ValueError("need 0 < c_floor <= c_cap")


@dataclass(frozen=True)
class StepConfig:
    """Tracker hyperparameters (tracker.py:74-96)."""

    lam: float
    rank: int
    step: Fixed | HessianBound = Fixed(0.01)
    warm_start: TensorSubspace | None = None
    init_scale: float = 1.0
    norm_cap: float | None = None

    def __post_init__(self):
        if self.lam < 0:
            raise ValueError("lambda must be nonnegative")
        if self.rank < 1:
            raise ValueError("rank must be at least 1")
        if self.init_scale <= 0:
            raise ValueError("init_scale must be positive")


@dataclass(frozen=True)
class TrackerState:
    """The single mutable object of the online loop (tracker.py:99-106)."""

    subspace: TensorSubspace
    config: StepConfig
    t: int = 1
    alpha_bar: float = 0.0


class StepReport:
    """Per-step outputs (tracker.py:109-116). Device values are copied to
    host (complex128 / float, like the reference) on first access."""

    __slots__ = ("_gamma", "_residual", "_cost", "_mu", "t", "_norm")

    def __init__(self, gamma, residual, cost, step_size, t, norm_exceeded=False):
        self._gamma, self._residual, self._cost, self._mu = gamma, residual, cost, step_size
        self.t = int(t)
        self._norm = norm_exceeded

    @staticmethod
    def _host(v, dtype):
        if isinstance(v, torch.Tensor):
            return v.detach().cpu().numpy().astype(dtype)
        return np.asarray(v, dtype=dtype)

    @property
    def gamma(self) -> np.ndarray:
        if not isinstance(self._gamma, np.ndarray):
            self._gamma = self._host(self._gamma, np.complex128).ravel()
        return self._gamma

    @property
    def residual(self) -> np.ndarray:
        if not isinstance(self._residual, np.ndarray):
            self._residual = self._host(self._residual, np.complex128).ravel()
        return self._residual

    @property
    def instantaneous_cost(self) -> float:
        if not isinstance(self._cost, float):
            self._cost = float(self._host(self._cost, np.float64).ravel()[0])
        return self._cost

    @property
    def step_size(self) -> float:
        if not isinstance(self._mu, float):
            self._mu = float(self._host(self._mu, np.float64).ravel()[0])
        return self._mu

    @property
    def norm_exceeded(self) -> bool:
        if callable(self._norm):
            self._norm = bool(self._norm())
        return bool(self._norm)

    # device views (no copy), for device-resident callers
    @property
    def gamma_device(self):
        return self._gamma if isinstance(self._gamma, torch.Tensor) else None


def random_subspace(dims, rank: int, rng, init_scale: float = 1.0) -> TensorSubspace:
    """Random init (tracker.py:119-126): entries i.i.d. complex Gaussian with
    scale init_scale / sqrt(N_m), drawn from the caller's host Generator so
    the values match the reference bit for bit."""
    factors = []
    for n in dims:
        scale = init_scale / np.sqrt(n)
        z = rng.standard_normal((n, rank)) + 1j * rng.standard_normal((n, rank))
        factors.append(scale * z / np.sqrt(2.0))
    return TensorSubspace(tuple(factors))


def init_state(config: StepConfig, dims, rng) -> TrackerState:
    """tracker.py:129-136."""
    if config.warm_start is not None:
        sub = config.warm_start
        if not isinstance(sub, TensorSubspace):
            sub = TensorSubspace(sub.factors)
        if sub.dims != tuple(dims) or sub.rank != config.rank:
            raise ValueError("warm-start subspace does not match dims/rank")
    else:
        sub = random_subspace(dims, config.rank, rng, config.init_scale)
    return TrackerState(subspace=sub, config=config)


def solve_gamma(phi, y, lam: float) -> np.ndarray:
    """Ridge projection (tracker.py:139-156) as the fp64 normal equations
    (Phi^H Phi + lam I) g = Phi^H y solved by LDL^H on the GPU; equal to the
    reference's SVD filter for lam > 0 (and for full-rank Phi at lam = 0)."""
    phi = np.asarray(phi, dtype=np.complex128)
    y = np.asarray(y, dtype=np.complex128).ravel()
    if phi.ndim != 2 or phi.shape[0] != y.size:
        raise ValueError(f"phi shape {phi.shape} inconsistent with y length {y.size}")
    if phi.shape[0] == 0:
        return np.zeros(phi.shape[1], dtype=np.complex128)
    dev = L.device()
    g = K.solve_gamma(torch.from_numpy(np.ascontiguousarray(phi)).to(dev), torch.from_numpy(y).to(dev), float(lam))
    return g.cpu().numpy()


def _index_inputs(subspace, descriptor, gamma):
    """Measurement factors, device index list and complex64 gamma for the
    standalone step pieces."""
    if not isinstance(subspace, TensorSubspace):
        subspace = TensorSubspace(subspace.factors)
    if subspace.dims != descriptor.shape:
        raise ValueError("descriptor does not match the subspace dimensions")
    kind = descriptor_kind(descriptor)
    ah, bh = subspace.measurement_factors(kind)
    dev = ah.device
    idx = torch.from_numpy(np.ascontiguousarray(descriptor.indices, dtype=np.int32)).to(dev)
    g = torch.from_numpy(np.asarray(gamma, dtype=np.complex128).ravel().astype(np.complex64)).to(dev)
    if g.numel() != subspace.rank:
        raise ValueError("gamma length does not match the rank")
    return subspace, kind, ah.contiguous(), bh.contiguous(), idx, g


def instantaneous_cost(subspace, batch, lam: float, t: int, gamma) -> float:
    """0.5 ||y - Phi gamma||^2 + 0.5 (lam/t)(||A||^2 + ||B||^2) (tracker.py:163-173),
    residual from the device kernel ``tt_residual``."""
    sub, kind, ah, bh, idx, g = _index_inputs(subspace, batch.descriptor, gamma)
    nx, ny = sub.dims
    L_ = batch.descriptor.nmeas
    e = torch.empty(max(L_, 1), dtype=torch.complex64, device=ah.device)
    if L_:
        y = batch.y_device()
        L.check(L.lib().tt_residual(L.stream_ptr(), nx, ny, sub.rank, L_, ah.data_ptr(), bh.data_ptr(),
                                    idx.data_ptr(), y.data_ptr(), g.data_ptr(), e.data_ptr()), "residual")
    en = float(torch.linalg.vector_norm(ah.to(torch.complex128)) ** 2 + torch.linalg.vector_norm(bh.to(torch.complex128)) ** 2)
    r2 = float(torch.linalg.vector_norm(e[:L_].to(torch.complex128)) ** 2) if L_ else 0.0
    return 0.5 * r2 + 0.5 * (lam / t) * en


def _data_terms(sub, kind, ah, bh, idx, g, residual):
    nx, ny = sub.dims
    R = sub.rank
    dev = ah.device
    L_ = int(idx.shape[0])
    e = torch.from_numpy(np.asarray(residual, dtype=np.complex128).ravel().astype(np.complex64)).to(dev) \
        if residual is not None else torch.zeros(max(L_, 1), dtype=torch.complex64, device=dev)
    dA = torch.empty(nx, R, dtype=torch.complex64, device=dev)
    dB = torch.empty(ny, R, dtype=torch.complex64, device=dev)
    cmax = torch.empty(R, dtype=torch.float64, device=dev)
    scr = torch.empty(int(L.lib().tt_terms_scratch_bytes(nx, ny, R)), dtype=torch.uint8, device=dev)
    L.check(L.lib().tt_data_terms(L.stream_ptr(), nx, ny, R, L_, ah.data_ptr(), bh.data_ptr(),
                                  idx.data_ptr() if L_ else None, e.data_ptr() if L_ else None, g.data_ptr(),
                                  dA.data_ptr(), dB.data_ptr(), cmax.data_ptr(), scr.data_ptr()), "data_terms")
    return dA, dB, cmax


def factor_gradient(subspace, gamma, descriptor, residual, lam: float, t: int) -> list:
    """(lam/t) F - conj(gamma) . sum_l e_l conj(w_l) per mode (tracker.py:241-262) from the
    device data terms. For Fourier masks the k-space gradient is mapped back with the
    inverse column FFT (the data term is conj(gamma) . F^-1 P)."""
    sub, kind, ah, bh, idx, g = _index_inputs(subspace, descriptor, gamma)
    if np.asarray(residual).size != descriptor.nmeas:
        raise ValueError("residual length does not match descriptor")
    dA, dB, _ = _data_terms(sub, kind, ah, bh, idx, g, residual)
    s_ = float(lam) / float(t)
    gA = ah * s_ - dA
    gB = bh * s_ - dB
    if kind == "fourier":
        gA = K.fft_cols(gA.contiguous(), inverse=True)
        gB = K.fft_cols(gB.contiguous(), inverse=True)
    return [gA.cpu().numpy().astype(np.complex128), gB.cpu().numpy().astype(np.complex128)]


def hessian_bound(subspace, gamma, descriptor, lam: float, t: int, c_floor: float = 0.0, c_cap: float = np.inf,
                  iters: int = 1000, tol: float = 1e-8) -> float:
    """Curvature bound alpha_t (tracker.py:337-364) in closed form: for Fourier and entry
    masks lambda_max(G_{m,r}) is exactly the largest per-line sum of |Bh|^2 (|Ah|^2), which
    the reference's power iteration approaches from below (within its tolerance)."""
    del iters, tol
    sub, kind, ah, bh, idx, g = _index_inputs(subspace, descriptor, gamma)
    _, _, cmax = _data_terms(sub, kind, ah, bh, idx, g, None)
    gam = np.asarray(gamma, dtype=np.complex128).ravel()
    top = float(np.max(np.abs(gam) ** 2 * cmax.cpu().numpy())) if descriptor.nmeas else 0.0
    return float(np.clip(lam / t + top, c_floor, c_cap))


def _step_params(cfg: StepConfig):
    if isinstance(cfg.step, HessianBound):
        return L.TT_STEP_HESSIAN, 0.0, float(cfg.step.c_floor), float(cfg.step.c_cap)
    return L.TT_STEP_FIXED, float(cfg.step.mu), 0.0, 0.0


def _norm_flag(cap, a, b):
    if cap is None:
        return False

    def check():
        return bool((torch.linalg.vector_norm(a) > cap).item() or (torch.linalg.vector_norm(b) > cap).item())

    return check


def track_step(state: TrackerState, batch: MeasurementBatch):
    """One acquisition step: ridge projection (S1) then the parallel factor
    update (S2) from the frozen step-entry subspace (tracker.py:367-411)."""
    cfg = state.config
    sub = state.subspace
    if not isinstance(sub, TensorSubspace):
        sub = TensorSubspace(sub.factors)
    t = int(state.t)
    desc = batch.descriptor
    kind = descriptor_kind(desc)
    if desc.shape != sub.dims:
        raise ValueError("batch descriptor does not match tracker dimensions")
    sub._require_two_modes()
    nx, ny = sub.dims
    R = sub.rank
    dev = L.device()
    mode, mu, c_floor, c_cap = _step_params(cfg)
    ma, mb = sub.measurement_factors(kind)
    out_kind = "image" if kind == "fourier" else "direct"
    ah_out = torch.empty_like(ma)
    bh_out = torch.empty_like(mb)
    alpha = torch.tensor([float(state.alpha_bar)], dtype=torch.float64, device=dev)
    gamma = torch.empty(R, dtype=torch.complex64, device=dev)
    cost = torch.empty(1, dtype=torch.float64, device=dev)
    mu_out = torch.empty(1, dtype=torch.float64, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    rows = desc.row_lines
    nmeas = desc.nmeas

    if nmeas > 0 and rows is not None and not K.rows_plan_fits(nx, ny, R, int(rows.size)):
        rows = None  # shared-memory plan does not fit (e.g. R = 64 at 1024^2): generic index kernels
    if nmeas > 0 and rows is not None:
        S = int(rows.size)
        y = batch.y_device().reshape(S, ny)
        rows_t = torch.from_numpy(np.ascontiguousarray(rows, dtype=np.int32)).to(dev)
        cnt_t = torch.tensor([S], dtype=torch.int32, device=dev)
        resid = torch.empty(S, ny, dtype=torch.complex64, device=dev)
        scr = K.rows_scratch(1, nx, ny, R, S)
        a = L.RowsArgs()
        a.nslices, a.nx, a.ny, a.rank, a.frames, a.max_rows, a.cluster = 1, nx, ny, R, 1, S, scr.cluster
        a.t0 = t
        a.ah_in, a.bh_in, a.ah_out, a.bh_out = ma.data_ptr(), mb.data_ptr(), ah_out.data_ptr(), bh_out.data_ptr()
        a.alpha_bar = alpha.data_ptr()
        a.policy = L.TT_POLICY_STATIC
        a.rows_tab, a.rows_cnt = rows_t.data_ptr(), cnt_t.data_ptr()
        a.y_mode, a.ysrc = L.TT_Y_PACKED, y.data_ptr()
        a.lam, a.step_mode, a.mu, a.c_floor, a.c_cap = float(cfg.lam), mode, mu, c_floor, c_cap
        a.gamma_out, a.cost_out, a.mu_out = gamma.data_ptr(), cost.data_ptr(), mu_out.data_ptr()
        a.resid_out = resid.data_ptr()
        a.status, a.scratch = status.data_ptr(), scr.buf.data_ptr()
        K.track_rows(a)
        residual = resid.reshape(-1)
    else:
        idx = torch.from_numpy(np.ascontiguousarray(desc.indices, dtype=np.int32)).to(dev) if nmeas else None
        y = batch.y_device() if nmeas else None
        resid = torch.empty(max(nmeas, 1), dtype=torch.complex64, device=dev)
        scr = K.entries_scratch(nx, ny, R)
        a = L.EntriesArgs()
        a.nx, a.ny, a.rank, a.nmeas, a.t = nx, ny, R, nmeas, t
        a.ah_in, a.bh_in, a.ah_out, a.bh_out = ma.data_ptr(), mb.data_ptr(), ah_out.data_ptr(), bh_out.data_ptr()
        a.alpha_bar = alpha.data_ptr()
        a.idx = idx.data_ptr() if idx is not None else None
        a.y = y.data_ptr() if y is not None else None
        a.lam, a.step_mode, a.mu, a.c_floor, a.c_cap = float(cfg.lam), mode, mu, c_floor, c_cap
        a.gamma_out, a.cost_out, a.mu_out = gamma.data_ptr(), cost.data_ptr(), mu_out.data_ptr()
        a.resid_out = resid.data_ptr() if nmeas else None
        a.status, a.scratch = status.data_ptr(), scr.data_ptr()
        K.track_entries(a)
        residual = resid[:nmeas]

    if nmeas == 0:
        # empty batch: time advances only (tracker.py:380-384)
        report = StepReport(gamma, residual, cost, 0.0, t)
        return replace(state, subspace=TensorSubspace._from_device(ah_out, bh_out, out_kind)
                       if sub._dev is not None else sub, t=t + 1), report
    new_sub = TensorSubspace._from_device(ah_out, bh_out, out_kind)
    if mode == L.TT_STEP_HESSIAN:
        alpha_bar = float(alpha.item())
        step_size = mu_out
    else:
        alpha_bar = state.alpha_bar
        step_size = float(mu)
    report = StepReport(gamma, residual, cost, step_size, t, _norm_flag(cfg.norm_cap, ah_out, bh_out))
    return TrackerState(subspace=new_sub, config=cfg, t=t + 1, alpha_bar=alpha_bar), report


def empirical_cost(state: TrackerState, batches) -> float:
    """Averaged cost (1/T) sum_tau f_tau at the current subspace, coefficients re-solved per frame
    (tracker.py:414-430): build_phi, the device ridge solve and the device residual per batch."""
    from .observation import build_phi

    batches = list(batches)
    if not batches:
        raise ValueError("empirical cost needs at least one batch")
    total = 0.0
    for tau, batch in enumerate(batches, start=1):
        phi = build_phi(state.subspace, batch.descriptor)
        gamma = solve_gamma(phi, np.asarray(batch.y), state.config.lam)
        total += instantaneous_cost(state.subspace, batch, state.config.lam, tau, gamma)
    return total / len(batches)


def empirical_cost_gradient(state: TrackerState, batches) -> list:
    """Per-mode partial factor gradient at the re-solved coefficients, averaged over the batches
    (tracker.py:433-453; the stationarity diagnostic)."""
    from .observation import build_phi

    batches = list(batches)
    if not batches:
        raise ValueError("empirical cost gradient needs at least one batch")
    sums = [np.zeros(f.shape, dtype=np.complex128) for f in state.subspace.factors]
    for tau, batch in enumerate(batches, start=1):
        phi = build_phi(state.subspace, batch.descriptor)
        y = np.asarray(batch.y, dtype=np.complex128).ravel()
        gamma = solve_gamma(phi, y, state.config.lam)
        residual = y - phi @ gamma
        grads = factor_gradient(state.subspace, gamma, batch.descriptor, residual, state.config.lam, tau)
        for acc, g in zip(sums, grads):
            acc += g
    return [g / len(batches) for g in sums]


def run(stream, config: StepConfig, epochs: int = 1, reshuffle: bool = False, rng=None,
        initial: TrackerState | None = None, rebalance_epochs: bool = True):
    """Fold track_step over a stream, optionally for several epochs
    (tracker.py:456-500): global time keeps growing, epochs after the first
    are rebalanced and optionally reshuffled from ``rng``."""
    if epochs < 1:
        raise ValueError("epochs must be at least 1")
    batches = list(stream)
    if not batches:
        raise ValueError("empty measurement stream")
    if initial is None:
        if rng is None:
            raise ValueError("rng is required when no initial state is given")
        state = init_state(config, batches[0].descriptor.shape, rng)
    else:
        state = initial
    reports = []
    for epoch in range(epochs):
        if rebalance_epochs and epoch > 0:
            state = replace(state, subspace=rebalance(state.subspace))
        order = np.arange(len(batches))
        if reshuffle and epoch > 0:
            if rng is None:
                raise ValueError("rng is required for reshuffling")
            order = rng.permutation(len(batches))
        for k in order:
            state, report = track_step(state, batches[k])
            reports.append(report)
    return state.subspace, reports
