"""CPU oracle for the tensortrack online hot path — TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product. Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and the
``--impl reference`` arm) may import it. The package
``paper_1609_04104_b200`` never imports it and has no CPU fallback.

It restates, in float64/complex128 NumPy, the algorithm of the reference
package ``tensortrack`` (`/root/reference/pkg/src/tensortrack/`) for the
path named in BASELINE.json: ``build_phi`` (Fourier/Entry), the SVD ridge
``solve_gamma``, residual/cost, the power-method ``hessian_bound``, the
Fourier/Entry ``factor_gradient``, the update, ``row_scores`` /
``entry_scores``, ``draw_samples``, ``variable_density_rows``,
``rebalance``, synthesis and NMSE. Each function cites the reference
file:line it follows.

Third-party arithmetic the reference leans on, restated here and pinned
against the library itself (numpy 2.3.5, in ``oracle/make_golden.py``):
  * numpy.random.Philox (Philox4x64-10, Random123 constants; counter
    pre-increments before every 4-word block) and ``Generator.random``
    (``(u64 >> 11) * 2**-53``);
  * ``Generator.choice(n, size, replace=True, p)`` = searchsorted(right) of
    the uniforms into ``cumsum(p) / cumsum(p)[-1]``.
The FFT (pocketfft) and SVD (LAPACK gesdd) are called through numpy as the
reference does.

Pinning: ``oracle/make_golden.py`` runs every function here against the
reference functions on seeded inputs (agreement to ~1e-12) and writes the
reference's own outputs as fixtures under ``tests/golden/``;
``tests/test_oracle.py`` re-checks the oracle against those fixtures.
"""

from __future__ import annotations

import numpy as np

# ---------------------------------------------------------------------------
# Philox4x64-10 (numpy.random.Philox restated; third-party, numpy 2.3.5)
# ---------------------------------------------------------------------------
_MASK = (1 << 64) - 1
PHILOX_M = (0xD2E7470EE14C6C93, 0xCA5A826395121157)
PHILOX_W = (0x9E3779B97F4A7C15, 0xBB67AE8584CAA73B)


def philox4x64_10(ctr, key):
    """One Philox4x64 block, 10 rounds (Random123 / numpy philox.h)."""
    c = [int(x) & _MASK for x in ctr]
    k0, k1 = int(key[0]) & _MASK, int(key[1]) & _MASK
    for rnd in range(10):
        if rnd:
            k0 = (k0 + PHILOX_W[0]) & _MASK
            k1 = (k1 + PHILOX_W[1]) & _MASK
        p0 = PHILOX_M[0] * c[0]
        p1 = PHILOX_M[1] * c[2]
        hi0, lo0 = p0 >> 64, p0 & _MASK
        hi1, lo1 = p1 >> 64, p1 & _MASK
        c = [hi1 ^ c[1] ^ k0, lo1, hi0 ^ c[3] ^ k1, lo0]
    return c


def philox_words(key, start, count):
    """uint64 words ``start .. start+count-1`` of a fresh ``Philox(key=key)``.

    numpy increments the 256-bit counter *before* producing each block of 4
    words, so word n comes from counter ``n // 4 + 1``, lane ``n % 4``.
    """
    out = np.empty(count, dtype=np.uint64)
    cache_blk, cache = -1, None
    for m in range(count):
        n = start + m
        blk = n // 4 + 1
        if blk != cache_blk:
            cache_blk, cache = blk, philox4x64_10([blk & _MASK, blk >> 64, 0, 0], key)
        out[m] = cache[n % 4]
    return out


def philox_uniforms(key, start, count):
    """``Generator(Philox(key)).random()`` values at stream positions start.."""
    w = philox_words(key, start, count)
    return (w >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def philox_key(seed: int, stream: int = 0):
    """Key words used by the build for ``Philox(key=seed + (stream << 64))``."""
    return (int(seed) & _MASK, int(stream) & _MASK)


# ---------------------------------------------------------------------------
# measurement operators (observation.py)
# ---------------------------------------------------------------------------
def fft_cols(x, inverse=False):
    """Ortho, unshifted 1-D DFT down the columns (observation.py:225-226)."""
    x = np.asarray(x, dtype=np.complex128)
    return np.fft.ifft(x, axis=0, norm="ortho") if inverse else np.fft.fft(x, axis=0, norm="ortho")


def dft2(x, inverse=False):
    """Unitary 2-D DFT (observation.py:171-178)."""
    x = np.asarray(x, dtype=np.complex128)
    return np.fft.ifft2(x, norm="ortho") if inverse else np.fft.fft2(x, norm="ortho")


def rows_to_entries(rows, n2):
    """Full phase-encode lines -> (i, j) pairs, row-major (observation.py:326-332)."""
    rows = np.asarray(rows, dtype=np.int64).ravel()
    return np.column_stack([np.repeat(rows, n2), np.tile(np.arange(n2, dtype=np.int64), rows.size)])


def measurement_factors(A, B, kind):
    """Factors as seen by the sketch: F_x A, F_y B for Fourier masks
    (observation.py:225-226); the factors themselves for entry masks."""
    if kind == "fourier":
        return fft_cols(A), fft_cols(B)
    if kind == "entry":
        return np.asarray(A, np.complex128), np.asarray(B, np.complex128)
    raise TypeError(kind)


def phi_matrix(A, B, idx, kind):
    """Regression matrix Phi[l, r] = Ah[i_l, r] Bh[j_l, r] (observation.py:219-228)."""
    Ah, Bh = measurement_factors(A, B, kind)
    idx = np.asarray(idx, dtype=np.int64).reshape(-1, 2)
    return Ah[idx[:, 0], :] * Bh[idx[:, 1], :]


# ---------------------------------------------------------------------------
# S1: ridge projection (tracker.py:139-156)
# ---------------------------------------------------------------------------
def ridge_svd(phi, y, lam):
    """gamma = V diag(s / (s^2 + lam)) U^H y via the thin SVD (tracker.py:153-156)."""
    phi = np.asarray(phi, dtype=np.complex128)
    y = np.asarray(y, dtype=np.complex128).ravel()
    if phi.shape[0] == 0:
        return np.zeros(phi.shape[1], dtype=np.complex128)
    U, s, Vh = np.linalg.svd(phi, full_matrices=False)
    filt = np.zeros_like(s)
    nz = s > 0
    filt[nz] = s[nz] / (s[nz] ** 2 + lam)
    return Vh.conj().T @ (filt * (U.conj().T @ y))


def ridge_normal(phi, y, lam):
    """(Phi^H Phi + lam I)^-1 Phi^H y — the test oracle of test_tracker.py:74-78."""
    phi = np.asarray(phi, dtype=np.complex128)
    g = phi.conj().T @ phi + lam * np.eye(phi.shape[1])
    return np.linalg.solve(g, phi.conj().T @ np.asarray(y, np.complex128).ravel())


# ---------------------------------------------------------------------------
# S2: gradient data terms (tracker.py:176-228) and curvature (tracker.py:265-364)
# ---------------------------------------------------------------------------
def theta_image(shape, idx, e):
    """Theta = ifft2(scatter(e)) for a Fourier mask (tracker.py:176-188)."""
    xi = np.zeros(shape, dtype=np.complex128)
    idx = np.asarray(idx, dtype=np.int64).reshape(-1, 2)
    xi[idx[:, 0], idx[:, 1]] = e
    return dft2(xi, inverse=True)


def data_terms(A, B, gamma, idx, e, kind):
    """D_m[:, r] = conj(gamma_r) sum_l e_l conj(w_{l,r,m}) (tracker.py:208-228)."""
    A = np.asarray(A, np.complex128)
    B = np.asarray(B, np.complex128)
    gc = np.conj(np.asarray(gamma, np.complex128))
    idx = np.asarray(idx, dtype=np.int64).reshape(-1, 2)
    if kind == "fourier":
        th = theta_image((A.shape[0], B.shape[0]), idx, e)
        return (th @ np.conj(B)) * gc, (th.T @ np.conj(A)) * gc
    if kind == "entry":
        dA = np.zeros_like(A)
        dB = np.zeros_like(B)
        np.add.at(dA, idx[:, 0], e[:, None] * np.conj(B[idx[:, 1], :]))
        np.add.at(dB, idx[:, 1], e[:, None] * np.conj(A[idx[:, 0], :]))
        return dA * gc, dB * gc
    raise TypeError(kind)


def mode_vectors(A, B, idx, kind, mode, r):
    """Rows w_l of the (L, N_mode) contracted-sketch matrix (tracker.py:265-286)."""
    idx = np.asarray(idx, dtype=np.int64).reshape(-1, 2)
    n = (A.shape[0], B.shape[0])
    L = len(idx)
    if kind == "entry":
        other = (B if mode == 0 else A)[:, r]
        coef = other[idx[:, 1 - mode]]
        S = np.zeros((L, n[mode]), dtype=np.complex128)
        S[np.arange(L), idx[:, mode]] = coef
        return S
    F = np.fft.fft(np.eye(n[mode]), axis=0, norm="ortho")
    other = fft_cols((B if mode == 0 else A)[:, r:r + 1])[:, 0]
    return F[:, idx[:, mode]].T * other[idx[:, 1 - mode]][:, None]


def power_top(S, iters=1000, tol=1e-8):
    """Power iteration for lambda_max(sum_l w_l w_l^H) (tracker.py:307-334)."""
    n = S.shape[1]
    if S.shape[0] == 0 or n == 0:
        return 0.0
    g = np.random.default_rng(0x7E5)
    v = g.standard_normal(n) + 1j * g.standard_normal(n)
    v /= np.linalg.norm(v)
    prev = -1.0
    for _ in range(iters):
        w = S.T @ (np.conj(S) @ v)
        nrm = np.linalg.norm(w)
        if nrm == 0.0:
            return 0.0
        v = w / nrm
        cur = float(np.linalg.norm(np.conj(S) @ v) ** 2)
        if prev >= 0 and abs(cur - prev) <= tol * max(cur, 1e-300):
            return cur
        prev = cur
    return prev


def alpha_power(A, B, gamma, idx, kind, lam, t, c_floor=0.0, c_cap=np.inf):
    """hessian_bound by the reference's power method (tracker.py:337-364)."""
    top = 0.0
    for m in (0, 1):
        for r in range(A.shape[1]):
            g2 = float(abs(gamma[r]) ** 2)
            if g2 == 0.0:
                continue
            top = max(top, g2 * power_top(mode_vectors(A, B, idx, kind, m, r)))
    return float(np.clip(lam / t + top, c_floor, c_cap))


def alpha_closed(A, B, gamma, idx, kind, lam, t, c_floor=0.0, c_cap=np.inf):
    """Closed form of the same bound: for Fourier and entry
    masks the per-(m, r) Gram is unitarily similar to a diagonal, so
    lambda_max(G_{0,r}) = max_i sum_{j:(i,j) in Omega} |Bh[j,r]|^2 and the
    mode-2 analogue with Ah. Used where the power method is infeasible."""
    Ah, Bh = measurement_factors(A, B, kind)
    idx = np.asarray(idx, dtype=np.int64).reshape(-1, 2)
    top = 0.0
    for r in range(Ah.shape[1]):
        g2 = float(abs(gamma[r]) ** 2)
        if g2 == 0.0 or len(idx) == 0:
            continue
        c0 = np.zeros(Ah.shape[0])
        np.add.at(c0, idx[:, 0], np.abs(Bh[idx[:, 1], r]) ** 2)
        c1 = np.zeros(Bh.shape[0])
        np.add.at(c1, idx[:, 1], np.abs(Ah[idx[:, 0], r]) ** 2)
        top = max(top, g2 * max(c0.max(), c1.max()))
    return float(np.clip(lam / t + top, c_floor, c_cap))


# ---------------------------------------------------------------------------
# one online step (tracker.py:367-411)
# ---------------------------------------------------------------------------
def track_step(A, B, t, alpha_bar, y, idx, kind, lam, step, power=True):
    """One S1+S2 step on frozen (A, B). ``step`` is ("fixed", mu) or
    ("hessian", c_floor, c_cap). Returns a dict with the new factors and the
    StepReport fields (tracker.py:109-116)."""
    A = np.asarray(A, np.complex128)
    B = np.asarray(B, np.complex128)
    y = np.asarray(y, np.complex128).ravel()
    idx = np.asarray(idx, dtype=np.int64).reshape(-1, 2)
    R = A.shape[1]
    energy = float(np.linalg.norm(A) ** 2 + np.linalg.norm(B) ** 2)
    if len(idx) == 0:  # tracker.py:380-384
        return dict(A=A, B=B, t=t + 1, alpha_bar=alpha_bar, gamma=np.zeros(R, np.complex128),
                    residual=np.zeros(0, np.complex128), cost=0.5 * (lam / t) * energy, mu=0.0)
    phi = phi_matrix(A, B, idx, kind)
    gamma = ridge_svd(phi, y, lam)
    e = y - phi @ gamma
    cost = 0.5 * float(np.linalg.norm(e) ** 2) + 0.5 * (lam / t) * energy  # :389
    if step[0] == "hessian":  # :391-398
        fn = alpha_power if power else alpha_closed
        alpha = fn(A, B, gamma, idx, kind, lam, t, step[1], step[2])
        alpha_bar = alpha_bar + alpha
        mu = 1.0 / alpha_bar
    else:
        mu = float(step[1])
    dA, dB = data_terms(A, B, gamma, idx, e, kind)
    gA = (lam / t) * A - dA  # tracker.py:262
    gB = (lam / t) * B - dB
    return dict(A=A - mu * gA, B=B - mu * gB, t=t + 1, alpha_bar=alpha_bar, gamma=gamma,
                residual=e, cost=cost, mu=mu)


# ---------------------------------------------------------------------------
# sampling policy (sampler.py, observation.py:274-323)
# ---------------------------------------------------------------------------
def _col_normalized_energy(F):
    """sum_r |F[i,r]|^2 / ||f_r||^2 (sampler.py:77-85)."""
    F = np.asarray(F, np.complex128)
    nrm = np.linalg.norm(F, axis=0)
    if (nrm == 0).any():
        raise ValueError("all-zero column; scores undefined")
    return np.sum(np.abs(F / nrm[None, :]) ** 2, axis=1)


def _blend(p, beta):
    """(1 - beta) s + beta / n, renormalised (sampler.py:88-92)."""
    q = (1.0 - beta) * p + beta / p.size
    return q / q.sum()


def row_probs(A, n2, beta=0.1):
    """row_scores (sampler.py:115-128): s(i) = (N2 e_i + R) / (R (N1 + N2))."""
    A = np.asarray(A, np.complex128)
    n1, R = A.shape
    s = (n2 * _col_normalized_energy(A) + R) / (R * (n1 + n2))
    s = s / s.sum()
    return _blend(s, beta)


def entry_probs(A, B, beta=0.1):
    """entry_scores (sampler.py:95-112)."""
    ea, eb = _col_normalized_energy(A), _col_normalized_energy(B)
    R = A.shape[1]
    s = (ea[:, None] + eb[None, :]) / (R * (A.shape[0] + B.shape[0]))
    s = s / s.sum()
    return _blend(s, beta)


def choice_with_replacement(p, size, uniforms):
    """numpy Generator.choice(n, size, replace=True, p) given its uniforms."""
    cdf = np.cumsum(np.asarray(p, np.float64))
    cdf /= cdf[-1]
    return np.searchsorted(cdf, uniforms[:size], side="right").astype(np.int64)


def draw_rows(p, k, forced, key, position):
    """draw_samples(replacement=True) (sampler.py:146-162) on a Philox stream
    at ``position``; returns (sorted unique omega, uniforms consumed)."""
    forced = np.unique(np.asarray([] if forced is None else forced, dtype=np.int64))
    remaining = k - forced.size
    if remaining < 0:
        raise ValueError("more forced indices than trials")
    u = philox_uniforms(key, position, remaining)
    drawn = choice_with_replacement(p, remaining, u) if remaining else np.empty(0, np.int64)
    return np.union1d(forced, drawn).astype(np.int64), remaining


def draw_rows_wor(p, k, forced, key, position):
    """draw_samples(replacement=False) (sampler.py:163-169) on a Philox stream at ``position``: the
    forced indices' weights zeroed, k - |forced| sequential renormalised draws, union with the forced
    ones; returns (sorted unique omega, uniforms consumed)."""
    forced = np.unique(np.asarray([] if forced is None else forced, dtype=np.int64))
    remaining = k - forced.size
    if remaining < 0:
        raise ValueError("more forced indices than trials")
    if k > np.asarray(p).size:
        raise ValueError("cannot draw more distinct indices than the domain holds")
    w = np.asarray(p, np.float64).copy()
    w[forced] = 0.0
    u = iter(philox_uniforms(key, position, remaining))
    drawn = draw_without_replacement(w, remaining, lambda: next(u)) if remaining else np.empty(0, np.int64)
    return np.union1d(forced, drawn).astype(np.int64), remaining


def draw_without_replacement(weights, k, uniform_fn):
    """Sequential renormalised draws (observation.py:279-297)."""
    w = np.asarray(weights, dtype=np.float64).copy()
    if k > np.count_nonzero(w):
        raise ValueError("cannot draw more items than have positive weight")
    out = np.empty(k, dtype=np.int64)
    for n in range(k):
        cdf = np.cumsum(w)
        u = uniform_fn() * cdf[-1]
        i = min(int(np.searchsorted(cdf, u, side="right")), len(w) - 1)
        out[n] = i
        w[i] = 0.0
    return out


def row_distance(n1):
    """|signed frequency| of each unshifted DFT row (observation.py:274-276)."""
    return np.abs(np.fft.fftfreq(n1, d=1.0 / n1)).astype(np.int64)


def vd_rows(n1, alpha, fraction, uniform_fn):
    """variable_density_rows (observation.py:300-323): DC first, then draws
    without replacement with weight d**alpha / 2, in draw order."""
    if not 0.0 < fraction <= 1.0:
        raise ValueError("fraction must be in (0, 1]")
    n_rows = int(np.ceil(fraction * n1))
    d = row_distance(n1)
    w = np.zeros(n1)
    w[d > 0] = d[d > 0].astype(float) ** alpha / 2.0
    rest = draw_without_replacement(w, n_rows - 1, uniform_fn) if n_rows > 1 else np.empty(0, np.int64)
    return np.concatenate([np.zeros(1, np.int64), rest])


# ---------------------------------------------------------------------------
# values (core.py, mri.py, metrics.py)
# ---------------------------------------------------------------------------
def synth(A, B, gamma):
    """A diag(gamma) B^T, plain transpose (core.py:91-104, mri.py:118-119)."""
    return (np.asarray(A, np.complex128) * np.asarray(gamma, np.complex128)[None, :]) @ np.asarray(B, np.complex128).T


def rebalance(A, B):
    """Per-component geometric-mean column norms (core.py:138-166)."""
    A = np.asarray(A, np.complex128)
    B = np.asarray(B, np.complex128)
    na, nb = np.linalg.norm(A, axis=0), np.linalg.norm(B, axis=0)
    dead = (na == 0) & (nb == 0)
    if (((na == 0) | (nb == 0)) & ~dead).any():
        raise ValueError("component zero in some modes but not all")
    g = np.ones_like(na)
    live = ~dead
    g[live] = np.sqrt(na[live] * nb[live])
    sa = np.ones_like(na)
    sb = np.ones_like(nb)
    sa[live] = g[live] / na[live]
    sb[live] = g[live] / nb[live]
    return A * sa[None, :], B * sb[None, :]


def nmse(truth, est):
    """||X - Xh||^2 / ||X||^2 (metrics.py:53-62)."""
    truth = np.asarray(truth, np.complex128)
    return float(np.linalg.norm(truth - np.asarray(est, np.complex128)) ** 2 / np.linalg.norm(truth) ** 2)


def random_subspace(n1, n2, rank, seed, init_scale=1.0):
    """random_subspace (tracker.py:119-126) from default_rng(seed)."""
    g = np.random.default_rng(seed)
    out = []
    for n in (n1, n2):
        z = g.standard_normal((n, rank)) + 1j * g.standard_normal((n, rank))
        out.append((init_scale / np.sqrt(n)) * z / np.sqrt(2.0))
    return out[0], out[1]


# ---------------------------------------------------------------------------
# the online loop (experiment.py:482-530 semantics, Fourier rows, pre-noised)
# ---------------------------------------------------------------------------
def online_run(kspace, A, B, lam, step, policy, clean=None, t0=1, alpha_bar=0.0, power=False,
               record_factors=False):
    """Per frame: [informative: row probabilities from Ah = F_x A (the k-space
    factor, as run_adaptive scores its k-space state, experiment.py:499-505),
    Philox draw with replacement + forced lines]; gather y = K_t[rows, :];
    one Fourier track_step; reconstruct A' diag(gamma) B'^T with the
    post-update factors (experiment.py:525); NMSE against ``clean``.

    ``policy``: {"kind": "static", "rows": [rows_f ...]} or
    {"kind": "informative", "k": K, "forced": [...], "beta": b, "key": (k0, k1),
     "position": 0, "replacement": True} or the run_adaptive schedule (experiment.py:462-497)
    {"kind": "schedule", "vd_frames": V, "alpha": a, "fraction": f, + the informative keys}: the first V
    frames take variable_density_rows (observation.py:300-323, draw order) from the same Philox stream,
    the rest informative draws (with or without replacement, sampler.py:146-169).
    """
    kspace = np.asarray(kspace)
    T, n1, n2 = kspace.shape
    t, pos = t0, int(policy.get("position", 0))
    out = dict(gamma=[], cost=[], mu=[], rows=[], nmse=[], A=[], B=[], probs=[], recon=[])
    for f in range(T):
        if policy["kind"] == "static":
            rows = np.asarray(policy["rows"][f], dtype=np.int64)
        elif policy["kind"] == "schedule" and f < policy["vd_frames"]:
            nr = int(np.ceil(policy["fraction"] * n1))
            u = iter(philox_uniforms(policy["key"], pos, max(nr - 1, 0)))
            rows = vd_rows(n1, policy["alpha"], policy["fraction"], lambda: next(u))
            pos += max(nr - 1, 0)
        else:
            p = row_probs(fft_cols(A), n2, policy.get("beta", 0.1))
            draw = draw_rows if policy.get("replacement", True) else draw_rows_wor
            rows, used = draw(p, policy["k"], policy.get("forced"), policy["key"], pos)
            pos += used
            out["probs"].append(p)
        idx = rows_to_entries(rows, n2)
        y = np.asarray(kspace[f], np.complex128)[rows, :].ravel()
        rep = track_step(A, B, t, alpha_bar, y, idx, "fourier", lam, step, power=power)
        A, B, t, alpha_bar = rep["A"], rep["B"], rep["t"], rep["alpha_bar"]
        X = synth(A, B, rep["gamma"])
        out["gamma"].append(rep["gamma"])
        out["cost"].append(rep["cost"])
        out["mu"].append(rep["mu"])
        out["rows"].append(rows)
        if record_factors:
            out["A"].append(A)
            out["B"].append(B)
        if clean is not None:
            out["nmse"].append(nmse(clean[f], X))
        out["recon"].append(X)
    out["final"] = (A, B, t, alpha_bar, pos)
    return out


def online_run_entries(kspace, Ah, Bh, lam, step, policy, clean=None, t0=1, alpha_bar=0.0, record_factors=False):
    """run_adaptive's entries mode (experiment.py:482-530 with sampler.adaptive_step(domain="entries"),
    sampler.py:190-238) on k-space factors (Ah, Bh) with EntryMask steps (test_mri.py:258-286): per frame
    [entry_scores of (Ah, Bh) (sampler.py:95-112), k trials with replacement over the nx*ny flat entries
    i*ny + j, union with the forced ones (sampler.py:146-162)] or a given entry list; y = K_t at those
    entries; one EntryMask track_step; image = F_x^-1 Ah' diag(gamma) (F_y^-1 Bh')^T with the
    post-update factors. ``policy``: {"kind": "static", "entries": [...]} or {"kind": "informative",
    "k": K, "forced": [...], "beta": b, "key": (k0, k1)}."""
    kspace = np.asarray(kspace)
    T, n1, n2 = kspace.shape
    t, pos = t0, int(policy.get("position", 0))
    out = dict(gamma=[], cost=[], mu=[], entries=[], nmse=[], A=[], B=[], probs=[], recon=[])
    for f in range(T):
        if policy["kind"] == "static":
            om = np.asarray(policy["entries"][f], dtype=np.int64)
        else:
            p = entry_probs(Ah, Bh, policy.get("beta", 0.1)).ravel()
            om, used = draw_rows(p, policy["k"], policy.get("forced"), policy["key"], pos)
            pos += used
            out["probs"].append(p)
        idx = np.stack([om // n2, om % n2], axis=1)
        y = np.asarray(kspace[f], np.complex128).ravel()[om]
        rep = track_step(Ah, Bh, t, alpha_bar, y, idx, "entry", lam, step, power=False)
        Ah, Bh, t, alpha_bar = rep["A"], rep["B"], rep["t"], rep["alpha_bar"]
        X = synth(fft_cols(Ah, inverse=True), fft_cols(Bh, inverse=True), rep["gamma"])
        out["gamma"].append(rep["gamma"])
        out["cost"].append(rep["cost"])
        out["mu"].append(rep["mu"])
        out["entries"].append(om)
        if record_factors:
            out["A"].append(Ah)
            out["B"].append(Bh)
        if clean is not None:
            out["nmse"].append(nmse(clean[f], X))
        out["recon"].append(X)
    out["final"] = (Ah, Bh, t, alpha_bar, pos)
    return out


def batch_run(kspace, A, B, lam, step, rows, epochs, rng=None, reshuffle=False, rebalance_epochs=True, t0=1,
              alpha_bar=0.0):
    """Multi-epoch batch mode (tracker.run tracker.py:456-500, experiment.run_tracking
    experiment.py:284-313) on row masks with FourierMask steps: the frames' data is revisited for
    ``epochs`` passes (rebalance between passes, order re-drawn by ``rng.permutation`` when
    ``reshuffle``, t growing globally); then every frame is re-projected onto the final subspace
    (gamma_t = ridge solve, tracker.py:139-156) when epochs > 1, else the online gammas are kept.
    Returns per-step reports in processing order, the orders, the final gammas and images."""
    kspace = np.asarray(kspace)
    T, n1, n2 = kspace.shape
    data = [(rows_to_entries(np.asarray(r), n2), np.asarray(kspace[f], np.complex128)[np.asarray(r), :].ravel())
            for f, r in enumerate(rows)]
    t, reps, orders, online = t0, [], [], {}
    for epoch in range(epochs):
        if rebalance_epochs and epoch > 0:
            A, B = rebalance(A, B)
        order = np.arange(T)
        if reshuffle and epoch > 0:
            order = rng.permutation(T)
        orders.append(order)
        for k in order:
            idx, y = data[k]
            rep = track_step(A, B, t, alpha_bar, y, idx, "fourier", lam, step, power=False)
            A, B, t, alpha_bar = rep["A"], rep["B"], rep["t"], rep["alpha_bar"]
            reps.append(rep)
            online[int(k)] = rep["gamma"]
    gammas = []
    for f in range(T):
        idx, y = data[f]
        g = ridge_svd(phi_matrix(A, B, idx, "fourier"), y, lam) if epochs > 1 else online[f]
        gammas.append(g)
    recon = [synth(A, B, g) for g in gammas]
    return dict(reports=reps, orders=orders, gamma=gammas, recon=recon, final=(A, B, t, alpha_bar))


# ---------------------------------------------------------------------------
# row-sharded step — decomposition check, k-space form
# ---------------------------------------------------------------------------
def row_shard_partials(Ah, Bh, rows, Y, r0, r1):
    """Partials of one rank owning k-space rows [r0, r1) of Ah (full Ah given
    for convenience; only the owned rows are read). Returns the payload that
    is summed across ranks: W (Ny x R), GA (R x R), ||Y_own||^2, ||Ah_own||^2."""
    rows = np.asarray(rows)
    own = np.flatnonzero((rows >= r0) & (rows < r1))
    As = np.asarray(Ah, np.complex128)[rows[own]]
    Yo = np.asarray(Y, np.complex128)[own]
    W = Yo.T @ np.conj(As)
    GA = As.conj().T @ As
    return dict(W=W, GA=GA, yn=float(np.sum(np.abs(Yo) ** 2)),
                an=float(np.sum(np.abs(np.asarray(Ah, np.complex128)[r0:r1]) ** 2)), own=own)


def row_shard_finish(Ah, Bh, rows, Y, r0, r1, red, lam, t, mu):
    """Given the all-reduced payload `red`, solve redundantly and update the
    owned rows of Ah and the replicated Bh (fixed step). Returns
    (Ah_own_new, Bh_new, gamma, cost)."""
    Ah = np.asarray(Ah, np.complex128)
    Bh = np.asarray(Bh, np.complex128)
    rows = np.asarray(rows)
    own = np.flatnonzero((rows >= r0) & (rows < r1))
    GB = Bh.conj().T @ Bh
    W, GA = red["W"], red["GA"]
    h = np.sum(np.conj(Bh) * W, axis=0)
    R = Ah.shape[1]
    gamma = np.linalg.solve(GA * GB + lam * np.eye(R), h)
    cost = 0.5 * (red["yn"] - float(np.real(np.vdot(gamma, h))) - lam * float(np.vdot(gamma, gamma).real)) \
        + 0.5 * (lam / t) * (red["an"] + float(np.real(np.trace(GB))))
    As = Ah[rows[own]]
    Z = np.asarray(Y, np.complex128)[own] @ np.conj(Bh)
    P = Z - (As * gamma[None, :]) @ GB.T
    Q = W - (Bh * gamma[None, :]) @ GA.T
    c = 1.0 - mu * lam / t
    A_own = c * Ah[r0:r1].copy()
    A_own[rows[own] - r0] += mu * np.conj(gamma)[None, :] * P
    B_new = c * Bh + mu * np.conj(gamma)[None, :] * Q
    return A_own, B_new, gamma, cost


def warm_up(kspace_warm, A, B, lam, step, epochs, t0=1):
    """experiment._warm_up (experiment.py:219-239): `warm_n` fully sampled frames
    tracked for `epochs` passes, rebalanced between passes (core.py:138-166), time
    continuing across passes. Full frames are all rows (Fourier, row-major)."""
    kspace_warm = np.asarray(kspace_warm)
    n1 = kspace_warm.shape[1]
    t, ab = t0, 0.0
    rows = [np.arange(n1)] * kspace_warm.shape[0]
    for epoch in range(epochs):
        if epoch > 0:
            A, B = rebalance(A, B)
        out = online_run(kspace_warm, A, B, lam, step, {"kind": "static", "rows": rows}, t0=t, alpha_bar=ab)
        A, B, t, ab, _ = out["final"]
    return A, B, t, ab


# ---------------------------------------------------------------------------
# per-patch independent trackers (experiment._run_tracking_patched, experiment.py:332-441;
# mri.PatchGrid / patch_partition / patch_assemble, mri.py:48-177)
# ---------------------------------------------------------------------------
def full_entries(shape):
    """All (i, j) of a frame, row-major (experiment.py:139-141)."""
    g = np.meshgrid(*[np.arange(n, dtype=np.int64) for n in shape], indexing="ij")
    return np.stack([x.ravel() for x in g], axis=1)


def patch_split(entries, values, N1, N2, n1, n2):
    """patch_batches' filter (experiment.py:352-370): for patch (p, q) in row-major order, the
    entries inside it in measurement order, shifted to local coordinates, with their values."""
    entries = np.asarray(entries, dtype=np.int64).reshape(-1, 2)
    values = np.asarray(values)
    out = []
    for p in range(N1 // n1):
        for q in range(N2 // n2):
            inside = ((entries[:, 0] >= p * n1) & (entries[:, 0] < (p + 1) * n1)
                      & (entries[:, 1] >= q * n2) & (entries[:, 1] < (q + 1) * n2))
            out.append((entries[inside] - np.array([p * n1, q * n2]), values[inside]))
    return out


def patch_assemble(tiles, N1, N2, n1, n2):
    """Inverse of the row-major tiling (mri.py:165-177)."""
    out = np.empty((N1, N2), dtype=np.result_type(*[np.asarray(t).dtype for t in tiles]))
    k2 = N2 // n2
    for k, tile in enumerate(tiles):
        p, q = divmod(k, k2)
        out[p * n1:(p + 1) * n1, q * n2:(q + 1) * n2] = tile
    return out


def patched_run(frames, A0s, B0s, lam, step, n1, n2, entries, warm_n, warm_epochs, epochs, rng=None,
                reshuffle=False, power=True):
    """_run_tracking_patched (experiment.py:332-441) on pre-noised frames (frames leading,
    (T, N1, N2)): one EntryMask tracker of rank rho per n1 x n2 patch, started from (A0s[p], B0s[p]);
    ``entries[t]`` the frame's global (i, j) list (the warm frames' are the full frame). Warm-up:
    ``warm_epochs`` passes over the warm frames, every patch rebalanced at the start of each pass
    after the first; then ``epochs`` passes over the remaining frames (all patches rebalanced
    between passes, order re-drawn by ``rng.permutation`` when ``reshuffle``); then every frame,
    warm ones included, is re-projected onto each patch's final subspace (ridge solve) and the tiles
    assembled. Returns the trace (per main step: gamma and residual concatenated over patches, cost
    summed, patch 0's step size and the pre-step t, as StepReport carries it, tracker.py:409), the
    reconstruction (T, N1, N2) and the final factors. ``power`` picks the reference's power method for
    the HessianBound step (else the closed form the device uses)."""
    frames = np.asarray(frames)
    T, N1, N2 = frames.shape
    npatch = (N1 // n1) * (N2 // n2)
    states = [[np.asarray(A0s[p], np.complex128), np.asarray(B0s[p], np.complex128), 1, 0.0] for p in range(npatch)]
    batches = [patch_split(entries[t], np.asarray(frames[t], np.complex128)[tuple(np.asarray(entries[t]).reshape(-1, 2).T)],
                           N1, N2, n1, n2) for t in range(T)]

    def step_patch(p, t):
        A, B, tt, ab = states[p]
        idx, y = batches[t][p]
        rep = track_step(A, B, tt, ab, y, idx, "entry", lam, step, power=power)
        states[p] = [rep["A"], rep["B"], rep["t"], rep["alpha_bar"]]
        return rep

    def rebalance_patch(p):
        A, B = rebalance(states[p][0], states[p][1])
        states[p][0], states[p][1] = A, B

    for epoch in range(warm_epochs):
        for t in range(warm_n):
            for p in range(npatch):
                if epoch > 0 and t == 0:
                    rebalance_patch(p)
                step_patch(p, t)
    trace, orders = [], []
    for epoch in range(epochs):
        if epoch > 0:
            for p in range(npatch):
                rebalance_patch(p)
        order = list(range(warm_n, T))
        if reshuffle and epoch > 0:
            order = [warm_n + int(i) for i in rng.permutation(T - warm_n)]
        orders.append(order)
        for t in order:
            reps = [step_patch(p, t) for p in range(npatch)]
            trace.append(dict(gamma=np.concatenate([r["gamma"] for r in reps]),
                              residual=np.concatenate([r["residual"] for r in reps]),
                              cost=float(sum(r["cost"] for r in reps)), mu=reps[0]["mu"], t=reps[0]["t"] - 1,
                              patch_gamma=np.stack([r["gamma"] for r in reps]),
                              patch_cost=np.array([r["cost"] for r in reps])))
    recon = np.zeros((T, N1, N2), np.complex128)
    gammas = np.zeros((T, npatch, A0s[0].shape[1]), np.complex128)
    for t in range(T):
        tiles = []
        for p in range(npatch):
            idx, y = batches[t][p]
            A, B = states[p][0], states[p][1]
            g = ridge_svd(phi_matrix(A, B, idx, "entry"), y, lam)
            gammas[t, p] = g
            tiles.append(synth(A, B, g))
        recon[t] = patch_assemble(tiles, N1, N2, n1, n2)
    return dict(trace=trace, orders=orders, recon=recon, gamma=gammas,
                final=[(s[0], s[1], s[2], s[3]) for s in states])
