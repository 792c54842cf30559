"""GPU parity of the entry-mask online loop (run_adaptive's entries mode on
k-space factors) and of the large-domain draw it uses, against the oracle / numpy semantics."""

import numpy as np
import pytest

from conftest import rel
from oracle import tt_oracle as O

pytestmark = pytest.mark.gpu


def _probs(n, seed):
    rng = np.random.default_rng(seed)
    p = rng.gamma(0.7, size=n)
    p[rng.integers(0, n, n // 50)] *= 40.0  # a few heavy entries
    return p / p.sum()


@pytest.mark.parametrize("force_exact", [False, True])
@pytest.mark.parametrize("n,k,nforced", [(65536, 16384, 16), (40000, 3000, 0), (20000, 1, 1), (100000, 50000, 7)])
def test_large_domain_draw_matches_numpy_choice(n, k, nforced, force_exact, monkeypatch):
    """tt_draw_with_replacement_large == Generator(Philox(key)).choice(n, k - |forced|, p) U forced, bit for bit,
    and the stream position advances by the draws consumed (sampler.py:146-162)."""
    import torch
    from paper_1609_04104_b200 import _lib as L

    if force_exact:  # every uniform counts as ambiguous: numpy's sequential cumsum path
        monkeypatch.setenv("TT_DRAW_FORCE_EXACT", "1")
    p = _probs(n, n + k)
    rng = np.random.default_rng(5)
    forced = np.sort(rng.choice(n, nforced, replace=False)).astype(np.int64)
    key = (2024, 3)
    dev = L.device()
    pd = torch.from_numpy(p).to(dev)
    fd = torch.from_numpy(forced.astype(np.int32)).to(dev)
    pos = torch.zeros(1, dtype=torch.int64, device=dev)
    om = torch.empty(k, dtype=torch.int32, device=dev)
    cnt = torch.zeros(1, dtype=torch.int32, device=dev)
    scr = torch.zeros(int(L.lib().tt_draw_scratch_bytes(n)), dtype=torch.uint8, device=dev)
    position = 0
    for call in range(2):  # the second call continues the stream
        L.check(L.lib().tt_draw_with_replacement_large(L.stream_ptr(), n, pd.data_ptr(), k,
                                                       fd.data_ptr() if nforced else None, nforced, key[0], key[1],
                                                       pos.data_ptr(), om.data_ptr(), cnt.data_ptr(),
                                                       scr.data_ptr()), "draw")
        want, used = O.draw_rows(p, k, forced, key, position)
        position += used
        c = int(cnt.item())
        np.testing.assert_array_equal(om[:c].cpu().numpy(), want)
        assert int(pos.item()) == position


def _entry_case(n=32, R=4, T=7, seed=41):
    from paper_1609_04104_b200.phantom import cine_phantom

    ph = cine_phantom(n, n, T, period=8.0, seed=seed)
    A0, B0 = O.random_subspace(n, n, R, seed=seed + 1)
    return ph, A0, B0


def test_static_entry_engine_matches_oracle():
    """Oracle entry lists fed in (BASELINE: "otherwise oracle masks are fed in"), in measurement
    order: per-frame gamma within 1e-4, final factors, NRMSE trajectory within 1e-3."""
    import paper_1609_04104_b200 as tt

    n, R, T, lam = 32, 4, 7, 0.1
    ph, A0, B0 = _entry_case(n, R, T)
    rng = np.random.default_rng(7)
    lists = [rng.permutation(rng.choice(n * n, int(0.3 * n * n), replace=False)) for _ in range(T)]
    Ah0, Bh0 = O.fft_cols(A0), O.fft_cols(B0)
    ref = O.online_run_entries(ph.kspace, Ah0, Bh0, lam, ("fixed", 0.01), {"kind": "static", "entries": lists},
                               clean=ph.clean, record_factors=True)
    S = max(len(x) for x in lists)
    tab = np.full((T, S), -1, np.int64)
    for f, x in enumerate(lists):
        tab[f, :len(x)] = x
    res = tt.run_online(ph.kspace, A0[None], B0[None], lam, tt.Fixed(0.01),
                        tt.StaticEntries(tab, np.array([len(x) for x in lists])), clean=ph.clean)
    for f in range(T):
        assert rel(res.gamma[f, 0], ref["gamma"][f]) < 1e-4, f
    assert rel(res.final_A[0], O.fft_cols(ref["A"][-1], inverse=True)) < 1e-4
    assert np.max(np.abs(np.sqrt(res.nmse[:, 0]) - np.sqrt(np.array(ref["nmse"])))) < 1e-3
    assert rel(res.recon[-1, 0], ref["recon"][-1]) < 1e-4


def test_informative_entry_engine_draws_are_numpy_choice_of_its_scores():
    """Each frame's entry set equals numpy choice over the engine's own entry scores of the previous
    frame's factors (bit-exact draw inside the loop), plus forced entries; graph replay == eager."""
    import torch
    import paper_1609_04104_b200 as tt
    from paper_1609_04104_b200 import _ops as K

    n, R, T, lam = 32, 4, 7, 0.1
    ph, A0, B0 = _entry_case(n, R, T)
    forced = (0, 1, n, n * n - 1)
    pol = tt.InformativeEntries(k=300, forced=forced, beta=0.1, key0=11, key1=2)
    runs = []
    for graph in (True, False):
        eng = tt.EntryEngine(n, n, R, lam, tt.Fixed(0.01), pol)
        eng.set_image_factors(A0, B0)
        kd = torch.from_numpy(ph.kspace.astype(np.complex64)).cuda()
        out = eng.run(kd, T, graph=graph)
        runs.append({k: v.cpu().numpy() for k, v in out.items()})
    for k in runs[0]:
        np.testing.assert_array_equal(runs[0][k], runs[1][k])
    out = runs[0]
    ah_prev = torch.from_numpy(O.fft_cols(A0).astype(np.complex64)).cuda()
    bh_prev = torch.from_numpy(O.fft_cols(B0).astype(np.complex64)).cuda()
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    position = 0
    for f in range(T):
        p = K.entry_scores(ah_prev, bh_prev, 0.1, st).cpu().numpy().ravel()
        want, used = O.draw_rows(p, 300, np.array(forced), (11, 2), position)
        position += used
        got = out["rows"][f, 0, :out["cnt"][f, 0]]
        np.testing.assert_array_equal(got, want)
        ah_prev = torch.from_numpy(out["ah"][f, 0]).cuda()
        bh_prev = torch.from_numpy(out["bh"][f, 0]).cuda()
    # the probabilities themselves track the oracle's (fp32 factors vs complex128: ~1e-7)
    p0 = K.entry_scores(torch.from_numpy(O.fft_cols(A0).astype(np.complex64)).cuda(),
                        torch.from_numpy(O.fft_cols(B0).astype(np.complex64)).cuda(), 0.1, st).cpu().numpy().ravel()
    assert rel(p0, O.entry_probs(O.fft_cols(A0), O.fft_cols(B0), 0.1).ravel()) < 1e-5


def test_run_online_informative_entries_end_to_end():
    import paper_1609_04104_b200 as tt

    n, R, T = 32, 4, 9
    ph, A0, B0 = _entry_case(n, R, T, seed=51)
    res = tt.run_online(ph.kspace, A0[None], B0[None], 0.1, tt.Fixed(0.01),
                        tt.InformativeEntries(k=320, forced=(0,), key0=3), clean=ph.clean)
    assert res.recon.shape == (T, 1, n, n) and res.gamma.shape == (T, 1, R)
    assert all(len(r[0]) <= 320 and 0 in r[0] for r in res.rows)
    assert np.all(np.isfinite(res.nmse)) and res.nmse[-1, 0] < res.nmse[0, 0]
    with pytest.raises(ValueError):
        tt.run_online(ph.kspace, A0[None], B0[None], 0.1, tt.Fixed(0.01),
                      tt.InformativeEntries(k=2, forced=(0, 1, 2)))


def test_run_online_entries_plan_cache_reuse():
    """A repeated run_online call with the same shapes/policy replays the cached frame graph on freshly
    uploaded data: results equal a fresh eager engine run on that data, bit for bit."""
    import torch
    import paper_1609_04104_b200 as tt
    from paper_1609_04104_b200 import engine as E
    from paper_1609_04104_b200.phantom import cine_phantom

    n, R, T = 32, 4, 6
    pol = tt.InformativeEntries(k=200, forced=(0,), key0=12)
    A0, B0 = O.random_subspace(n, n, R, seed=91)
    E._ENTRY_PLANS.clear()
    for seed in (92, 93, 92):  # miss, hit with other data, hit
        ph = cine_phantom(n, n, T, period=8.0, seed=seed)
        got = tt.run_online(ph.kspace, A0[None], B0[None], 0.1, tt.Fixed(0.01), pol)
        eng = tt.EntryEngine(n, n, R, 0.1, tt.Fixed(0.01), pol)
        eng.set_image_factors(A0, B0)
        out = eng.run(torch.from_numpy(ph.kspace.astype(np.complex64)).cuda(), T, graph=False)
        np.testing.assert_array_equal(got.gamma, out["gamma"].cpu().numpy())
        np.testing.assert_array_equal(got.recon, eng.reconstruct(out).cpu().numpy())
    assert len(E._ENTRY_PLANS) == 1
