"""GPU parity of the sampling policy: fp64 score kernels against the
reference's golden scores (1e-12), and bit-exact Philox draws (with and
without replacement) against numpy / the reference for the same
probabilities."""

import numpy as np
import pytest

from conftest import load_golden, rel

pytestmark = pytest.mark.gpu
G = load_golden("sampling_cases")


def test_row_and_entry_scores_match_reference_golden():
    import paper_1609_04104_b200 as tt

    for c in range(int(G["nscores"])):
        A, B, beta = G[f"s{c}__A"], G[f"s{c}__B"], float(G[f"s{c}__beta"])
        # fp64 arithmetic on fp32-rounded factors: compare to the oracle on the same rounded inputs
        from oracle import tt_oracle as O

        A32, B32 = A.astype(np.complex64), B.astype(np.complex64)
        sub = tt.TensorSubspace((A32, B32))
        rs = tt.row_scores(sub, beta).scores
        es = tt.entry_scores(sub, beta).scores
        assert rel(rs, O.row_probs(A32, B.shape[0], beta)) < 1e-12
        assert rel(es, O.entry_probs(A32, B32, beta)) < 1e-12
        # and to the reference's fp64 scores to fp32 input precision
        assert rel(rs, G[f"s{c}__rows"]) < 1e-6


def test_zero_column_rejected():
    import paper_1609_04104_b200 as tt

    f1 = np.ones((4, 2), dtype=complex)
    f1[:, 1] = 0.0
    with pytest.raises(ValueError):
        tt.row_scores(tt.TensorSubspace((f1, np.ones((3, 2), complex))))


def test_draw_with_replacement_bit_exact_with_reference():
    import paper_1609_04104_b200 as tt

    for c in range(int(G["ndraws"])):
        p, k = G[f"d{c}__p"], int(G[f"d{c}__k"])
        forced = G[f"d{c}__forced"]
        key = tuple(int(v) for v in G[f"d{c}__key"])
        gen = np.random.Generator(np.random.Philox(key=key[0] + (key[1] << 64)))
        dist = tt.SamplingDistribution(p, "rows")
        for rep in range(3):  # the stream continues across frames
            plan = tt.draw_samples(dist, k, True, gen, forced=forced if forced.size else None)
            np.testing.assert_array_equal(plan.omega, G[f"d{c}__omega{rep}"])


def test_draw_matches_numpy_choice_many_seeds():
    import paper_1609_04104_b200 as tt

    rng = np.random.default_rng(7)
    for trial in range(40):
        n = int(rng.integers(2, 1500))
        p = rng.random(n) ** 6 + (0 if trial % 3 else 1e-300)
        p /= p.sum()
        key = int(rng.integers(1 << 63))
        k = int(rng.integers(1, min(n, 400) + 1))
        g1 = np.random.Generator(np.random.Philox(key=key))
        g2 = np.random.Generator(np.random.Philox(key=key))
        g1.random(int(rng.integers(0, 7)))  # arbitrary start position
        g2.bit_generator.state = g1.bit_generator.state
        want = np.union1d(np.empty(0, np.int64), g1.choice(n, size=k, replace=True, p=p))
        plan = tt.draw_samples(tt.SamplingDistribution(p, "rows"), k, True, g2)
        np.testing.assert_array_equal(plan.omega, want)
        assert g1.random() == g2.random()  # host generator advanced in step


def test_without_replacement_and_vd_rows_bit_exact():
    import paper_1609_04104_b200 as tt

    for c in range(int(G["nvd"])):
        key = tuple(int(v) for v in G[f"v{c}__key"])
        gen = np.random.Generator(np.random.Philox(key=key[0] + (key[1] << 64)))
        rows = tt.variable_density_rows(int(G[f"v{c}__n1"]), float(G[f"v{c}__alpha"]), float(G[f"v{c}__frac"]), gen)
        np.testing.assert_array_equal(rows, G[f"v{c}__rows"])
    gen = np.random.Generator(np.random.Philox(key=3))
    plan = tt.draw_samples(tt.SamplingDistribution(np.full(30, 1 / 30), "rows"), 12, False, gen)
    assert plan.size == 12 and len(np.unique(plan.omega)) == 12
    plan = tt.draw_samples(tt.SamplingDistribution(np.full(10, 0.1), "rows"), 4, False, gen, forced=[0, 5])
    assert plan.size == 4 and {0, 5} <= set(plan.omega.tolist())


def test_point_mass_and_trial_count_edges():
    import paper_1609_04104_b200 as tt

    s = np.zeros(20)
    s[7] = 1.0
    plan = tt.draw_samples(tt.SamplingDistribution(s, "rows"), 50, True, np.random.Generator(np.random.Philox(0)))
    assert plan.omega.tolist() == [7]
    d = tt.SamplingDistribution(np.full(5, 0.2), "rows")
    with pytest.raises(ValueError):
        tt.draw_samples(d, 0, True, np.random.Generator(np.random.Philox(0)))
    with pytest.raises(ValueError):
        tt.draw_samples(d, 6, False, np.random.Generator(np.random.Philox(0)))


def _ref_draw_samples(flat, k, replacement, rng, forced=None):
    """draw_samples (sampler.py:131-170) restated in the test: numpy's own choice / sequential draws."""
    from oracle import tt_oracle as O

    forced_idx = np.unique(np.asarray([] if forced is None else forced, dtype=np.int64))
    remaining = k - forced_idx.size
    if replacement:
        drawn = rng.choice(flat.size, size=remaining, replace=True, p=flat) if remaining else np.empty(0, np.int64)
        return np.union1d(forced_idx, drawn)
    w = flat.copy()
    w[forced_idx] = 0.0
    return np.union1d(forced_idx, O.draw_without_replacement(w, remaining, rng.random))


@pytest.mark.parametrize("bitgen", ["pcg64", "mt19937", "sfc64"])
def test_draws_with_any_bit_generator(bitgen):
    """np.random.default_rng(seed) (PCG64) is how the reference builds every generator
    (experiment.py:257,338,453): the device draws take their uniforms from the host generator and
    equal numpy's draws; the generator ends in the same state as after numpy's own calls."""
    import paper_1609_04104_b200 as tt

    mk = {"pcg64": np.random.PCG64, "mt19937": np.random.MT19937, "sfc64": np.random.SFC64}[bitgen]
    rng = np.random.default_rng(11)
    for trial in range(12):
        n = int(rng.integers(3, 900))
        p = rng.random(n) ** 4
        p /= p.sum()
        k = int(rng.integers(2, min(n, 200)))
        forced = [0, n - 1] if trial % 2 else None
        seed = int(rng.integers(1 << 62))
        for replacement in (True, False):
            g1, g2 = np.random.Generator(mk(seed)), np.random.Generator(mk(seed))
            want = _ref_draw_samples(p, k, replacement, g1, forced)
            plan = tt.draw_samples(tt.SamplingDistribution(p, "rows"), k, replacement, g2, forced=forced)
            np.testing.assert_array_equal(plan.omega, want)
            assert g1.random() == g2.random()
    # variable-density rows (observation.py:300-323) and the bare sequential draw
    for seed in range(5):
        g1, g2 = np.random.default_rng(seed), np.random.default_rng(seed)
        from oracle import tt_oracle as O

        want = O.vd_rows(256, -1.0, 0.25, g1.random)
        np.testing.assert_array_equal(tt.variable_density_rows(256, -1.0, 0.25, g2), want)
        assert g1.random() == g2.random()


def test_large_domain_draw_with_host_uniforms():
    """Entry-domain draws (beyond one CTA) with a PCG64 generator: numpy choice semantics."""
    import paper_1609_04104_b200 as tt

    rng = np.random.default_rng(3)
    n = 128 * 96
    p = rng.random(n) ** 3
    p /= p.sum()
    g1, g2 = np.random.default_rng(99), np.random.default_rng(99)
    want = np.union1d([5], g1.choice(n, size=799, replace=True, p=p))
    plan = tt.draw_samples(tt.SamplingDistribution(p.reshape(128, 96), "entries"), 800, True, g2, forced=[5])
    np.testing.assert_array_equal(plan.omega, want)


def test_scores_of_a_fourier_tracked_subspace_use_image_factors():
    """row_scores / entry_scores always score subspace.factors (sampler.py:77-85), even for a subspace
    the tracker produced on the device from a FourierMask step."""
    import paper_1609_04104_b200 as tt
    from oracle import tt_oracle as O

    rng = np.random.default_rng(4)
    n1, n2, R = 48, 40, 5
    A, B = O.random_subspace(n1, n2, R, seed=6)
    idx = np.argwhere(rng.random((n1, n2)) < 0.3)
    y = rng.standard_normal(len(idx)) + 1j * rng.standard_normal(len(idx))
    st = tt.TrackerState(tt.TensorSubspace((A, B)), tt.StepConfig(0.1, R, tt.Fixed(0.05)))
    new, _ = tt.track_step(st, tt.MeasurementBatch(y, tt.FourierMask((n1, n2), idx)))
    Ah, Bh = (f.astype(np.complex64) for f in new.subspace.factors)
    assert rel(tt.row_scores(new.subspace).scores, O.row_probs(Ah, n2, 0.1)) < 1e-9
    assert rel(tt.entry_scores(new.subspace).scores, O.entry_probs(Ah, Bh, 0.1)) < 1e-9
    # the same values as a host-built subspace of the same factors
    host = tt.TensorSubspace(new.subspace.factors)
    assert rel(tt.row_scores(new.subspace).scores, tt.row_scores(host).scores) < 1e-12


def test_subspace_from_device_tensors_stays_on_device():
    import torch

    import paper_1609_04104_b200 as tt

    a = torch.randn(20, 3, dtype=torch.complex64, device="cuda")
    b = torch.randn(16, 3, dtype=torch.complex64, device="cuda")
    sub = tt.TensorSubspace((a, b))
    assert sub._host is None and sub.dims == (20, 16) and sub.rank == 3
    a.zero_()  # constructed values are copies (core.py:6-7)
    fa, fb = sub.torch_factors()
    assert float(fa.abs().sum()) > 0 and fb.is_cuda
    np.testing.assert_allclose(sub.factors[1], b.cpu().numpy(), rtol=0, atol=0)
    with pytest.raises(ValueError):
        tt.TensorSubspace((a, torch.zeros(5, 2, dtype=torch.complex64, device="cuda")))
