"""The large-domain draw's ambiguity bound (csrc/tt_sample.cu big_bound) against exact arithmetic:
numpy's normalised sequential cumsum c_i = cumsum(p)[i] / cumsum(p)[-1] (the CDF numpy's
Generator.choice searches, sampler.py:146-162) stays within u x_i (i (1 - x_i) + n - i + 1) of the exact
prefix fraction x_i at every index, for flat, heavy-tailed and front/back-loaded distributions.
A draw farther than this bound (plus our scan's own depth term) from both bucket edges therefore
lands where numpy's does; nearer ones take the exact sequential path."""

from fractions import Fraction

import numpy as np
import pytest

U = 2.0 ** -53


def _bound(x, n):
    i = np.arange(n)
    return 1.05 * U * (x * (i * (1 - x) + (n - i) + 1))


@pytest.mark.parametrize("kind", ["gamma", "heavy", "front", "back"])
def test_sequential_cumsum_error_within_bound(kind):
    n = 12000
    rng = np.random.default_rng(len(kind))
    p = rng.gamma(0.7, size=n)
    if kind == "heavy":
        p[rng.integers(0, n, n // 50)] *= 40
    if kind == "front":
        p[: n // 100] *= 1e4
    if kind == "back":
        p[-n // 100:] *= 1e4
    p /= p.sum()
    c = np.cumsum(p)
    c = c / c[-1]
    s = Fraction(0)
    pref = []
    for v in p:
        s += Fraction(float(v))
        pref.append(s)
    x = np.array([float(q / s) for q in pref])
    assert np.all(np.abs(c - x) <= _bound(x, n))
