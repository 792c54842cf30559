"""CTEN container I/O (cten.py:1-74) through the native C ABI against files written by the
reference's own writer (tests/golden/cten, made by oracle/make_golden_cten.py). Host-only."""

import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden", "cten")
CASES = ["f64_2x3", "f32_vec", "f64_3d", "f64_special", "f32_special", "scalar", "empty"]
BAD = ["bad_magic", "bad_version", "bad_dtype", "truncated_dims", "short_payload", "long_payload", "tiny"]


@pytest.fixture(scope="module")
def gold():
    return np.load(os.path.join(GOLD, "cases.npz"))


@pytest.mark.parametrize("name", CASES)
def test_reads_reference_files_bit_exactly(gold, name):
    from paper_1609_04104_b200 import cten

    got = cten.read_cten(os.path.join(GOLD, name + ".cten"))
    want = gold[name]
    assert got.dtype == np.complex128 and got.shape == want.shape
    assert got.view(np.float64).tobytes() == want.view(np.float64).tobytes()


@pytest.mark.parametrize("name", CASES)
def test_writes_reference_bytes(gold, tmp_path, name):
    from paper_1609_04104_b200 import cten

    p = tmp_path / "x.cten"
    cten.write_cten(p, gold[name + "__src"], int(gold[name + "__code"]))
    assert p.read_bytes() == open(os.path.join(GOLD, name + ".cten"), "rb").read()


def test_reference_nonfinite_imag_quirk(gold):
    from paper_1609_04104_b200 import cten

    got = cten.read_cten(os.path.join(GOLD, "raw_nonfinite.cten"))
    want = gold["raw_nonfinite"]
    np.testing.assert_array_equal(np.isnan(got.real), np.isnan(want.real))
    np.testing.assert_array_equal(got[~np.isnan(want.real)], want[~np.isnan(want.real)])


@pytest.mark.parametrize("name", BAD)
def test_malformed_files_raise(name):
    from paper_1609_04104_b200 import cten

    with pytest.raises(cten.CtenFormatError):
        cten.read_cten(os.path.join(GOLD, name + ".cten"))
    assert issubclass(cten.CtenFormatError, ValueError)


def test_tensor_loader_and_errors(tmp_path):
    from paper_1609_04104_b200 import cten

    rng = np.random.default_rng(9)
    x = rng.standard_normal((4, 6, 5)) + 1j * rng.standard_normal((4, 6, 5))
    for code in (0, 1):
        p = tmp_path / f"t{code}.cten"
        cten.write_cten(p, x, code)
        assert cten.cten_info(p) == (code, (4, 6, 5))
        t = cten.read_cten_tensor(p, pin=False)
        np.testing.assert_array_equal(t.numpy(), x.astype(np.complex64))
    with pytest.raises(FileNotFoundError):
        cten.read_cten(tmp_path / "missing.cten")
    with pytest.raises(cten.CtenFormatError):
        cten.write_cten(tmp_path / "y.cten", x, 3)
