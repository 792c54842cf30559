"""Golden CTEN files written by the reference's own writer (cten.py:33-46).

Test infrastructure only: run in the build container (where /root/reference
exists); the files and the expected arrays are committed under
tests/golden/cten/ and the GPU box never needs the reference. The malformed
variants are the ones the reference's read_cten rejects (cten.py:49-74).
"""

from __future__ import annotations

import importlib
import os
import sys
import types

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_PKG = "/root/reference/pkg/src/tensortrack"
OUT = os.path.join(HERE, "..", "tests", "golden", "cten")


def main():
    if "tensortrack" not in sys.modules:
        pkg = types.ModuleType("tensortrack")
        pkg.__path__ = [REF_PKG]
        sys.modules["tensortrack"] = pkg
    cten = importlib.import_module("tensortrack.cten")
    os.makedirs(OUT, exist_ok=True)
    rng = np.random.default_rng(20240917)
    special = np.array([0.0, -0.0, 1e-310, -np.inf, np.inf, 1.5, -2.25, 3.4e38, 1e-45], dtype=np.float64)
    cases = {
        "f64_2x3": (rng.standard_normal((2, 3)) + 1j * rng.standard_normal((2, 3)), 1),
        "f32_vec": (rng.standard_normal(7) - 1j * rng.standard_normal(7), 0),
        "f64_3d": (rng.standard_normal((2, 3, 4)) + 1j * rng.standard_normal((2, 3, 4)), 1),
        "f64_special": (special + 1j * special[::-1], 1),
        "f32_special": (special + 1j * special[::-1], 0),
        "scalar": (np.array(2.5 - 0.5j), 1),
        "empty": (np.zeros((0, 5), dtype=np.complex128), 0),
    }
    arrays = {}
    for name, (arr, code) in cases.items():
        path = os.path.join(OUT, name + ".cten")
        cten.write_cten(path, arr, code)
        arrays[name] = cten.read_cten(path)  # what the reference reads back
        arrays[name + "__src"] = np.asarray(arr, dtype=np.complex128)
        arrays[name + "__code"] = np.array(code)
    # raw pairs (finite real, non-finite imaginary) written byte by byte: the reference reader's
    # real + 1j * imag assembly (cten.py:72-73) turns those real parts into NaN
    raw = np.array([[1.0, np.inf], [2.0, -np.inf], [3.0, np.nan], [4.0, 5.0]], dtype="<f8")
    path = os.path.join(OUT, "raw_nonfinite.cten")
    with open(path, "wb") as fh:
        fh.write(b"CTEN" + bytes([1, 1, 1]) + (4).to_bytes(4, "little") + raw.tobytes())
    arrays["raw_nonfinite"] = cten.read_cten(path)
    good = open(os.path.join(OUT, "f64_2x3.cten"), "rb").read()
    bad = {
        "bad_magic": b"CTEM" + good[4:],
        "bad_version": good[:4] + bytes([2]) + good[5:],
        "bad_dtype": good[:5] + bytes([7]) + good[6:],
        "truncated_dims": good[:9],
        "short_payload": good[:-3],
        "long_payload": good + b"\x00",
        "tiny": b"CTE",
    }
    for name, blob in bad.items():
        path = os.path.join(OUT, name + ".cten")
        with open(path, "wb") as fh:
            fh.write(blob)
        try:
            cten.read_cten(path)
        except cten.CtenFormatError:
            continue
        raise AssertionError(f"reference accepted {name}")
    np.savez(os.path.join(OUT, "cases.npz"), **arrays)
    print(f"wrote {len(cases)} golden and {len(bad)} malformed CTEN files to {OUT}")


if __name__ == "__main__":
    main()
