"""CTEN I/O throughput: the native C reader/writer behind paper_1609_04104_b200.cten
vs the reference's numpy implementation (cten.py:32-74), same file, host only. Runs in the build
container (imports the reference from /root/reference for the comparison; test/measurement use only).
Usage: python profiles/tools/cten_io_bench.py"""

import importlib
import os
import sys
import tempfile
import time
import types

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import paper_1609_04104_b200 as tt  # noqa: E402

REF = "/root/reference/pkg/src/tensortrack"


def best(fn, reps=3):
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return min(ts)


def main():
    pkg = types.ModuleType("tensortrack")
    pkg.__path__ = [REF]
    sys.modules.setdefault("tensortrack", pkg)
    ref = importlib.import_module("tensortrack.cten")
    rng = np.random.default_rng(0)
    x = (rng.standard_normal((256, 256, 200)) + 1j * rng.standard_normal((256, 256, 200))).astype(np.complex128)
    mb = x.size * 16 / 1e6  # complex128 payload as both sides store it (dtype code 1)
    with tempfile.TemporaryDirectory() as d:
        pa, pb = os.path.join(d, "a.cten"), os.path.join(d, "b.cten")
        w_ref = best(lambda: ref.write_cten(pa, x))
        w_our = best(lambda: tt.write_cten(pb, x))
        assert open(pa, "rb").read() == open(pb, "rb").read()  # byte-identical files
        r_ref = best(lambda: ref.read_cten(pa))
        r_our = best(lambda: tt.read_cten(pa))
        np.testing.assert_array_equal(ref.read_cten(pa), tt.read_cten(pa))
    print(f"payload {mb:.0f} MB (complex128)")
    print(f"write: reference {mb / w_ref:.0f} MB/s, ours {mb / w_our:.0f} MB/s")
    print(f"read:  reference {mb / r_ref:.0f} MB/s, ours {mb / r_our:.0f} MB/s")


if __name__ == "__main__":
    main()
