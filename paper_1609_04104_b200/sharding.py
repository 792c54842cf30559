"""Work partitioning across ranks (one process per GPU).

* Slice sharding (BASELINE config 3): independent slices, contiguous blocks
  per rank, no data-path collective.
* Row sharding (config 4): rank r owns a contiguous block of k-space rows of
  Ah (B̂ replicated). Per frame, the partial sums of GA = Ah_S^H Ah_S,
  W = Y^T conj(Ah_S), ||Y||^2 and the Ah column norms are summed across ranks
  (one all-reduce of `row_shard_payload_len` complex values), after which
  every rank solves the R x R ridge system redundantly and updates its own
  rows plus the replicated Bh identically.
"""

from __future__ import annotations


import numpy as np

__all__ = ["block_range", "slice_partition", "row_partition", "row_shard_payload_len", "payload_doubles",
           "pack_payload", "unpack_payload", "packed_index"]


def block_range(n: int, parts: int, p: int) -> tuple[int, int]:
    """[begin, end) of part p of n items split into `parts` contiguous blocks
    (sizes differ by at most one; same rule as the kernels' part_begin)."""
    if parts < 1 or not 0 <= p < parts:
        raise ValueError("bad partition index")
    return (n * p) // parts, (n * (p + 1)) // parts


def slice_partition(nslices: int, world: int, rank: int) -> list[int]:
    b, e = block_range(nslices, world, rank)
    return list(range(b, e))


def row_partition(nx: int, world: int, rank: int) -> tuple[int, int]:
    return block_range(nx, world, rank)


def row_shard_payload_len(ny: int, rank: int) -> int:
    """complex values per frame in the all-reduce: W (ny x R), GA (R x R),
    then ||Y||^2 and ||Ah||^2 packed as one complex."""
    return ny * rank + rank * rank + 1


def payload_doubles(ny: int, rank: int) -> int:
    """float64 words of a frame's payload in the kernel's layout (tensortrack_b200.h, tt_rows_args.xw/xg):
    W as complex128 [ny][R] (re, im interleaved), then GA packed (R(R+1)/2 complex128, lower triangle
    row by row: entry r(r+1)/2 + q holds GA[r][q], q <= r), then ||Y||^2 and ||Ah||^2."""
    return 2 * ny * rank + rank * (rank + 1) + 2


def packed_index(rank: int):
    """(r, q) of every packed Gram entry, in the kernels' order (tri_decode)."""
    r = np.concatenate([np.full(i + 1, i) for i in range(rank)])
    q = np.concatenate([np.arange(i + 1) for i in range(rank)])
    return r, q


def pack_payload(W, GA, yn: float, an: float) -> np.ndarray:
    """One rank's partials -> the float64 payload the all-reduce sums (same layout as phase 1 writes)."""
    W = np.asarray(W, np.complex128)
    ny, R = W.shape
    r, q = packed_index(R)
    ga = np.asarray(GA, np.complex128)[r, q]
    out = np.empty(payload_doubles(ny, R), np.float64)
    out[:2 * ny * R] = W.view(np.float64).ravel()
    out[2 * ny * R:2 * ny * R + 2 * ga.size] = ga.view(np.float64)
    out[-2] = yn
    out[-1] = an
    return out


def unpack_payload(buf, ny: int, rank: int) -> dict:
    """The summed payload -> W (ny x R), GA (R x R Hermitian), ||Y||^2, ||Ah||^2."""
    b = np.asarray(buf, np.float64)
    R = rank
    W = b[:2 * ny * R].copy().view(np.complex128).reshape(ny, R)
    r, q = packed_index(R)
    ga = b[2 * ny * R:2 * ny * R + R * (R + 1)].copy().view(np.complex128)
    GA = np.zeros((R, R), np.complex128)
    GA[r, q] = ga
    GA[q, r] = np.conj(ga)
    return dict(W=W, GA=GA, yn=float(b[-2]), an=float(b[-1]))
