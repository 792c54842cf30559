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

__all__ = ["block_range", "slice_partition", "row_partition", "row_shard_payload_len"]


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
