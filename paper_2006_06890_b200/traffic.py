"""Per-iteration request statistics of a traversal's list reads.

The GPU's request model (zc_kernels.cu ``k_model_*``) counts, for each
iteration, the requests of 1..4 32-byte sectors on the edge stream and on the
weight stream (SSSP).  This module turns that u64[8] vector into the record the
reference returns in ``TraversalResult.per_iteration_traffic`` -- same public
attributes and methods as the reference's ``TrafficStats``
(coalesce.py:44-85: ``hist``, ``request_count``, ``payload_bytes``,
``dram_bytes``, ``amplification``, ``fraction``, ``mean_request_bytes``,
``merged_with``, ``with_amplification``, ``zero``, ``from_size_counts``) so
result rows stay comparable.  The hardware counterpart of the same numbers is
ncu's ``syslts__t_{requests,sectors}_aperture_sysmem_op_read``.
"""
from __future__ import annotations

from typing import Sequence

import numpy as np

SIZES = (32, 64, 96, 128)
_SIZE_VEC = np.array(SIZES, dtype=np.int64)
# bytes the host DRAM moves per request: its bursts are 64 B, so one- and
# two-sector requests cost a burst, three and four sectors two (coalesce.py:69-70)
_DRAM_VEC = np.array([64, 64, 128, 128], dtype=np.int64)


class TrafficStats:
    """Request-size histogram of one iteration (or a sum of iterations)."""

    __slots__ = ("_counts", "amplification")

    def __init__(self, counts, amplification: float = 0.0):
        self._counts = np.asarray(counts, dtype=np.int64).reshape(4)
        self.amplification = float(amplification)

    # -- constructors
    @classmethod
    def zero(cls) -> "TrafficStats":
        return cls(np.zeros(4, np.int64))

    @classmethod
    def from_size_counts(cls, counts_by_sectors: Sequence[int]) -> "TrafficStats":
        """counts_by_sectors[i] = requests spanning i+1 sectors (edge + weight
        streams already added)."""
        c = np.zeros(4, np.int64)
        v = np.asarray(list(counts_by_sectors), dtype=np.int64)
        c[: min(4, v.size)] = v[:4]
        return cls(c)

    @classmethod
    def from_device_hist(cls, row) -> "TrafficStats":
        """One iteration of zc_run_traffic: [edge 1..4 sectors, weight 1..4]."""
        r = np.asarray(row, dtype=np.int64)
        return cls(r[:4] + r[4:8])

    # -- the reference's attributes
    @property
    def hist(self) -> dict:
        return {s: int(n) for s, n in zip(SIZES, self._counts)}

    @property
    def request_count(self) -> int:
        return int(self._counts.sum())

    @property
    def payload_bytes(self) -> int:
        return int(self._counts @ _SIZE_VEC)

    @property
    def dram_bytes(self) -> int:
        return int(self._counts @ _DRAM_VEC)

    @property
    def mean_request_bytes(self) -> float:
        n = self.request_count
        return self.payload_bytes / n if n else 0.0

    def fraction(self, size: int) -> float:
        n = self.request_count
        return self.hist.get(size, 0) / n if n else 0.0

    def merged_with(self, other: "TrafficStats") -> "TrafficStats":
        return TrafficStats(self._counts + other._counts)

    __add__ = merged_with

    def with_amplification(self, dataset_bytes: int) -> "TrafficStats":
        return TrafficStats(self._counts, self.payload_bytes / dataset_bytes)

    def __eq__(self, other) -> bool:
        return (isinstance(other, TrafficStats) and np.array_equal(self._counts, other._counts)
                and self.amplification == other.amplification)

    def __repr__(self) -> str:
        return (f"TrafficStats(hist={self.hist}, request_count={self.request_count}, "
                f"payload_bytes={self.payload_bytes}, dram_bytes={self.dram_bytes}, "
                f"amplification={self.amplification})")
