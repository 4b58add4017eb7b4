"""Request-size statistics (reference coalesce.py:44-85).

On the B200 path the modelled histogram is computed on the GPU from each
iteration's frontier (zc_kernels.cu, k_model_*); the hardware counterpart is
ncu's syslts__t_{sectors,requests}_aperture_sysmem_op_read.
"""
from __future__ import annotations

from dataclasses import dataclass, replace
from typing import Sequence

SIZES = (32, 64, 96, 128)


@dataclass
class TrafficStats:
    """Histogram of request sizes plus derived byte counts for one trace."""

    hist: dict
    request_count: int
    payload_bytes: int
    dram_bytes: int
    amplification: float = 0.0

    @classmethod
    def zero(cls) -> "TrafficStats":
        return cls({s: 0 for s in SIZES}, 0, 0, 0)

    @classmethod
    def from_size_counts(cls, counts_by_sectors: Sequence[int]) -> "TrafficStats":
        """counts_by_sectors[i] = requests spanning i+1 sectors."""
        hist = {s: 0 for s in SIZES}
        for i, c in enumerate(counts_by_sectors):
            hist[32 * (i + 1)] = int(c)
        payload = sum(size * n for size, n in hist.items())
        # host DRAM serves 64-byte bursts (reference coalesce.py:69-70)
        dram = 64 * (hist[32] + hist[64]) + 128 * (hist[96] + hist[128])
        return cls(hist, sum(hist.values()), payload, dram)

    def merged_with(self, other: "TrafficStats") -> "TrafficStats":
        hist = {s: self.hist.get(s, 0) + other.hist.get(s, 0) for s in SIZES}
        return TrafficStats(hist, self.request_count + other.request_count,
                            self.payload_bytes + other.payload_bytes,
                            self.dram_bytes + other.dram_bytes)

    def fraction(self, size: int) -> float:
        return self.hist.get(size, 0) / self.request_count if self.request_count else 0.0

    @property
    def mean_request_bytes(self) -> float:
        return self.payload_bytes / self.request_count if self.request_count else 0.0

    def with_amplification(self, dataset_bytes: int) -> "TrafficStats":
        return replace(self, amplification=self.payload_bytes / dataset_bytes)
