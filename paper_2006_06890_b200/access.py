"""Access strategies (reference access.py:28-37).

The strategy selects which CUDA expansion kernel runs; it never changes the
results (the reference's strategy-independence contract).
"""
from __future__ import annotations

from enum import Enum

WARP_LANES = 32
LINE_BYTES = 128
SECTOR_BYTES = 32


class AccessStrategy(Enum):
    NAIVE = "naive"
    MERGED = "merged"
    MERGED_ALIGNED = "merged-aligned"


# "packed" is a B200 extension beyond the reference's three (include/zcgraph.h
# ZC_PACKED): windows are the aligned 32-element blocks of the union of the
# frontier's lists, fetched once each.  Results are identical.
# "compressed" (ZC_COMPRESSED) streams the lists sorted and delta-encoded in
# 128-byte lines (hub lists in whole lines, short lists sharing lines, SSSP
# weights alongside); every result is independent of the order inside a list.
# "direction-optimizing" (ZC_DIRECTION_OPT, BFS only) runs compressed top-down
# steps and switches to bottom-up steps over the compressed in-lists when the
# frontier is large (Beamer et al.); levels, iterations and traversed_edges
# (the frontier's out-degrees) are the reference's.
_IDS = {"naive": 0, "merged": 1, "merged-aligned": 2, "packed": 3, "compressed": 4,
        "direction-optimizing": 5}


def strategy_id(strategy) -> int:
    """C-ABI id of a strategy given as our enum, the reference's enum or its name."""
    name = getattr(strategy, "value", strategy)
    try:
        return _IDS[name]
    except (KeyError, TypeError):
        raise ValueError(f"unknown strategy {strategy!r}") from None


def aligned_start(start_elem: int, elem_bytes: int) -> int:
    """First element of the 128-byte line holding start_elem (access.py:34-37)."""
    return start_elem & ~(LINE_BYTES // elem_bytes - 1)
