"""B200-native EMOGI: BFS / SSSP / CC over CSR graphs whose edge list stays in
pinned host memory and is read by the GPU with zero-copy, cache-line-sized
loads (arxiv 2006.06890).

Drop-in for the traversal path of the reference package ``zcgraph``
(/root/reference/pkg/src/zcgraph/__init__.py:9-37): same ``CsrGraph``,
generators, EMGI IO, ``AccessStrategy`` and ``bfs`` / ``sssp`` / ``cc``
returning ``TraversalResult``.  The traversals execute in hand-written sm_100a
CUDA kernels behind a C ABI (include/zcgraph.h); there is no CPU fallback.
"""
from .access import LINE_BYTES, SECTOR_BYTES, WARP_LANES, AccessStrategy
from .csr import (CsrGraph, DegreeCdf, degree_cdf, generate_powerlaw, generate_uniform,
                  load_csr_binary, load_edge_list_text, pick_sources, store_csr_binary, symmetrized, validate,
                  with_uniform_weights)
from .device import (DeviceGraph, device_graph, evict, generate_rmat, generate_uniform_device,
                     link_probe, open_emgi, pinned_empty, release)
from .traffic import TrafficStats
from .traversal import (SCHEDULES, UNREACHED_DIST, UNREACHED_LEVEL, TraversalResult, bfs,
                        bfs_many, cc, pagerank, sssp, sssp_many)

__version__ = "0.1.0"

__all__ = [
    "AccessStrategy", "CsrGraph", "SCHEDULES", "DegreeCdf", "DeviceGraph", "LINE_BYTES", "SECTOR_BYTES",
    "TrafficStats", "TraversalResult", "UNREACHED_DIST", "UNREACHED_LEVEL", "WARP_LANES",
    "bfs", "bfs_many", "cc", "degree_cdf", "device_graph", "evict", "generate_powerlaw", "generate_rmat",
    "generate_uniform", "generate_uniform_device", "link_probe", "load_csr_binary", "load_edge_list_text", "open_emgi",
    "pagerank", "pick_sources", "pinned_empty", "release", "sssp", "sssp_many", "store_csr_binary", "symmetrized",
    "validate", "with_uniform_weights",
]
