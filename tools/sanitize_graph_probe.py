"""Minimal device-driven-loop run (one CUDA graph with a conditional WHILE
node) for compute-sanitizer: does synccheck flag the graph path itself?"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_06890_b200 as zc

g = zc.with_uniform_weights(zc.generate_powerlaw(3000, 12.0, 2.0, seed=2))
src = int(zc.pick_sources(g, 1)[0])
zc.bfs(g, src, sys.argv[1] if len(sys.argv) > 1 else "merged-aligned", collect_traffic=False)
print("graph probe ok")
