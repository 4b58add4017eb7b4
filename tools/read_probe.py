"""Zero-copy read microbenchmark sweep: request size x pattern x allocation."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_06890_b200.device as d

size = int(sys.argv[1]) if len(sys.argv) > 1 else 4 << 30
for alloc in ("pinned", "thp"):
    for random in (False, True):
        row = []
        for chunk in (32, 64, 96, 128, 256, 512):
            row.append(f"{chunk}B:{d.read_probe(size, chunk, random, alloc):6.2f}")
        print(f"{alloc:6s} {'random' if random else 'seq':6s} " + " ".join(row), flush=True)
for mode, name in ((2, "warp-streams"), (3, "cta-streams")):
    print(f"pinned {name:12s} " + " ".join(f"{c}B:{d.read_probe(size, c, mode, 'pinned'):6.2f}"
                                          for c in (32, 128, 512)), flush=True)
print("hbm    random " + " ".join(f"{c}B:{d.read_probe(size, c, True, 'hbm'):8.1f}"
                               for c in (32, 64, 128, 512)), flush=True)
