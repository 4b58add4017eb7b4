import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_06890_b200.device as d
chunk, rnd = int(sys.argv[1]), sys.argv[2] == "random"
print(chunk, sys.argv[2], d.read_probe(1 << 30, chunk, rnd, "pinned", iters=1))
