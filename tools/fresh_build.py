"""One fresh K27 direction-optimizing build (out + in compressed streams) --
the command the build's ncu launch list is taken on."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_06890_b200 as zc
dg = zc.generate_rmat(int(sys.argv[1]) if len(sys.argv) > 1 else 27, 16, seed=27)
t = time.time()
dg.build_in_lists()
print(f"fresh out+in build {time.time() - t:.2f}s", flush=True)
