"""Per-level composition of a compressed-stream BFS on K27: long-list lines
vs short lists (their bytes and the distinct shared lines they touch), next
to the measured per-level expansion time -> achieved line requests/s."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2006_06890_b200 as zc

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 27
dg = zc.generate_rmat(scale, 16, seed=27)
nb = dg.build_compressed()
g = dg.as_csr()
src = int(zc.pick_sources(g, 64, seed=7)[0])
zc.bfs(dg, src, "compressed", collect_traffic=False)
r = zc.bfs(dg, src, "compressed", collect_traffic=False)
prof = dg.expand_profile(r.iterations)
idx = dg.compressed_index()
long_ = (idx[:-1] >> np.uint64(63)).astype(bool)
pos = (idx & np.uint64((1 << 63) - 1)).astype(np.int64)
span = np.diff(pos)
deg = np.diff(g.offsets)
line = pos[:-1] >> 10
print(f"stream {nb/2**30:.2f} GiB; long lists {long_.sum()} ({deg[long_].sum()/g.num_edges:.1%} of edges, "
      f"{span[long_].sum()/8/deg[long_].sum():.2f} B/edge); short lists {(~long_ & (deg>0)).sum()} "
      f"({span[~long_].sum()/8/max(deg[~long_].sum(),1):.2f} B/edge incl. padding)")
for k in range(r.iterations):
    f = r.values == k
    fl, fs = f & long_, f & ~long_ & (deg > 0)
    lines_long = int(span[fl].sum() // 1024)
    short_lines = np.unique(line[fs]).size
    short_bytes = int(span[fs].sum() // 8)
    req = lines_long + short_lines
    ms = prof[k]
    print(f"it {k} front={int(f.sum()):10d} edges={int(deg[f].sum()):11d} | long {int(fl.sum()):8d} lists "
          f"{lines_long:9d} lines | short {int(fs.sum()):9d} lists {short_bytes/2**20:8.1f} MiB in "
          f"{short_lines:9d} lines | {ms:8.2f} ms  {req/ms/1e3 if ms else 0:7.1f} M lines/s  "
          f"{(lines_long*128+short_bytes)/ms/1e6 if ms else 0:6.1f} GB/s stored")
