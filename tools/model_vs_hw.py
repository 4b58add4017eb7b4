"""Reference request model (coalesce.py:165-207, evaluated on the GPU) next to
the hardware: per level, modelled payload / requests vs ncu's sysmem sector
fills.  Run twice: plain (model numbers) and under ncu (hardware numbers):

  python tools/model_vs_hw.py --scale 25                       > model.txt
  ncu --metrics syslts__t_sectors_srcunit_tex_aperture_sysmem_op_read_lookup_miss.sum,\
pcie__read_bytes.sum -k regex:"k_expand_(sweep|naive)" --csv \
      python tools/model_vs_hw.py --scale 25 --no-model     > hw.csv
"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_06890_b200 as zc

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=25)
ap.add_argument("--no-model", action="store_true")
ap.add_argument("--strategies", default="naive,merged,merged-aligned")
a = ap.parse_args()
dg = zc.generate_rmat(a.scale, 16, seed=27)
src = int(zc.pick_sources(dg.as_csr(), 1, seed=7)[0])
for s in a.strategies.split(","):
    r = zc.bfs(dg, src, s, collect_traffic=not a.no_model)
    if a.no_model:
        continue
    for k in range(r.iterations):
        t = r.per_iteration_traffic[k]
        print(f"{s} L{k} edges={r.traversed_edges[k]} requests={t.request_count} "
              f"payload={t.payload_bytes} h={t.hist[32]},{t.hist[64]},{t.hist[96]},{t.hist[128]}",
              flush=True)
