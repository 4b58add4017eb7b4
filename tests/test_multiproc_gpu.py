"""The partitioned driver as the bench runs it at N>1 -- one process per
partition, torch.distributed between them -- with 2 processes sharing the one
GPU of the test box (gloo, host-staged reduce-scatter; the fused exchange
through same-device CUDA IPC).  CudaPartition engines, every exchange,
against the oracle."""
import multiprocessing as mp
import os
import random

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, q, srcs):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    import torch
    import torch.distributed as dist
    from paper_2006_06890_b200.multi import (exchange_buffers, generate_rmat_part,
                                             run_partition)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = []
    try:
        for sym, algo, strat in ((False, "bfs", "merged-aligned"), (False, "bfs", "packed"),
                                 (True, "cc", "merged-aligned"), (True, "bfs", "merged-aligned"),
                                 (False, "bfs", "direction-optimizing")):
            part = generate_rmat_part(14, world, rank, 16, seed=21, symmetrize=sym, device=0)
            bufs = exchange_buffers(algo, world, part.stride, torch.device("cuda", 0))
            for fused, bx in ((False, "bitmap"), (True, "bitmap"), (True, "store")):
                if bx == "store" and (algo != "bfs" or not fused):
                    continue
                r = run_partition(part, algo, srcs[sym], strat, stage_host=True, buffers=bufs,
                                  fused=fused, bfs_exchange=bx)
                out.append((sym, algo, strat, f"{fused}/{bx}", r.values, r.iterations,
                            list(r.traversed_edges), r.exchange_bytes, r.local_traversed))
            part.close()
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_two_processes_one_gpu_match_oracle():
    import oracle
    import paper_2006_06890_b200 as zc
    world = 2
    refs, handles, srcs = {}, [], {}
    for sym in (False, True):  # as_csr views the handle's pinned lists: keep it open
        h = zc.generate_rmat(14, 16, seed=21, symmetrize=sym)
        handles.append(h)
        refs[sym] = h.as_csr()
        srcs[sym] = int(zc.pick_sources(refs[sym], 1, seed=7)[0])
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = random.randint(20000, 40000)
    ps = [ctx.Process(target=_worker, args=(r, world, port, q, srcs)) for r in range(world)]
    for p in ps:
        p.start()
    got = dict(q.get(timeout=600) for _ in range(world))
    for p in ps:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in ps)
    for k, (sym, algo, strat, fused, _, iters, trav, xb, lt) in enumerate(got[0]):
        g = refs[sym]
        ref = oracle.run(algo, g, srcs[sym], threads=4)
        assert ref.iterations > 3
        vals = np.concatenate([got[r][k][4] for r in range(world)])
        assert np.array_equal(vals, ref.values), (sym, algo, strat, fused)
        assert iters == ref.iterations and trav == ref.traversed_edges, (sym, algo, strat, fused)
        assert got[1][k][5] == iters and got[1][k][6] == trav  # every rank agrees
        # each rank streamed its own share; together the reference's work
        assert got[0][k][8] + got[1][k][8] == sum(ref.traversed_edges)
        assert xb > 0 and got[1][k][7] > 0, (sym, algo, strat, fused)  # both ranks sent
    for h in handles:
        h.close()
