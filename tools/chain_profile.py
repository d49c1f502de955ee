"""The collision chain at two ranks inside ONE process on one GPU (in-process
ranks share device 0), for launch lists / ncu captures of the chain's kernels
(pre-sum, collision update, E_co pack) — ncu runs single-process only.
Config-4 per-rank shape: 2,048 UIH samples per rank, Zipf(1.1) over 10M rows
per table, D = 256 fp32, PRESUM, reduce_chunk 64; `tables` tables in total
(default 8: 2 ranks x 41 GB of table on the one GPU).
usage: python tools/chain_profile.py [iters] [tables] [direct_mask]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2604_24073_b200 import embedding as E  # noqa: E402
from paper_2604_24073_b200 import workload  # noqa: E402
from paper_2604_24073_b200.comm import DeviceFabric  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 4
tables = int(sys.argv[2]) if len(sys.argv) > 2 else 8
direct = int(sys.argv[3]) if len(sys.argv) > 3 else 0
world, rpt, dim, seed, samples = 2, 10_000_000, 256, 20261018, 2048
batches = [[workload.cfg_tokens(seed, i, r, samples, tables, rpt)[1] for r in range(world)]
           for i in range(iters + 1)]
cap = max(b.size for it in batches for b in it) + 1024
geom = E.TableGeometry(tables * rpt, dim, world)
fabric = DeviceFabric(world, [0] * world)


def body(rank):
    ctx = E.Context(0, rank, world)
    shard = E.ShardView(geom, rank, 0.05, 7, dtype="f32", ctx=ctx)
    eng = E.PrioritizedEmbedding(shard, fabric.communicator(rank), max_occurrences=cap, reduce_chunk=64,
                                 presum=True)
    if direct:
        eng.set_eco_direct(direct & 1, cog=bool(direct & 2))
    s = torch.cuda.Stream()
    d = [torch.from_numpy(it[rank].view(np.int64)).cuda() for it in batches]
    g = torch.full((cap, dim), 1e-3, device="cuda")
    out = torch.empty((cap, dim), device="cuda")
    with torch.cuda.stream(s):
        for i in range(iters):
            n = batches[i][rank].size
            eng.forward(d[i], d[i + 1], out=out[:n], stream=s)
            eng.backward(g[:n], stream=s)
        eng.finalize(stream=s)
    s.synchronize()
    st = eng.stats()
    if rank == 0:
        print(f"rank 0: ids/iter {batches[0][0].size}, collision rows {[x.collision_rows for x in st]}", flush=True)
    eng.close()


fabric.run(body)
