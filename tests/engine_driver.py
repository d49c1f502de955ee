"""Shared driver for engine parity tests: the Python restatement of
tests/test_embedding.cpp:22-63 (run_engine) over libfsx engines."""
import numpy as np
import torch

from paper_2604_24073_b200 import embedding as E
from paper_2604_24073_b200.comm import DeviceFabric


def run_engine(prioritized, batches, geom, lr, seed, dtype="f64", reduce_chunk=0,
               grad_scale=0.125, grad_shift=0.0625, devices=None, with_stats=False, presum=False,
               direct=0, direct_from=0):
    """batches[i][r] = rank r's ids of iteration i. Returns the final table
    (f64, global order) and rank 0's IterationStats (prioritized).
    direct (prioritized): collision-chain transfer mask (1 = E_co, 2 = CO_G by
    direct stores), switched on between iterations direct_from - 1 and direct_from."""
    world = geom.num_shards
    iters = len(batches)
    cap = max([len(b) for it in batches for b in it] + [1])
    fabric = DeviceFabric(world, devices)
    shards = [None] * world
    stats = {}

    def body(rank):
        dev = fabric.device_of(rank)
        ctx = E.Context(dev, rank, world)
        shard = E.ShardView(geom, rank, lr, seed, dtype=dtype, ctx=ctx)
        comm = fabric.communicator(rank)
        if prioritized:
            eng = E.PrioritizedEmbedding(shard, comm, max_occurrences=cap, reduce_chunk=reduce_chunk,
                                         presum=presum)
        else:
            eng = E.SynchronizedEmbedding(shard, comm, max_occurrences=cap, reduce_chunk=reduce_chunk)
        stream = torch.cuda.Stream(device=dev)
        with torch.cuda.stream(stream):
            for i in range(iters):
                cur = batches[i][rank]
                if prioritized and direct and i == direct_from:
                    eng.set_eco_direct(direct & 1, cog=bool(direct & 2))
                if prioritized:
                    nxt = batches[i + 1][rank] if i + 1 < iters else None
                    rows = eng.forward(cur, nxt, stream=stream)
                else:
                    rows = eng.forward(cur, stream=stream)
                grads = rows * grad_scale + grad_shift
                eng.backward(grads, stream=stream)
            if prioritized:
                eng.finalize(stream=stream)
        stream.synchronize()
        ctx.sync()
        shards[rank] = shard
        if prioritized and rank == 0 and with_stats:
            stats["s"] = eng.stats()
        eng.close()

    fabric.run(body)
    table = E.gather_full_table(shards)
    return table, stats.get("s")
