"""Stress check (one process per GPU, torchrun): the prioritized engine over
large, skewed per-rank batches (1x..2x the config-4 share, Zipf ids, D = 256
fp32, PRESUM) with the collision chain on the copy engines and with direct
stores (mask 3); the two runs must leave bit-identical tables. Prints
STRESS_OK / STRESS_FAIL on rank 0.
usage: torchrun --nproc-per-node N tests/mp_stress_direct.py [iters] [mask]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2604_24073_b200 import embedding as E  # noqa: E402
from paper_2604_24073_b200 import workload  # noqa: E402
from paper_2604_24073_b200.comm import ProcessGroupFabric  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 12
mask = int(sys.argv[2]) if len(sys.argv) > 2 else 3
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dev = int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(dev)
dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
tables, rpt, dim, seed = 8 * world, 1_000_000, 256, 20261018
batches = [workload.cfg_tokens(seed, i, rank, 2048 * (1 + rank % 2), tables, rpt)[1] for i in range(iters + 1)]
n_max = torch.tensor([max(b.size for b in batches)], device=dev)
dist.all_reduce(n_max, op=dist.ReduceOp.MAX)
cap = int(n_max.item()) + 1024
geom = E.TableGeometry(tables * rpt, dim, world)


def run(m):
    ctx = E.Context(dev, rank, world)
    shard = E.ShardView(geom, rank, 0.05, 7, dtype="f32", ctx=ctx)
    eng = E.PrioritizedEmbedding(shard, ProcessGroupFabric(rank, world, dev).communicator(), max_occurrences=cap,
                                 reduce_chunk=64, presum=True)
    eng.set_ids_ready(True)
    if m:
        eng.set_eco_direct(m & 1, cog=bool(m & 2))
    s = torch.cuda.Stream()
    d = [torch.from_numpy(b.view(np.int64)).to(dev) for b in batches]
    g = torch.full((cap, dim), 1e-3, device=dev)
    with torch.cuda.stream(s):
        for i in range(iters):
            n = batches[i].size
            rows = eng.forward(d[i], d[i + 1] if i + 1 < iters else None, stream=s)
            eng.backward(rows * 0.125 + g[:n], stream=s)
        eng.finalize(stream=s)
    s.synchronize()
    out = shard.device_values().cpu().numpy().copy()
    eng.close()
    return out


a = run(0)
b = run(mask)
same = bool(np.array_equal(a.view(np.uint8), b.view(np.uint8)))
t = torch.tensor([1 if same else 0], device=dev)
dist.all_reduce(t, op=dist.ReduceOp.MIN)
if rank == 0:
    print(f"[stress] world={world} iters={iters} mask={mask} ids/rank {[b.size for b in batches[:1]]} "
          f"tables identical on every rank: {bool(t.item())}")
    print("STRESS_OK" if t.item() else "STRESS_FAIL", flush=True)
dist.barrier()
dist.destroy_process_group()
