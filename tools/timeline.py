"""Debug tool (not a test): per-rank span timeline of a few steady prioritized
iterations of the bench workload, optionally with the config-5 victim
between forward and backward. Run under torchrun, e.g.
  torchrun --nproc-per-node 4 tools/timeline.py --victim 1 --presum 1
Prints every rank's spans (phase, start, end, length; ms from the rank's
first span) to gpurun_out/timeline_r<rank>.txt and a per-phase summary."""
import argparse
import os
import time
import sys

os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402
from paper_2604_24073_b200 import embedding as E  # noqa: E402
from paper_2604_24073_b200.comm import DeviceFabric, ProcessGroupFabric  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--victim", type=int, default=1)
ap.add_argument("--presum", type=int, default=1)
ap.add_argument("--balance", type=int, default=1)
ap.add_argument("--iters", type=int, default=8)
ap.add_argument("--profile-from", type=int, default=5)
cli = ap.parse_args()

rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
local = int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
if world > 1:
    dist.init_process_group("nccl", device_id=dev)
    fabric = ProcessGroupFabric(rank, world, local)
else:
    fabric = DeviceFabric(1, [local])


class A:
    tables_per_rank, rows_per_table, samples, seed, dim = 8, 10_000_000, 2048, 20261018, 256


args = A()
ctx = E.Context(local, rank, world)
batches, blens = bench.batches_for(args, rank, world, cli.iters + 1, with_lens=True)
if cli.balance and world > 1:
    bi, bl = bench.balance_batches(args, world, rank, cli.iters + 1, 0, ctx)
    batches = [bi[i] for i in range(cli.iters + 1)]
    blens = [bl[i] for i in range(cli.iters + 1)]
cap = int(max(b.size for b in batches) * 1.05) + 1024
if world > 1:
    t = torch.tensor([cap], dtype=torch.int64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    cap = int(t.item())
shard = E.ShardView(E.TableGeometry(8 * world * 10_000_000, 256, world), rank, 0.05, 7, dtype="f32", ctx=ctx)
eng = E.PrioritizedEmbedding(shard, fabric.communicator(rank), max_occurrences=cap, reduce_chunk=64,
                             presum=bool(cli.presum))
eng.set_ids_ready(True)
victim = bench.Victim(dev) if cli.victim else None
s = torch.cuda.Stream()
d = [torch.from_numpy(b.view(np.int64)).to(dev) for b in batches]
g = torch.full((cap, 256), 1e-3, device=dev)
out = torch.empty((cap, 256), device=dev)
hmarks = []
with torch.cuda.stream(s):
    for i in range(cli.iters):
        if i == cli.profile_from:
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            eng.set_profiling(True)
            eng.spans()
        n = batches[i].size
        hmarks.append(("fwd>", i, time.monotonic_ns() * 1e-6))
        eng.forward(d[i], d[i + 1], out=out[:n], stream=s)
        hmarks.append(("fwd<", i, time.monotonic_ns() * 1e-6))
        if victim:
            victim.run(blens[i])
        hmarks.append(("bwd>", i, time.monotonic_ns() * 1e-6))
        eng.backward(g[:n], stream=s)
        hmarks.append(("bwd<", i, time.monotonic_ns() * 1e-6))
torch.cuda.synchronize()
tr = eng.trace()
CH = ["ids", "rows", "grads", "ex", "mask", "cog", "exg", "cor", "idx", "grp", "ag"]
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
# host clock aligned so that the earliest span's issue == its GPU start
# (the profiled window starts on an idle GPU, after a synchronize)
first = min(tr, key=lambda x: x[3])
h0 = first[5] - first[3]
with open(os.path.join(ROOT, "gpurun_out", f"timeline_r{rank}.txt"), "w") as f:
    f.write("phase      lane ch     gpu_start  gpu_end    len   host_issue  gpu_start-host\n")
    def chname(ch):
        if ch < 0:
            return "-"
        if ch >= 1000:  # one copy of an all-to-all: channel, destination
            return f"{CH[(ch - 1000) // 16]}>{(ch - 1000) % 16}"
        return CH[ch]
    rows = [(a, f"{ph:10s} {lane}    {chname(ch):6s} {a:8.3f} {b:8.3f} {b - a:7.3f}  {h - h0:8.3f}  {a - h + h0:8.3f}")
            for ph, lane, ch, a, b, h in tr]
    rows += [(t - h0, f"HOST {m} {i:3d}                                      {t - h0:8.3f}")
             for m, i, t in hmarks if t - h0 >= -1.0]
    for _, line in sorted(rows):
        f.write(line + "\n")
sp = [(ph, a, b) for ph, lane, ch, a, b, h in tr if ch < 1000]
tot = {}
for ph, a, b in sp:
    tot[ph] = tot.get(ph, 0.0) + (b - a)
steps = cli.iters - cli.profile_from
print(f"rank {rank}: ids {batches[cli.profile_from].size} victim_units "
      f"{victim.run.__self__.cost_us(blens[cli.profile_from]) / victim.unit_us if victim else 0:.0f} "
      + " ".join(f"{k}={v / steps:.3f}" for k, v in sorted(tot.items())), flush=True)
if world > 1:
    dist.barrier()
    dist.destroy_process_group()
