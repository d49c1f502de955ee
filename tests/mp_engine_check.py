"""Multi-process engine parity (one process per GPU, CUDA-IPC receive windows,
copy-engine transfers + stream-memory-op flags). Launched by
tests/test_gpu_multiproc.py as

    torchrun --nproc-per-node N tests/mp_engine_check.py [f64|f32]

Each rank runs the reference's run_engine protocol (test_embedding.cpp:22-63)
on its shard; rank 0 gathers the table and compares it with the oracle:
bit-exact for f64, and sync == prio bitwise for f32."""
import os
import sys

os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2604_24073_b200 import embedding as E  # noqa: E402
from paper_2604_24073_b200 import workload  # noqa: E402
from paper_2604_24073_b200.comm import ProcessGroupFabric  # noqa: E402

OVERSUB = os.environ.get("FSX_MP_OVERSUB") == "1"


def run(prio, dtype, batches, geom, rank, world, dev, chunk, presum=False, transport="ce", direct=0):
    fabric = ProcessGroupFabric(rank, world, dev)
    ctx = E.Context(dev, rank, world)
    shard = E.ShardView(geom, rank, 0.05, 3, dtype=dtype, ctx=ctx)
    cap = max(len(b) for it in batches for b in it)
    cls = E.PrioritizedEmbedding if prio else E.SynchronizedEmbedding
    kw = {"presum": True} if (prio and presum) else {}
    eng = cls(shard, fabric.communicator(), max_occurrences=cap, reduce_chunk=chunk, transport=transport, **kw)
    if prio and direct:
        eng.set_eco_direct(direct & 1, cog=bool(direct & 2))
    s = torch.cuda.Stream(device=dev)
    with torch.cuda.stream(s):
        for i in range(len(batches)):
            if prio:
                nxt = batches[i + 1][rank] if i + 1 < len(batches) else None
                rows = eng.forward(batches[i][rank], nxt, stream=s)
            else:
                rows = eng.forward(batches[i][rank], stream=s)
            eng.backward(rows * 0.125 + 0.0625, stream=s)
        if prio:
            eng.finalize(stream=s)
    s.synchronize()
    ctx.sync()
    stats = eng.stats() if prio else None
    vals = torch.from_numpy(shard.values()).to(dev)
    eng.close()
    # gather the table (gather_full_table, embedding.cpp:611-631)
    sizes = [geom.local_rows(r) for r in range(world)]
    gdev = "cpu" if OVERSUB else dev
    parts = [torch.zeros((sizes[r], geom.dim), dtype=torch.float64, device=gdev) for r in range(world)]
    dist.all_gather(parts, vals.to(gdev))
    full = np.zeros((geom.total_rows, geom.dim), np.float64)
    for r in range(world):
        full[r::world] = parts[r].cpu().numpy()
    return full, stats


def main():
    dtype = sys.argv[1] if len(sys.argv) > 1 else "f64"
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = int(os.environ["LOCAL_RANK"])
    if OVERSUB:
        # more ranks than GPUs (e.g. 8 ranks on a 4-GPU box): ranks share GPUs,
        # windows still cross processes by CUDA IPC; gloo carries the checks
        dev %= torch.cuda.device_count()
        torch.cuda.set_device(dev)
        dist.init_process_group("gloo")
    else:
        torch.cuda.set_device(dev)
        dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
    rows, dim, iters = 40_000, 32, 5
    batches = [[workload.zipf_batch(50 + r, 4000, rows, offset=4000 * i) for r in range(world)]
               for i in range(iters)]
    geom = E.TableGeometry(rows, dim, world)
    chunk = 0 if dtype == "f64" else 64
    presum = "presum" in sys.argv[2:]
    # "nccl": the blocking baseline over NCCL (the comparison transport) must
    # produce the same table bit for bit
    sync_tr = "nccl" if "nccl" in sys.argv[2:] and not OVERSUB else "ce"
    t_sync, _ = run(False, dtype, batches, geom, rank, world, dev, chunk, transport=sync_tr)
    direct = 3 if "direct" in sys.argv[2:] else 0
    t_prio, stats = run(True, dtype, batches, geom, rank, world, dev, chunk, presum, direct=direct)
    ok = True
    if rank == 0:
        from oracle import Oracle
        O = Oracle()
        f32 = dtype == "f32"
        # bitwise against the oracle's model of the same numeric path: the
        # fp32 storage model, the chunk association and (prio) PRESUM
        want_s, want_stats = O.run_engine(world, batches, rows, dim, 0.05, 3, with_stats=True, store_f32=f32,
                                          reduce_chunk=chunk)
        want_p, _ = O.run_engine(world, batches, rows, dim, 0.05, 3, store_f32=f32, reduce_chunk=chunk,
                                 presum=presum)
        ok_s = np.array_equal(t_sync.view(np.uint64), want_s.view(np.uint64))
        ok_p = np.array_equal(t_prio.view(np.uint64), want_p.view(np.uint64))
        got_stats = np.array([[s.collision_rows, s.unique_next_rows, s.blocking_bytes] for s in stats], np.uint64)
        st_ok = np.array_equal(got_stats, want_stats)
        print(f"[mp] world={world} dtype={dtype} chunk={chunk} presum={presum} direct={direct} "
              f"sync transport={sync_tr}: "
              f"sync bit-exact vs oracle {ok_s}, "
              f"prio bit-exact vs oracle {ok_p}, stats equal {st_ok}")
        ok &= ok_s and ok_p and st_ok
        print("MP_OK" if ok else "MP_FAIL", flush=True)
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
