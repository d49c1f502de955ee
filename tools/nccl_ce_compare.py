"""NCCL >= 2.28's copy-engine collectives as a comparator for the engine's own
copy-engine all-to-all (the reference's PAPER.md names NCCL's
CE collectives as the off-the-shelf SM-free alternative).

One process per GPU (torchrun). For each NCCL CTA policy — DEFAULT (SM
kernels) and ZERO (NCCL_CTA_POLICY_ZERO: no CTAs; with buffers registered as
symmetric windows NCCL moves the data with the copy engines) — a fresh NCCL
communicator (ncclCommInitRankConfig), send / receive buffers from
ncclMemAlloc registered with ncclCommWindowRegister(NCCL_WIN_COLL_SYMMETRIC),
then ncclAlltoAll:
  * alone: GB/s out per GPU (CUDA events, max over ranks);
  * under load: the config-5 victim (bench.Victim, bf16 GEMMs) on the compute
    stream while the same number of all-to-alls run on a side stream; the
    victim's own duration vs alone = the SMs the collective takes.
Also the engine's copy-engine all-to-all (fsx_a2a_ce) under the same load.
Prints one JSON line (rank 0).
usage: torchrun --nproc-per-node N tools/nccl_ce_compare.py [per_peer_MiB]"""
import ctypes as C
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402

per_peer = (int(sys.argv[1]) if len(sys.argv) > 1 else 8) << 20
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)

nccl = C.CDLL("libnccl.so.2", mode=C.RTLD_GLOBAL)
INT_MIN = -2147483648


class NcclConfig(C.Structure):  # ncclConfig_v22800 (nccl.h)
    _fields_ = [("size", C.c_size_t), ("magic", C.c_uint), ("version", C.c_uint), ("blocking", C.c_int),
                ("cgaClusterSize", C.c_int), ("minCTAs", C.c_int), ("maxCTAs", C.c_int), ("netName", C.c_char_p),
                ("splitShare", C.c_int), ("trafficClass", C.c_int), ("commName", C.c_char_p),
                ("collnetEnable", C.c_int), ("CTAPolicy", C.c_int), ("shrinkShare", C.c_int), ("nvlsCTAs", C.c_int),
                ("nChannelsPerNetPeer", C.c_int), ("nvlinkCentricSched", C.c_int)]


class UniqueId(C.Structure):  # ncclUniqueId: 128 bytes, passed by value
    _fields_ = [("internal", C.c_char * 128)]


def check(r, what):
    if r != 0:
        nccl.ncclGetErrorString.restype = C.c_char_p
        raise RuntimeError(f"{what}: {nccl.ncclGetErrorString(r).decode()}")


ver = C.c_int()
check(nccl.ncclGetVersion(C.byref(ver)), "version")


def make_comm(policy):
    uid = UniqueId()
    if rank == 0:
        check(nccl.ncclGetUniqueId(C.byref(uid)), "unique id")
    t = torch.frombuffer(bytearray(C.string_at(C.addressof(uid), 128)), dtype=torch.uint8).to(dev)
    dist.broadcast(t, 0)
    C.memmove(C.addressof(uid), bytes(t.cpu().numpy()), 128)
    cfg = NcclConfig(C.sizeof(NcclConfig), 0xcafebeef, ver.value, INT_MIN, INT_MIN, INT_MIN, INT_MIN, None,
                     INT_MIN, INT_MIN, None, INT_MIN, policy, INT_MIN, INT_MIN, INT_MIN, INT_MIN)
    comm = C.c_void_p()
    check(nccl.ncclCommInitRankConfig(C.byref(comm), world, uid, rank, C.byref(cfg)), "comm init")
    return comm


def sym_buffer(comm, nbytes):
    p = C.c_void_p()
    check(nccl.ncclMemAlloc(C.byref(p), C.c_size_t(nbytes)), "mem alloc")
    win = C.c_void_p()
    check(nccl.ncclCommWindowRegister(comm, p, C.c_size_t(nbytes), C.byref(win), 1), "window register")
    return p, win


def agree_max(x):
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


victim = bench.Victim(dev)
lens = [512] * 2048  # a fixed config-5-like load (same on every rank)
side = torch.cuda.Stream(device=dev)


def measure(issue, name):
    # alone: GB/s out per GPU
    for _ in range(3):
        issue()
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 20
    e0.record(side)
    for _ in range(n):
        issue()
    e1.record(side)
    torch.cuda.synchronize()
    ms = agree_max(e0.elapsed_time(e1) / n)
    gbs = (world - 1) * per_peer / (ms * 1e-3) / 1e9
    # victim alone, then with concurrent all-to-alls (equal call counts on every rank)
    def victim_ms(calls):
        v0, v1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        dist.barrier()
        cur = torch.cuda.current_stream(dev)
        v0.record(cur)
        for _ in range(4):
            victim.run(lens)
        v1.record(cur)
        for _ in range(calls):
            issue()
        torch.cuda.synchronize()
        return agree_max(v0.elapsed_time(v1))
    alone = victim_ms(0)
    calls = max(1, int(alone / ms))
    loaded = victim_ms(calls)
    return {"ms_per_call": round(ms, 4), "gbs_out_per_gpu": round(gbs, 1), "victim_ms_alone": round(alone, 3),
            "victim_ms_loaded": round(loaded, 3), "calls": calls,
            "victim_slowdown_pct": round(100.0 * (loaded / alone - 1.0), 2)}


out = {"tool": "nccl_ce_compare", "world": world, "per_peer_mib": per_peer >> 20, "nccl_version": ver.value}
for name, policy in (("nccl_default", 0), ("nccl_cta_policy_zero", 2)):
    try:
        comm = make_comm(policy)
        sp, _ = sym_buffer(comm, world * per_peer)
        rp, _ = sym_buffer(comm, world * per_peer)

        def issue(comm=comm, sp=sp, rp=rp):
            check(nccl.ncclAlltoAll(sp, rp, C.c_size_t(per_peer), 0, comm, C.c_void_p(side.cuda_stream)), "alltoall")
        out[name] = measure(issue, name)
    except Exception as e:  # noqa: BLE001
        out[name] = {"error": str(e)[:200]}

# the engine's copy-engine all-to-all under the same load
from paper_2604_24073_b200 import _lib, embedding as E  # noqa: E402
from paper_2604_24073_b200.comm import ProcessGroupFabric  # noqa: E402

ctx = E.Context(local, rank, world)
fabric = ProcessGroupFabric(rank, world, local)
shard = E.ShardView(E.TableGeometry(world * 1024, 256, world), rank, 0.05, 1, dtype="f32", ctx=ctx)
eng = E.PrioritizedEmbedding(shard, fabric.communicator(), max_occurrences=max(1, per_peer // 1024))
n64 = per_peer // 8
send = torch.zeros(world * n64, dtype=torch.int64, device=dev)
recv = torch.empty(world * n64, dtype=torch.int64, device=dev)
offs = (C.c_uint64 * world)(*[d * per_peer for d in range(world)])
nb = (C.c_uint64 * world)(*[per_peer] * world)
got = (C.c_uint64 * world)()


def ce_issue():
    # the raw byte all-to-all API: staging copy in, exchange, copy out, host syncs
    _lib.call("fsx_a2a_ce", eng.h, C.c_void_p(send.data_ptr()), offs, nb, C.c_void_p(recv.data_ptr()), per_peer, got,
              C.c_void_p(side.cuda_stream))


def staged_issue():
    # the exchange as the engine's protocol runs it (payload already in the windows)
    _lib.call("fsx_engine_a2a_staged", eng.h, per_peer, C.c_void_p(side.cuda_stream))


for key, fn in (("fsx_copy_engine_protocol", staged_issue), ("fsx_a2a_ce_api", ce_issue)):
    try:
        out[key] = measure(fn, key)
    except Exception as e:  # noqa: BLE001
        out[key] = {"error": str(e)[:200]}
eng.close()
if rank == 0:
    print(json.dumps(out), flush=True)
dist.barrier()
dist.destroy_process_group()
