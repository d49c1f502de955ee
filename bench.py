"""Benchmark of the B200-native FreeScale embedding hot path.

One step = one prioritized embedding iteration (PrioritizedEmbedding.forward
of batch i with batch i+1 prefetched, then backward with the collision-first
SGD update) of one rank's share of BASELINE.json config 4: 8 tables x 10M rows
x 256 fp32 per GPU (64 tables over 8 GPUs), 2,048 UIH samples per rank per
iteration (16K global at 8 GPUs), power-law UIH lengths 16..8192, Zipf(1.1)
rows, row-wise `gid mod N` sharding. Weak scaling: per-GPU work is fixed.

metric: lookup+update rows/s = (occurrence rows served batch-major + unique
rows updated) per second, whole job. Also reported: exposed embedding-comm
ms/iter (compute-stream stall on embedding traffic, max over ranks).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl fsx|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...     (N > 1)
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
# keep NCCL's version banner off stdout (the bench prints one JSON line); an
# explicit NCCL_DEBUG=INFO / TRACE request is kept
if os.environ.get("NCCL_DEBUG", "VERSION").upper() == "VERSION":
    os.environ["NCCL_DEBUG"] = "WARN"
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

import numpy as np  # noqa: E402

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="fsx", choices=["fsx", "reference"])
    ap.add_argument("--mode", default="prio", choices=["prio", "sync"])
    ap.add_argument("--transport", default=None, choices=["ce", "nccl"],
                    help="all-to-all transport (default: ce for prio, nccl for the sync baseline)")
    ap.add_argument("--tables-per-rank", type=int, default=8)
    ap.add_argument("--rows-per-table", type=int, default=10_000_000)
    ap.add_argument("--dim", type=int, default=256)
    ap.add_argument("--samples", type=int, default=2048, help="UIH samples per rank per iteration")
    ap.add_argument("--reduce-chunk", type=int, default=64)
    ap.add_argument("--presum", type=int, default=-1,
                    help="prioritized: pre-sum collision gradients per (source, row) before the "
                         "collision all-to-all (-1: on when N>1)")
    ap.add_argument("--seed", type=int, default=20261018)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-phases", type=int, default=1)
    ap.add_argument("--cfg5-direct", type=int, default=0,
                    help="config 5: also the arms with the collision chain's transfers as direct NVLink stores "
                         "(fsx_engine_set_eco_direct mask 3; opt-in, see DESIGN.md §6)")
    ap.add_argument("--cfg5-partition", choices=("vbs", "fbs"), default="fbs",
                    help="config 5 load balancer: FBS (default) or VBS")
    ap.add_argument("--cfg5-alpha", type=float, default=2.0, help="VBS weight exponent (uih_len^alpha)")
    ap.add_argument("--cfg5", type=int, default=-1,
                    help="also run config 5 (embedding + HSTU-style victim; blocking NCCL vs "
                         "prioritized copy-engine); default: on when N > 1")
    ap.add_argument("--victim-layers", type=int, default=1)
    ap.add_argument("--cfg1", type=int, default=-1,
                    help="also time config 1 (1M x 128 fp32, Zipf batches of 4,096, one rank) beside the "
                         "reference at full size; default: on at N = 1")
    ap.add_argument("--cfg2", type=int, default=-1,
                    help="also time config 2 (FBS / VBS over 65,536 samples, 8 ranks) on the GPU beside the "
                         "reference's FBS; default: on at N = 1")
    ap.add_argument("--cfg3", type=int, default=-1,
                    help="also time config 3's pooled lookup + scatter (8 x 10M x 128 fp32 tables, bags of "
                         "(sample, table)); default: on at N = 1")
    ap.add_argument("--cfg2-ref-vbs", action="store_true",
                    help="time the reference's VBS (alpha 1 and 2, ~60-80 s each) live instead of citing "
                         "profiles/r2_cfg2_reference.json")
    return ap.parse_args()


# ---- workload -----------------------------------------------------------------
def batches_for(args, rank, world, iters, with_lens=False):
    from paper_2604_24073_b200 import workload
    tables = args.tables_per_rank * world
    out, lens = [], []
    for i in range(iters):
        ln, ids = workload.cfg_tokens(args.seed, i, rank, args.samples, tables, args.rows_per_table)
        out.append(ids)
        lens.append(ln)
    return (out, lens) if with_lens else out


def balance_batches(args, world, rank, iters, first, ctx):
    """Config 5's load-balancing stage on the GPU: for every iteration >=
    first, the global batch (every rank's UIH samples, regenerated
    deterministically here) is partitioned across ranks by uih length and
    this rank keeps its assigned samples in receive order. --cfg5-partition
    vbs (default): variable batch sizes, min-max cut of uih_len^alpha
    (partition.cpp:178-209, alpha 2: the cost model's quadratic term
    dominates at these lengths), so every rank's compute is close to equal;
    fbs: equal sample counts, snake order (partition.cpp:157-176)."""
    from paper_2604_24073_b200 import partition as P
    from paper_2604_24073_b200 import workload
    tables = args.tables_per_rank * world
    out_ids, out_lens = {}, {}
    for i in range(first, iters):
        per = [workload.cfg_tokens(args.seed, i, r, args.samples, tables, args.rows_per_table)
               for r in range(world)]
        metas = [P.GlobalSampleMeta(r, k, int(l)) for r in range(world) for k, l in enumerate(per[r][0])]
        if getattr(args, "cfg5_partition", "fbs") == "fbs":
            plan = P.fbs_partition(metas, world, ctx=ctx)
        else:
            plan = P.vbs_partition(metas, world, getattr(args, "cfg5_alpha", 2.0), ctx=ctx)
        offs = [np.concatenate([[0], np.cumsum(per[r][0].astype(np.int64))]) for r in range(world)]
        ids, lens = [], []
        for g in plan.receive_order[rank]:
            m = metas[int(g)]
            o = offs[m.origin_rank]
            ids.append(per[m.origin_rank][1][o[m.local_index]:o[m.local_index + 1]])
            lens.append(m.uih_len)
        out_ids[i] = np.concatenate(ids) if ids else np.zeros(0, np.uint64)
        out_lens[i] = np.asarray(lens, np.uint64)
    return out_ids, out_lens


def work_rows(batches, world=1):
    """occurrences served + unique rows updated, per iteration (rank-local
    batches; for world>1 the unique rows are counted per owner shard by the
    caller's all-reduce, here approximated by the rank's own unique ids)."""
    return [int(b.size) + int(np.unique(b).size) for b in batches]


# ---- clocks ---------------------------------------------------------------------
class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (FileNotFoundError, OSError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if len(r) > 2 and r[1].replace('.', '', 1).isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) > 2 and r[2].replace('.', '', 1).isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4)
                          if len(r) > 5 + k and r[5 + k].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ---- config 5: synthetic HSTU-style attention "victim" ---------------------------
class Victim:
    """The dense model between embedding forward and backward (config 5): a
    compute kernel whose per-rank cost follows the reference's CostModel,
    c0 + c1*sum(L) + c2*sum(L^2) (sim.hpp:24-35; attention mode c2 > 0,
    SPEC.md:679), realised as r back-to-back bf16 tensor-core GEMMs of one
    fixed shape ([4096 x 4096] x [4096 x 1024], ~34 GFLOP each) so it runs
    at cuBLAS speed with no per-shape planning. The unit count r is the cost
    in microseconds / unit_us, unit_us measured once. Its SMs are what an
    SM-resident collective (NCCL) competes with; copy-engine traffic does
    not."""

    def __init__(self, dev, c0=50.0, c1=0.004, c2=1e-5):
        import torch
        self.torch = torch
        g = torch.Generator(device=dev)
        g.manual_seed(5)
        self.a = torch.randn(4096, 4096, generator=g, device=dev).to(torch.bfloat16)
        self.b = torch.randn(4096, 1024, generator=g, device=dev).to(torch.bfloat16)
        self.c = torch.empty(4096, 1024, device=dev, dtype=torch.bfloat16)
        self.c0, self.c1, self.c2 = c0, c1, c2
        for _ in range(20):
            torch.matmul(self.a, self.b, out=self.c)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(100):
            torch.matmul(self.a, self.b, out=self.c)
        e1.record()
        torch.cuda.synchronize()
        self.unit_us = e0.elapsed_time(e1) * 1e3 / 100
        # one unit size for every rank (same GPUs): the victim's per-rank time
        # then follows the cost model alone, not each GPU's calibration noise
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
            t = torch.tensor([self.unit_us], dtype=torch.float64, device=dev)
            dist.all_reduce(t)
            self.unit_us = float(t.item()) / dist.get_world_size()

    def cost_us(self, lens):
        lens = np.asarray(lens, np.float64)
        return self.c0 + self.c1 * float(lens.sum()) + self.c2 * float((lens * lens).sum())

    def run(self, lens):
        r = max(1, int(round(self.cost_us(lens) / self.unit_us)))
        for _ in range(r):
            self.torch.matmul(self.a, self.b, out=self.c)
        return r


# ---- CPU baseline (the reference library, oracle/_ref) --------------------------
def host_info():
    """The GPU box's host: core count and CPU model."""
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model}


def cpu_reference(args, world_threads, sample_samples, iters=5):
    """The reference's PrioritizedEmbedding (embedding.cpp:301-607) on an
    InProcessFabric with one thread per rank, tables shrunk to 125K rows each
    (the full 10M-row tables do not fit host RAM in f64), the same token stream
    folded onto the shrunk tables, `sample_samples` samples per rank per
    iteration. Returns rows/s over the steady iterations (iteration 0 is the
    synchronized bootstrap)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import Reference
    from paper_2604_24073_b200 import workload
    kind = "reference"
    R = Reference() if Reference.available() else None
    if R is None:
        raise RuntimeError("oracle/_ref/libfsref.so not built")
    small_rows = 125_000
    tables = args.tables_per_rank * world_threads
    batches = []
    for i in range(iters):
        row = []
        for r in range(world_threads):
            lens, ids = workload.cfg_tokens(args.seed, i, r, sample_samples, tables, args.rows_per_table)
            t = ids // np.uint64(args.rows_per_table)
            rr = ids % np.uint64(args.rows_per_table)
            row.append(t * np.uint64(small_rows) + (rr % np.uint64(small_rows)))
        batches.append(row)
    total_rows = tables * small_rows
    us = R.bench_engine(True, world_threads, batches, total_rows, args.dim, 0.05, 7)
    steady = list(range(1, iters - 1)) or [iters - 1]
    work = 0
    for i in steady:
        for r in range(world_threads):
            work += batches[i][r].size
        allids = np.concatenate(batches[i])
        work += np.unique(allids).size
    secs = sum(us[i] for i in steady) * 1e-6
    return {"value": work / secs, "unit": "rows/s", "cores": world_threads, "kind": kind,
            "sample": (f"reference PrioritizedEmbedding, {world_threads} rank thread(s) (one per rank, as the "
                       f"reference runs), {sample_samples} samples/rank/iter (~{batches[1][0].size} ids, the GPU "
                       f"arm's shape), {args.tables_per_rank * world_threads} tables x {small_rows} rows x "
                       f"{args.dim} f64 (the 10M-row tables folded to fit host RAM), {len(steady)} steady "
                       f"iteration(s) timed"),
            "host": host_info()}


def reference_arm(args, world, rank):
    """The reference's own CPU path on the GPU arm's shape: one rank thread
    per GPU rank (the reference runs exactly one thread per rank,
    comm.cpp:140-149), the GPU arm's samples per rank, its tables folded to
    fit host RAM, bootstrap + 3 steady + final iteration per step."""
    if rank != 0:
        return
    threads = max(1, world)
    vals = []
    t0 = time.time()
    for k in range(args.steps):
        r = cpu_reference(args, threads, args.samples, iters=5)
        vals.append(r["value"])
        if time.time() - t0 > 150:
            break
    value = float(np.median(vals))
    line = {"metric": "lookup+update rows/s", "value": value, "unit": "rows/s", "n_gpus": world,
            "steps": len(vals), "warmup": args.warmup, "higher_is_better": True, "impl": "reference",
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": "BASELINE config4 per-GPU share (the GPU arm's samples per rank and tables "
                                   "per rank; rows folded to fit host RAM)",
                       "samples_per_rank": args.samples, "tables": args.tables_per_rank * threads,
                       "parallelism": f"{threads} rank thread(s)"},
            "cpu_baseline": {"value": value, "unit": "rows/s", "cores": threads, "kind": "reference",
                             "sample": r["sample"], "host": r["host"]},
            "e2e": {"value": value, "unit": "rows/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "vs_baseline": None}
    print(json.dumps(line), flush=True)


# ---- config 5: SM contention of the all-to-all transports --------------------------
def contention(eng, victim, lens, dev, world, per_peer_bytes=32 << 20, reps=4):
    """The victim's own duration (CUDA events on its stream) alone, then with
    all-to-all traffic running concurrently on another stream: (a) the
    copy-engine all-to-all (fsx_engine_a2a_staged: the engine's windows,
    cudaMemcpyAsync peer copies + stream memory-op flags, no kernels), (b) NCCL's all-to-all
    (torch.distributed.all_to_all_single: SM-resident kernels). Also the
    transfers' own rate (bytes out per GPU / time) while the victim runs and
    alone. Collective: every rank calls it."""
    import ctypes as C
    import torch
    import torch.distributed as dist
    from paper_2604_24073_b200 import _lib
    n64 = per_peer_bytes // 8
    send = torch.zeros(world * n64, dtype=torch.int64, device=dev)
    recv = torch.empty(world * n64, dtype=torch.int64, device=dev)
    side = torch.cuda.Stream(device=dev)
    offs = (C.c_uint64 * world)(*[d * per_peer_bytes for d in range(world)])
    nb = (C.c_uint64 * world)(*[per_peer_bytes] * world)
    got = (C.c_uint64 * world)()

    def ce_once():
        # the engine's exchange as its protocol runs it: payload already in
        # the staging windows, copy-engine peer copies + flags, no host sync
        _lib.call("fsx_engine_a2a_staged", eng.h, per_peer_bytes, C.c_void_p(side.cuda_stream))

    def nccl_once():
        with torch.cuda.stream(side):
            dist.all_to_all_single(recv, send)

    def agree_max(x, op=None):
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def per_call_ms(fn, n=6):
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        for _ in range(n):
            fn()
        side.synchronize()
        return agree_max((time.perf_counter() - t0) * 1e3 / n)

    def victim_ms(traffic, calls=0):
        """The victim on the compute stream while this rank issues exactly
        `calls` all-to-alls (the same count on every rank: collectives must
        match) on the side stream."""
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        dist.barrier()
        cur = torch.cuda.current_stream(dev)
        e0.record(cur)
        for _ in range(reps):
            victim.run(lens)
        e1.record(cur)
        t0 = time.perf_counter()
        for c in range(calls):
            traffic()
            if c % 4 == 3:
                side.synchronize()
        side.synchronize()
        wall = (time.perf_counter() - t0) * 1e3
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps, wall

    def alone_rate(fn, n=8):
        return (world - 1) * per_peer_bytes / (per_call_ms(fn, n) * 1e-3) / 1e9

    out = {"per_peer_mib": per_peer_bytes >> 20}
    ce_once(); nccl_once(); side.synchronize()  # warm both paths
    alone = victim_ms(None)[0]
    out["victim_ms_alone"] = round(alone, 4)
    for name, fn in (("ce", ce_once), ("nccl", nccl_once)):
        # enough calls to cover the victim's whole run, agreed across ranks
        calls = int(np.ceil(agree_max(alone * reps / per_call_ms(fn))))
        v, wall = victim_ms(fn, calls)
        out[f"victim_ms_with_{name}_a2a"] = round(v, 4)
        out[f"{name}_a2a_calls"] = calls
        out[f"{name}_a2a_gbs_out_per_gpu_during_victim"] = round((world - 1) * per_peer_bytes * calls /
                                                                 (wall * 1e-3) / 1e9, 1)
    out["ce_a2a_gbs_out_per_gpu_alone"] = round(alone_rate(ce_once), 1)
    out["nccl_a2a_gbs_out_per_gpu_alone"] = round(alone_rate(nccl_once), 1)
    out["victim_slowdown_pct"] = {
        "ce": round(100.0 * (out["victim_ms_with_ce_a2a"] / out["victim_ms_alone"] - 1), 2),
        "nccl": round(100.0 * (out["victim_ms_with_nccl_a2a"] / out["victim_ms_alone"] - 1), 2)}
    return out


# ---- config 3: pooled lookup + scatter ---------------------------------------------
def run_cfg3(args, ctx, dev, W, K, rank=0):
    """BASELINE config 3's operator at one GPU's share: 8 tables x 10M rows x
    128 fp32 (41 GB), 2,048 UIH samples per iteration, every (sample, table)
    bag sum-pooled (PooledEmbedding: fused pooled gather + the backward's row
    plan), then each bag's gradient scattered to its tokens and applied
    (collision-free SGD with the chunk association). All 8 tables are local at
    one rank (table-wise ownership gives one table per GPU at 8 GPUs; the
    owner-side work per bag is the same). Ids resident; inputs >> L2."""
    import torch
    from paper_2604_24073_b200 import embedding as E
    from paper_2604_24073_b200 import workload
    T, R, dim = 8, args.rows_per_table, 128
    iters = W + K + 1
    bag_ids, bag_offs, tokens = [], [], []
    for i in range(iters):
        lens, ids = workload.cfg_tokens(args.seed + 3, i, rank, args.samples, T, R)
        t = ids // np.uint64(R)
        smp = np.repeat(np.arange(lens.size), lens.astype(np.int64))
        order = np.lexsort((np.arange(ids.size), t, smp))  # bags = (sample, table), token order kept
        key = smp[order] * T + t[order].astype(np.int64)
        counts = np.bincount(key, minlength=lens.size * T)
        bag_ids.append(ids[order])
        bag_offs.append(np.concatenate([[0], np.cumsum(counts)]).astype(np.uint64))
        tokens.append(ids.size)
    shard = E.ShardView(E.TableGeometry(T * R, dim, 1), 0, 0.05, 7, dtype="f32", ctx=ctx)
    cap = max(tokens) + 1
    pe = E.PooledEmbedding(shard, max_occurrences=cap, max_bags=args.samples * T, reduce_chunk=args.reduce_chunk)
    d_ids = [torch.from_numpy(b.view(np.int64)).to(dev) for b in bag_ids]
    d_offs = [torch.from_numpy(o.view(np.int64)).to(dev) for o in bag_offs]
    out = torch.empty((args.samples * T, dim), dtype=torch.float32, device=dev)
    g = (torch.rand((args.samples * T, dim), device=dev) - 0.5) * 1e-3
    s = torch.cuda.Stream(device=dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ef, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fwd_ms = bwd_ms = 0.0
    with torch.cuda.stream(s):
        for i in range(W):
            pe.forward(d_ids[i], d_offs[i], out=out, stream=s)
            pe.backward(g, stream=s)
        s.synchronize()
        e0.record(s)
        for i in range(W, W + K):
            pe.forward(d_ids[i], d_offs[i], out=out, stream=s)
            pe.backward(g, stream=s)
        e1.record(s)
        s.synchronize()
        # forward / backward split (separate pass: events between the halves)
        for i in range(W, W + K):
            ef.record(s)
            pe.forward(d_ids[i], d_offs[i], out=out, stream=s)
            eb.record(s)
            pe.backward(g, stream=s)
            s.synchronize()
            fwd_ms += ef.elapsed_time(eb)
    ms = e0.elapsed_time(e1) / K
    fwd_ms /= K
    ntok = float(np.mean(tokens[W:W + K]))
    uq = float(np.mean([np.unique(b).size for b in bag_ids[W:W + K]]))
    nb = args.samples * T
    rb = dim * 4
    # forward: each token's id + row read, each bag row written; the
    # backward's sort/plan traffic is excluded (index work, bytes << rows)
    fwd_bytes = ntok * (8 + rb) + nb * rb
    peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else PEAKS_FALLBACK["hbm_gbs"]
    pe.close()
    del shard
    torch.cuda.synchronize()
    return {"workload": "BASELINE config3 operator, one GPU's share: 8 tables x 10M x 128 fp32, 2,048 UIH samples, "
                        "sum-pooled (sample, table) bags, bag gradients scattered to tokens + row update",
            "bags_per_iter": nb, "tokens_per_iter": int(ntok), "unique_rows_per_iter": int(uq),
            "ms_per_iter": round(ms, 4), "forward_ms": round(fwd_ms, 4),
            "rows_per_s": round((ntok + uq) / (ms * 1e-3), 1),
            "forward_roofline": {"bound": "hbm", "achieved": round(fwd_bytes / (fwd_ms * 1e-3) / 1e9, 1),
                                 "peak": peak, "unit": "GB/s",
                                 "frac": round(fwd_bytes / (fwd_ms * 1e-3) / 1e9 / peak, 4),
                                 "note": "forward includes the backward's row sort + plan (index work)"}}


# ---- config 1 and config 2 beside the reference ----------------------------------
def run_cfg1(args, ctx, dev, W, K):
    """BASELINE config 1: one 1M x 128 fp32 table, Zipf(1.1) batches of 4,096
    ids, one rank: collision detection + prioritized (collision-first)
    update per iteration, through the public API with resident ids. The
    reference runs the same batches at full size (1M x 128 f64) on one host
    core (Reference.bench_engine, PrioritizedEmbedding under InProcessFabric)."""
    import torch
    from paper_2604_24073_b200 import embedding as E
    from paper_2604_24073_b200 import workload
    rows, dim, n, seed = 1_000_000, 128, 4096, 20261019
    iters = W + K + 2
    batches = [workload.zipf_batch(seed, n, rows, offset=n * i) for i in range(iters)]
    shard = E.ShardView(E.TableGeometry(rows, dim, 1), 0, 0.05, seed, dtype="f32", ctx=ctx)
    eng = E.PrioritizedEmbedding(shard, max_occurrences=n, reduce_chunk=args.reduce_chunk)
    eng.set_ids_ready(True)
    d = [torch.from_numpy(b.view(np.int64)).to(dev) for b in batches]
    out = torch.empty((n, dim), dtype=torch.float32, device=dev)
    g = (torch.rand((n, dim), device=dev) - 0.5) * 1e-3
    s = torch.cuda.Stream(device=dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        for i in range(W):
            eng.forward(d[i], d[i + 1], out=out, stream=s)
            eng.backward(g, stream=s)
        eng.join(s)
        s.synchronize()
        e0.record(s)
        for i in range(W, W + K):
            eng.forward(d[i], d[i + 1], out=out, stream=s)
            eng.backward(g, stream=s)
        eng.join(s)
        e1.record(s)
        s.synchronize()
    ms = e0.elapsed_time(e1) / K
    rows_it = float(np.mean([b.size + np.unique(b).size for b in batches[W:W + K]]))
    eng.close()
    del shard
    res = {"workload": "BASELINE config1: 1M x 128 fp32, Zipf(1.1) batches of 4,096 ids, 1 rank, collision "
                       "detect + prioritized row-wise update (forward + backward per iteration, ids resident)",
           "gpu_us_per_iter": round(ms * 1e3, 2), "gpu_rows_per_s": round(rows_it / (ms * 1e-3), 1)}
    if not args.no_cpu_baseline:
        try:
            sys.path.insert(0, os.path.join(ROOT, "oracle"))
            from oracle import Reference
            R = Reference()
            cb = [[b] for b in batches[:5]]
            us = R.bench_engine(True, 1, cb, rows, dim, 0.05, seed)
            steady = float(np.mean(us[1:4]))
            res["reference"] = {"us_per_iter": round(steady, 1), "rows_per_s": round(rows_it / (steady * 1e-6), 1),
                                "cores": 1, "kind": "reference",
                                "sample": "reference PrioritizedEmbedding at full size (1M x 128 f64), 1 rank "
                                          "thread, the same batches, steady iterations 1-3",
                                "host": host_info()}
            res["speedup_gpu_over_reference"] = round(steady / (ms * 1e3), 1)
        except Exception as ex:  # noqa: BLE001
            res["reference"] = {"unavailable": str(ex)}
    return res


def run_cfg2(args, ctx):
    """BASELINE config 2: 65,536 UIH samples (8 ranks x 8,192, power-law
    lengths 16-8192) partitioned over 8 ranks by FBS and by VBS (alpha 1, 2)
    with the GPU partitioner through the public API (host lists in, plan
    out), wall time per call, beside the reference's own partitioners on the
    same metas (FBS live; VBS live with --cfg2-ref-vbs, else the committed
    measurement of the reference on this pool's host)."""
    import torch
    from paper_2604_24073_b200 import partition as P
    from paper_2604_24073_b200 import workload
    gold = os.path.join(ROOT, "tests", "golden", "cfg2_partition.npz")
    if os.path.exists(gold):
        z = np.load(gold)
        lens, origin, local = z["lens"], z["origin"], z["local"]
        src = "tests/golden/cfg2_partition.npz (the reference's own generator, make_cfg2_golden.py)"
    else:
        lens = workload.uih_lengths(20261020, 65536)
        origin = np.repeat(np.arange(8), 8192).astype(np.int32)
        local = np.tile(np.arange(8192), 8).astype(np.int32)
        src = "workload.uih_lengths(20261020, 65536)"
    out = {"workload": "BASELINE config2: 65,536 UIH samples, power-law lengths 16..8192, 8 ranks", "inputs": src,
           "call": "partition.{fbs,vbs}_partition_arrays: the C ABI's argument form (host arrays in, plan out)"}
    gpu = {}
    for name, fn in (("fbs", lambda: P.fbs_partition_arrays(lens, origin, local, 8, ctx=ctx)),
                     ("vbs_alpha1", lambda: P.vbs_partition_arrays(lens, origin, local, 8, 1.0, ctx=ctx)),
                     ("vbs_alpha2", lambda: P.vbs_partition_arrays(lens, origin, local, 8, 2.0, ctx=ctx))):
        fn()  # warm
        torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            ts.append((time.perf_counter() - t0) * 1e3)
        gpu[name] = round(float(np.median(ts)), 3)
    out["gpu_ms_per_call"] = gpu
    if args.no_cpu_baseline:
        return out
    try:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        from oracle import Reference
        R = Reference()
        t0 = time.perf_counter()
        R.fbs(lens, origin, local, 8)
        ref = {"fbs": round((time.perf_counter() - t0) * 1e3, 3)}
        if args.cfg2_ref_vbs:
            for a in (1.0, 2.0):
                t0 = time.perf_counter()
                R.vbs(lens, origin, local, 8, a)
                ref[f"vbs_alpha{int(a)}"] = round((time.perf_counter() - t0) * 1e3, 1)
            ref["vbs_source"] = "timed live in this run"
        else:
            cached = os.path.join(ROOT, "profiles", "r2_cfg2_reference.json")
            if os.path.exists(cached):
                c = json.load(open(cached))
                for k in ("vbs_alpha1", "vbs_alpha2"):
                    ref[k] = c["reference_ms_per_call"][k]
                ref["vbs_source"] = ("profiles/r2_cfg2_reference.json (the reference's VBS timed on this "
                                     "pool's GPU-box host, bench.py --cfg2-ref-vbs)")
        out["reference_ms_per_call"] = ref
        out["reference_cores"] = 1
        out["host"] = host_info()
        out["speedup_gpu_over_reference"] = {k: round(ref[k] / gpu[k], 1) for k in gpu if k in ref}
    except Exception as ex:  # noqa: BLE001
        out["reference_ms_per_call"] = {"unavailable": str(ex)}
    return out


# ---- GPU arm ----------------------------------------------------------------------
def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        reference_arm(args, world, rank)
        return

    import torch
    import torch.distributed as dist
    from paper_2604_24073_b200 import _lib
    from paper_2604_24073_b200 import embedding as E
    from paper_2604_24073_b200.comm import DeviceFabric, ProcessGroupFabric

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        fabric = ProcessGroupFabric(rank, world, local)
    else:
        fabric = DeviceFabric(1, [local])
    comm = fabric.communicator(rank)

    W, K = max(args.warmup, 3), args.steps
    cfg5 = args.cfg5 if args.cfg5 >= 0 else int(world > 1)
    iters = W + 3 * K + 4 + (4 * K + 4 if cfg5 else 0)
    t_gen = time.time()
    batches, blens = batches_for(args, rank, world, iters, with_lens=True)
    ctx = E.Context(local, rank, world)
    cfg5_first = W + 3 * K + 2
    if cfg5 and world > 1 and args.mode == "prio":
        bi, bl = balance_batches(args, world, rank, iters, cfg5_first, ctx)
        for i in bi:
            batches[i], blens[i] = bi[i], bl[i]
    t_gen = time.time() - t_gen
    cap = int(max(b.size for b in batches) * 1.05) + 1024
    if world > 1:  # every rank's engine must use the same capacity (same window layout)
        t = torch.tensor([cap], dtype=torch.int64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        cap = int(t.item())
    tables = args.tables_per_rank * world
    total_rows = tables * args.rows_per_table
    geom = E.TableGeometry(total_rows, args.dim, world)
    t0 = time.time()
    shard = E.ShardView(geom, rank, 0.05, 7, dtype="f32", ctx=ctx)
    t_init = time.time() - t0
    cls = E.PrioritizedEmbedding if args.mode == "prio" else E.SynchronizedEmbedding
    transport = args.transport or ("ce" if args.mode == "prio" or world == 1 else "nccl")
    presum = args.mode == "prio" and (args.presum > 0 or (args.presum < 0 and world > 1))
    kw = {"presum": True} if presum else {}
    eng = cls(shard, comm, max_occurrences=cap, reduce_chunk=args.reduce_chunk, transport=transport, **kw)

    stream = torch.cuda.Stream(device=dev)
    if hasattr(eng, "set_ids_ready"):
        eng.set_ids_ready(True)  # the resident id tensors are uploaded before timing
    d_ids = [torch.from_numpy(b.view(np.int64)).to(dev) for b in batches]
    h_ids = [torch.from_numpy(b.view(np.int64)).pin_memory() for b in batches]
    slots = [torch.empty(cap, dtype=torch.int64, device=dev) for _ in range(3)]
    maxn = max(b.size for b in batches)
    out = torch.empty((maxn, args.dim), dtype=torch.float32, device=dev)
    gen = torch.Generator(device=dev)
    gen.manual_seed(1)
    grads_full = (torch.rand((maxn, args.dim), generator=gen, device=dev, dtype=torch.float32) - 0.5) * 1e-3
    res_h = torch.empty((2, 8), dtype=torch.float32).pin_memory()

    def upload(i):
        """H2D of iteration i's ids from pinned host memory into slot i % 3."""
        n = batches[i].size
        slots[i % 3][:n].copy_(h_ids[i], non_blocking=True)
        return slots[i % 3][:n]

    def step(i, e2e=False):
        n = batches[i].size
        if args.mode == "prio":
            if e2e:
                # the next batch's ids go from pinned host memory straight to
                # the engine's side lane (its own H2D)
                eng.forward(h_ids[i], h_ids[i + 1], out=out[:n], stream=stream)
            else:
                eng.forward(d_ids[i], d_ids[i + 1], out=out[:n], stream=stream)
        else:
            cur = upload(i) if e2e else d_ids[i]
            eng.forward(cur, out=out[:n], stream=stream)
        eng.backward(grads_full[:n], stream=stream)
        if e2e:
            # the step's result read back: last served row's first 8 values
            res_h[i % 2].copy_(out[n - 1, :8], non_blocking=True)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    with torch.cuda.stream(stream):
        # warm-up (iteration 0 is the synchronized bootstrap)
        for i in range(W):
            step(i)
        barrier()
        launches0 = ctx.launches()
        if args.mode == "prio":
            eng.exposed_ms()  # reset the accumulator
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with Clocks(local) as clk:
            barrier()
            ev0.record(stream)
            th0 = time.perf_counter()
            for i in range(W, W + K):
                step(i)
            host_enqueue_ms = (time.perf_counter() - th0) * 1e3
            eng.join(stream)  # every engine lane's work of the timed steps inside the window
            ev1.record(stream)
            barrier()
        ms_dev = ev0.elapsed_time(ev1)
        launches = ctx.launches() - launches0
        exp_timed = eng.exposed_ms() / K
        # phase timing (CUDA events around every phase, on the stream each
        # runs on) in a separate section of K steps, so the event overhead is
        # not inside the timed region above
        prof_lo = W + K
        phases = {}
        span_us = span_n = None
        if args.profile_phases and hasattr(eng, "set_profiling"):
            eng.set_profiling(True)
            eng.phase_ms()  # reset
            ctx.kernel_span(True)  # the row-update kernel's own device-side span
        for i in range(prof_lo, prof_lo + K):
            step(i)
        barrier()
        if args.profile_phases and hasattr(eng, "set_profiling"):
            phases = eng.phase_ms()
            eng.set_profiling(False)
            span_us, span_n = ctx.kernel_span(False)
        eng.exposed_ms()
        # end-to-end: host ids -> device each step, stats read back (two
        # untimed steps first: the switch from resident to host ids)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for i in range(W + 2 * K, W + 2 * K + 2):
            step(i, e2e=True)
        first_e2e = W + 2 * K + 2
        barrier()
        e0.record(stream)
        n_e2e = 0
        for i in range(first_e2e, min(first_e2e + K, iters - 1)):
            step(i, e2e=True)
            n_e2e += 1
        eng.join(stream)
        e1.record(stream)
        barrier()
        ms_e2e = e0.elapsed_time(e1)
    stats = eng.stats() if args.mode == "prio" else []

    # ---- config 5: embedding + victim, blocking NCCL vs prioritized CE ----
    cfg5_out = None
    if cfg5 and args.mode == "prio":
        it0 = first_e2e + n_e2e  # next iteration of the prioritized engine
        assert world == 1 or it0 >= cfg5_first
        victim = Victim(dev)
        vt0, vt1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        res = {}
        with torch.cuda.stream(stream):
            # (0) victim alone (no embedding traffic): its undisturbed time
            barrier()
            vt0.record(stream)
            for i in range(it0, it0 + K):
                victim.run(blens[i])
            vt1.record(stream)
            barrier()
            victim_alone = vt0.elapsed_time(vt1) / K
            # dense synchronisation of a data-parallel step (the model's
            # gradient all-reduce, 1 MiB here) after the victim, before the
            # embedding backward — the synchronized variant of every arm:
            # ranks leave the dense part together, so the exposed embedding
            # time no longer carries the wait for the slowest rank's victim
            dense = torch.zeros(1 << 18, dtype=torch.float32, device=dev)

            def dense_sync():
                if world > 1:
                    dist.all_reduce(dense)

            def prio_loop(first, sync):
                eng.join(stream)
                stream.synchronize()
                eng.exposed_ms()
                barrier()
                e0.record(stream)
                for i in range(first, first + K):
                    n = batches[i].size
                    eng.forward(d_ids[i], d_ids[i + 1], out=out[:n], stream=stream)
                    victim.run(blens[i])
                    if sync:
                        dense_sync()
                    eng.backward(grads_full[:n], stream=stream)
                eng.join(stream)
                e1.record(stream)
                barrier()
                return e0.elapsed_time(e1) / K, eng.exposed_ms() / K

            # (B) prioritized + copy engines, victim between forward and backward
            res["prio_ce"] = prio_loop(it0, False)
            if world > 1:
                # (B') with --cfg5-direct: the same with the collision chain's
                # transfers stored by its kernels straight into the peers'
                # windows — the pre-sum into the owners' CO_G slots, the
                # collision update into the requesters' E_co slots (SM-issued
                # NVLink stores, no copy-engine hop); then the prioritized
                # arm(s) with the dense sync
                nxt = it0 + K
                if args.cfg5_direct:
                    mask = int(os.environ.get("FSX_BENCH_DIRECT_MASK", "3"))  # (A/B: 1 = E_co only, 2 = CO_G only)
                    eng.set_eco_direct(bool(mask & 1), cog=bool(mask & 2))
                    res["prio_direct"] = prio_loop(nxt, False)
                    res["prio_direct_sync"] = prio_loop(nxt + K, True)
                    nxt += 2 * K
                    eng.set_eco_direct(False)
                res["prio_ce_sync"] = prio_loop(nxt, True)
        # (A) the blocking baseline: synchronized engine, NCCL all-to-all (N>1)
        base_tr = "nccl" if world > 1 else "ce"
        sync_eng = E.SynchronizedEmbedding(shard, comm, max_occurrences=cap,
                                           reduce_chunk=args.reduce_chunk, transport=base_tr)
        with torch.cuda.stream(stream):
            for i in range(it0, it0 + 2):
                n = batches[i].size
                sync_eng.forward(d_ids[i], out=out[:n], stream=stream)
                victim.run(blens[i])
                sync_eng.backward(grads_full[:n], stream=stream)

            def base_loop(sync):
                barrier()
                sync_eng.exposed_ms()
                e0.record(stream)
                for i in range(it0, it0 + K):
                    n = batches[i].size
                    sync_eng.forward(d_ids[i], out=out[:n], stream=stream)
                    victim.run(blens[i])
                    if sync:
                        dense_sync()
                    sync_eng.backward(grads_full[:n], stream=stream)
                e1.record(stream)
                barrier()
                return e0.elapsed_time(e1) / K, sync_eng.exposed_ms() / K

            res["sync_" + base_tr] = base_loop(False)
            if world > 1:
                res["sync_" + base_tr + "_sync"] = base_loop(True)
        sync_eng.close()
        cont = None
        if world > 1:
            with torch.cuda.stream(stream):
                eng.join(stream)
                stream.synchronize()
                cont = contention(eng, victim, blens[it0], dev, world)
        b_key = "sync_" + base_tr
        step_b = max_over_ranks(res[b_key][0])
        step_p = max_over_ranks(res["prio_ce"][0])
        exp_b = max_over_ranks(res[b_key][1])
        exp_p = max_over_ranks(res["prio_ce"][1])
        # straggler share: rank r's exposed wait includes (slowest victim - own
        # victim) spent waiting for peers' collision chains, which no transport
        # removes; report the remainder as well (per rank, then max over ranks)
        skew = max_over_ranks(victim_alone) - victim_alone
        exp_b_ns = max_over_ranks(max(0.0, res[b_key][1] - skew))
        exp_p_ns = max_over_ranks(max(0.0, res["prio_ce"][1] - skew))
        exp_d = exp_d_ns = None
        if "prio_direct" in res:
            exp_d = max_over_ranks(res["prio_direct"][1])
            exp_d_ns = max_over_ranks(max(0.0, res["prio_direct"][1] - skew))
        exp_b_sum = sum_over_ranks(res[b_key][1])
        exp_p_sum = sum_over_ranks(res["prio_ce"][1])
        sync_out = None
        if world > 1:
            # every arm with the dense all-reduce between the victim and the
            # embedding backward: exposed embedding time from a synchronized start
            sb = max_over_ranks(res[b_key + "_sync"][1])
            sync_out = {"dense_sync": "1 MiB NCCL all-reduce after the victim, before the embedding backward "
                                      "(not counted as embedding exposed time), in every arm",
                        "exposed_ms_per_iter_max_over_ranks": {b_key: round(sb, 4)},
                        "exposed_reduction_pct": {},
                        "step_ms": {b_key: round(max_over_ranks(res[b_key + "_sync"][0]), 4)}}
            for k in ("prio_ce_sync", "prio_direct_sync"):
                if k not in res:
                    continue
                x = max_over_ranks(res[k][1])
                sync_out["exposed_ms_per_iter_max_over_ranks"][k] = round(x, 4)
                sync_out["exposed_reduction_pct"][k] = round(100.0 * (1 - x / sb), 2) if sb > 0 else None
                sync_out["step_ms"][k] = round(max_over_ranks(res[k][0]), 4)
        cfg5_out = {
            "load_balancer": (("FBS (partition.cpp:157-176)" if args.cfg5_partition == "fbs" else
                               f"VBS alpha {args.cfg5_alpha} (partition.cpp:178-209)") +
                              " over the global batch of each iteration, on the GPU"
                              if world > 1 else "none (1 rank)"),
            "workload": ("config 5: config-4 embeddings + synthetic HSTU-style compute between forward and "
                         f"backward, per-rank cost c0+c1*sum(L)+c2*sum(L^2) = {victim.c0}+{victim.c1}*sum(L)+"
                         f"{victim.c2}*sum(L^2) us as bf16 GEMMs"),
            "baseline": f"SynchronizedEmbedding, blocking {base_tr.upper()} all-to-all on the compute stream",
            "freescale": "PrioritizedEmbedding, copy-engine all-to-all on side lanes (0 SMs)",
            "exposed_ms_per_iter_max_over_ranks": {b_key: round(exp_b, 4), "prio_ce": round(exp_p, 4)},
            "exposed_ms_per_iter_sum_over_ranks": {b_key: round(exp_b_sum, 4), "prio_ce": round(exp_p_sum, 4)},
            "exposed_reduction_pct": round(100.0 * (1 - exp_p / exp_b), 2) if exp_b > 0 else None,
            # the collision chain's CO_G and E_co by SM-issued NVLink stores
            # from the pre-sum and collision-update kernels (no copy-engine hop)
            "prio_direct": ({"exposed_ms_per_iter_max_over_ranks": round(exp_d, 4),
                             "exposed_reduction_pct": round(100.0 * (1 - exp_d / exp_b), 2),
                             "exposed_reduction_pct_beyond_victim_skew":
                                 round(100.0 * (1 - exp_d_ns / exp_b_ns), 2) if exp_b_ns > 0 else None,
                             "step_ms": round(max_over_ranks(res["prio_direct"][0]), 4),
                             "comm_sms": ("CO_G / E_co rows stored by the pre-sum and collision-update "
                                          "kernels' own SMs (no extra kernel); the other all-to-alls on "
                                          "the copy engines")}
                            if exp_d is not None else None),
            "exposed_ms_per_iter_beyond_victim_skew_max_over_ranks": {b_key: round(exp_b_ns, 4),
                                                                       "prio_ce": round(exp_p_ns, 4)},
            "exposed_reduction_pct_beyond_victim_skew": (round(100.0 * (1 - exp_p_ns / exp_b_ns), 2)
                                                         if exp_b_ns > 0 else None),
            "step_ms": {b_key: round(step_b, 4), "prio_ce": round(step_p, 4)},
            "victim_alone_ms": round(max_over_ranks(victim_alone), 4),
            # straggler share of the exposed wait: the slowest rank's victim
            # holds every peer's collision chain (both engines pay it)
            "victim_alone_ms_min_over_ranks": round(-max_over_ranks(-victim_alone), 4),
            # prio_ce: every inter-rank byte moves on the copy engines
            # (FSX_ECO_DIRECT is off: no kernel stores to a peer window)
            "comm_sms": {b_key: "NCCL kernels (SM-resident)" if base_tr == "nccl" else 0, "prio_ce": 0},
            "contention": cont,
            "synchronized_step": sync_out,
            "notes": ("the NCCL baseline's ids all-to-all needs host-known counts: its 8-byte size round "
                      "(comm.cpp:328-341) is followed by one stream sync, inside the baseline's exposed window"),
        }

    ms_dev = max_over_ranks(ms_dev)
    ms_e2e = max_over_ranks(ms_e2e)
    def rows_of(lo, hi):
        """occurrences served + unique rows updated on this rank's shard:
        U_i of this shard is IterationStats[i-1].unique_next_rows."""
        occ = sum(int(batches[i].size) for i in range(lo, hi))
        if stats:
            upd = sum(int(stats[i - 1].unique_next_rows) for i in range(lo, hi))
        else:
            upd = sum(int(np.unique(batches[i]).size) for i in range(lo, hi))
        return occ + upd

    rows_timed = rows_of(W, W + K)
    rows_e2e = rows_of(first_e2e, first_e2e + n_e2e)
    rows_timed = sum_over_ranks(rows_timed)
    rows_e2e = sum_over_ranks(rows_e2e)
    value = rows_timed / (ms_dev * 1e-3)
    e2e_value = rows_e2e / (ms_e2e * 1e-3)
    exposed_ms = max_over_ranks(exp_timed)
    exposed_sum = sum_over_ranks(exp_timed)

    # roofline of the dominant row-moving phase (rank 0's view), over the
    # profiled section's batches
    rb = args.dim * 4
    timed = batches[W:W + K]
    profiled = batches[prof_lo:prof_lo + K]
    occ = sum(b.size for b in profiled)
    uq = sum(np.unique(b).size for b in profiled)
    algo = {
        # reads occ_slot + row pointer + the row, writes the row
        "merge": occ * (2 * rb + 12),
        # reads send_pos/dst/slot/flag/rank + the grad row, writes it
        "split": occ * (2 * rb + 14),
        "serve": occ * (4 * rb + 16),
        # gradient rows in (+ perm / source / rank / pointer indices), each
        # unique row read and written once
        "update": occ * (rb + 24) + uq * 2 * rb,
    }
    if world == 1:
        # one rank: the whole update runs as the collision-lane update
        algo["co_update"] = algo["update"]
    peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(peaks_path):
        peaks = json.load(open(peaks_path))
        peak, peak_src = float(peaks["hbm_gbs"]), "measured"
    else:
        peak, peak_src = PEAKS_FALLBACK["hbm_gbs"], "fallback"
    roof = None
    if phases:
        cand = [(k, phases[k][0], phases[k][1]) for k in algo if k in phases and phases[k][1] > 0]
        if cand:
            name, tot_ms, spans = max(cand, key=lambda x: x[1])
            per_launch_ms = tot_ms / spans
            per_launch_bytes = algo[name] / spans
            achieved = per_launch_bytes / (per_launch_ms * 1e-3) / 1e9
            traffic = None
            tpath = os.path.join(ROOT, "profiles", "traffic.json")
            if os.path.exists(tpath):
                traffic = json.load(open(tpath)).get(f"n{world}", {}).get(name)
            roof = {"bound": "hbm", "kernel": name, "achieved": round(achieved, 1), "peak": peak,
                    "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": traffic,
                    "peak_source": peak_src, "launch_ms": round(per_launch_ms, 4),
                    "algorithmic_bytes_per_launch": int(per_launch_bytes)}
            if name == "co_update" and world == 1 and span_n == spans and span_us:
                # the same launches timed by the kernel itself (first CTA start
                # -> last CTA end, device globaltimer): the event window above
                # also holds the wait for SMs the concurrent side lane occupies
                roof["kernel_span_us"] = round(span_us, 2)
                roof["kernel_span_frac"] = round(per_launch_bytes / (span_us * 1e-6) / 1e9 / peak, 4)

    cfg1_out = cfg2_out = cfg3_out = None
    if rank == 0 and world == 1 and (args.cfg1 if args.cfg1 >= 0 else 1):
        cfg1_out = run_cfg1(args, ctx, dev, W, K)
    if rank == 0 and world == 1 and (args.cfg2 if args.cfg2 >= 0 else 1):
        cfg2_out = run_cfg2(args, ctx)
    if rank == 0 and world == 1 and (args.cfg3 if args.cfg3 >= 0 else 1):
        cfg3_out = run_cfg3(args, ctx, dev, W, K)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_reference(args, 1, args.samples, iters=5)
        except Exception as ex:  # noqa: BLE001
            cpu = {"value": None, "unit": "rows/s", "cores": 1, "kind": "reference", "sample": f"failed: {ex}"}

    if rank == 0:
        clocks = clk.summary()
        line = {
            "metric": "lookup+update rows/s",
            "value": round(value, 1),
            "unit": "rows/s",
            "n_gpus": world,
            "steps": K,
            "warmup": W,
            "ms_per_step": round(ms_dev / K, 4),
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": "BASELINE config4 per-GPU share: 8 tables x 10M rows x 256 fp32 per GPU, "
                                   "2048 UIH samples/GPU/iter (16K global at 8 GPUs), Zipf(1.1) ids, "
                                   "power-law UIH 16..8192, row-wise gid mod N, prioritized collision-first "
                                   "update",
                       "mode": args.mode, "transport": transport, "tables": tables, "rows_per_table": args.rows_per_table,
                       "dim": args.dim, "samples_per_rank": args.samples,
                       "ids_per_rank_per_iter": int(np.mean([b.size for b in timed])),
                       "reduce_chunk": args.reduce_chunk, "presum": presum, "grads": "fixed synthetic upstream gradient",
                       "l2": "inputs larger than L2 (82 GB table, ~1 GB moved per step)",
                       "parallelism": f"row-wise sharded x{world}"},
            "exposed_comm_ms_per_iter": round(exposed_ms, 4),
            "exposed_comm_ms_per_iter_sum_over_ranks": round(exposed_sum, 4),
            "e2e": {"value": round(e2e_value, 1), "unit": "rows/s",
                    "h2d_bytes_per_step": int(np.mean([b.size for b in timed])) * 8,
                    "d2h_bytes_per_step": 32},
            "gpu_launches": int(launches),
            # host time to issue the K timed steps (python + C ABI + launches);
            # close to ms_per_step means the step is host-bound
            "host_enqueue_ms_per_step": round(host_enqueue_ms / K, 4),
            "roofline": roof,
            "phases_ms_per_step": {k: round(v[0] / K, 4) for k, v in phases.items() if v[1]},
            "cpu_baseline": cpu,
            "cfg5": cfg5_out,
            "cfg1": cfg1_out,
            "cfg2": cfg2_out,
            "cfg3": cfg3_out,
            "clocks": clocks,
            "setup_s": {"workload_gen": round(t_gen, 2), "table_init": round(t_init, 2)},
            "collision_fraction": round(float(np.mean([s.collision_fraction for s in stats[W:W + K]])), 4)
            if stats else None,
        }
        print(json.dumps(line), flush=True)
    eng.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
