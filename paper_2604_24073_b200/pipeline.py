"""The five-stage training-loop harness around the embedding hot path
(pipeline.hpp:25-122, pipeline.cpp:118-323): data load
(optionally through the three-stage Balancer), forward (SynchronizedEmbedding
or PrioritizedEmbedding on the GPU), the reference's toy dense model, backward,
and the optimizer step with one synchronizing reduction of the dense gradient
sums, loss and sample count — one thread per rank, every rank on its GPU
context, collectives on the copy engines.

Determinism and parity: the embedding engines run f64 tables (bit-exact with
the reference); the toy model runs on the host in the reference's loop order
(pooled sums over a sample's rows in order, the projection summed over d in
order, gradient expressions evaluated left to right) and the dense reduction
sums ranks 0..p-1 from 0.0 as comm.cpp:418-424 does, so run() returns the
reference's full_checkpoint byte for byte (tests/test_gpu_pipeline.py against
goldens from the reference's own pipeline::run).

Not restated: the reference's logical clock, event log and per-iteration
metric records (its simulator's timing); run() returns losses, final dense
weights and the checkpoints.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import balancer as B
from . import embedding as E
from . import workload
from .comm import DeviceFabric
from .errors import ProtocolError
from .sim import CostModel


class Mode:
    Synchronized = "synchronized"
    Prioritized = "prioritized"


class ToyModel:
    """pipeline.hpp:64-81: mean-pool a sample's UIH rows, project with w,
    squared error against the label; closed-form gradients."""

    def __init__(self, dim: int, w: np.ndarray):
        self.dim = dim
        self.w = w

    @staticmethod
    def init(dim: int, seed: int) -> "ToyModel":
        # pipeline.cpp:36-42: rng_double from state seed ^ 0xd15ea5e0f1e1d
        st = (int(seed) ^ 0xD15EA5E0F1E1D) & 0xFFFFFFFFFFFFFFFF
        u = workload.rng_double(st, dim)
        return ToyModel(dim, (u - 0.5) * 0.2)

    def forward_backward(self, batch: B.Batch, emb: np.ndarray, global_samples: int):
        """pipeline.cpp:51-90 in the same evaluation order. emb: [occurrences x dim]."""
        dim, w = self.dim, self.w
        n = float(global_samples)
        loss_sum = 0.0
        dense = np.zeros(dim, np.float64)
        grads = np.zeros_like(emb)
        occ = 0
        for s in batch.samples:
            L = int(s.uih.size)
            pooled = np.zeros(dim, np.float64)
            for k in range(L):
                pooled = pooled + emb[occ + k]
            if L:
                pooled = pooled / float(L)
            y = 0.0
            for d in range(dim):
                y += float(pooled[d]) * float(w[d])
            err = y - s.label
            loss_sum += err * err
            dense = dense + (2.0 * err) * pooled
            if L:
                scale = 2.0 * err / (float(L) * n)
                grads[occ:occ + L] = scale * w
            occ += L
        if occ != emb.shape[0]:
            raise ValueError("toy model: embedding rows do not match batch occurrences")
        return loss_sum, dense, grads


@dataclass
class RunConfig:
    """pipeline.hpp:84-100"""
    mode: str = Mode.Synchronized
    balancer_enabled: bool = False
    partition: str = "fbs"
    alpha: float = 1.0
    autotune_step: int = 1
    autotune_delta: float = 0.05
    autotune_decay: float = 0.9
    prefetch_depth: int = 1
    cost: CostModel = field(default_factory=CostModel)
    table_rows: int = 1024
    dim: int = 8
    lr_embedding: float = 0.05
    lr_dense: float = 0.05
    model_seed: int = 1


@dataclass
class RunResult:
    losses: list
    final_dense: np.ndarray
    table_checkpoint: bytes
    full_checkpoint: bytes
    samples_processed: int


def _comm_for(fabric: DeviceFabric, rank: int, world: int, ctx, cap: int):
    """The rank's collective channel for the balancer and the dense reduction:
    a small engine's copy-engine windows (CeComm), the hand-off at one rank."""
    if world == 1:
        return B.LocalComm(), None
    shard = E.ShardView(E.TableGeometry(world, 1, world), rank, 0.0, 0, dtype="f64", ctx=ctx)
    eng = E.SynchronizedEmbedding(shard, fabric.communicator(rank), max_occurrences=cap)
    return B.CeComm(eng), (shard, eng)


def _all_reduce_sum(comm, v: np.ndarray) -> np.ndarray:
    """comm.cpp:390-424: every rank's vector, summed in rank order from 0.0."""
    parts = comm.all_gather_u64(np.ascontiguousarray(v, np.float64).view(np.uint64))
    out = np.zeros(v.size, np.float64)
    for p in parts:
        if p.size != v.size:
            from .errors import CollectiveError
            raise CollectiveError("all_reduce_sum: vector length mismatch across ranks")
        out = out + p.view(np.float64)
    return out


def run(iterations: list, world: int, batch_size: int, config: RunConfig,
        devices: Optional[list] = None) -> RunResult:
    """pipeline::run: iterations[i][r] = rank r's Batch of iteration i."""
    for it in iterations:
        if len(it) != world:
            raise ValueError("pipeline: iteration without one batch per rank")
    num_iters = len(iterations)
    global_samples = world * batch_size
    geom = E.TableGeometry(config.table_rows, config.dim, world)
    if num_iters == 0:
        full = E.ShardView(E.TableGeometry(config.table_rows, config.dim, 1), 0, config.lr_embedding,
                           config.model_seed, dtype="f64").values()  # initial_value table
        w = ToyModel.init(config.dim, config.model_seed).w
        tc = E.checkpoint_bytes(geom, full)
        return RunResult([], w, tc, tc + w.tobytes(), 0)
    # engine capacity: a balanced batch can hold any samples of its iteration
    cap = max(sum(b.total_uih_tokens() for b in it) for it in iterations) + 1
    comm_cap = max(1 << 16, 16 * (cap + 64 * world * batch_size))
    fabric = DeviceFabric(world, devices)
    shards: list = [None] * world
    losses = [0.0] * num_iters
    dense_out: dict = {}

    def body(rank: int) -> None:
        dev = fabric.device_of(rank)
        ctx = E.Context(dev, rank, world)
        shard = E.ShardView(geom, rank, config.lr_embedding, config.model_seed, dtype="f64", ctx=ctx)
        comm_e = fabric.communicator(rank)
        if config.mode == Mode.Synchronized:
            eng = E.SynchronizedEmbedding(shard, comm_e, max_occurrences=cap)
        else:
            eng = E.PrioritizedEmbedding(shard, comm_e, max_occurrences=cap)
        comm, keep = _comm_for(fabric, rank, world, ctx, comm_cap)
        model = ToyModel.init(config.dim, config.model_seed)
        hooks = B.HookRegistry()
        bal = None
        if config.balancer_enabled:
            bc = B.BalancerConfig(partition=config.partition, alpha=config.alpha,
                                  autotune_step=config.autotune_step, autotune_delta=config.autotune_delta,
                                  autotune_decay=config.autotune_decay,
                                  lead=config.prefetch_depth + (1 if config.mode == Mode.Prioritized else 0))
            bal = B.Balancer(comm, bc, lambda i: iterations[i][rank] if 0 <= i < num_iters else None,
                             num_iters, ctx=ctx)
            bal.install_hooks(hooks)
        import torch
        s = torch.cuda.Stream(device=dev)
        for i in range(num_iters):
            hooks.fire(B.HookPoint.DataLoad, i)
            batch = bal.take(i) if bal else iterations[i][rank]
            lengths = [int(x.uih.size) for x in batch.samples]
            hooks.fire(B.HookPoint.PreForward, i)
            ids_cur = batch.uih_ids()[0]
            with torch.cuda.stream(s):
                if config.mode == Mode.Synchronized:
                    rows = eng.forward(ids_cur, stream=s)
                else:
                    nxt = None
                    if i + 1 < num_iters:
                        nb = bal.peek(i + 1) if bal else iterations[i + 1][rank]
                        nxt = nb.uih_ids()[0]
                    rows = eng.forward(ids_cur, nxt, stream=s)
                emb = rows.double().cpu().numpy().reshape(-1, config.dim) if ids_cur.size else \
                    np.zeros((0, config.dim))
            compute_us = config.cost.compute_time_for_lengths(lengths, ctx=ctx)
            loss_sum, dense, grads = model.forward_backward(batch, emb, global_samples)
            hooks.fire(B.HookPoint.PostForward, i)
            with torch.cuda.stream(s):
                eng.backward(torch.from_numpy(grads).to(device=dev), stream=s)
            s.synchronize()
            # optimizer step: one synchronizing reduction of the dense gradient
            # sums, the loss and the sample count (pipeline.cpp:266-287)
            payload = np.concatenate([dense, [loss_sum, float(len(batch.samples))]])
            reduced = _all_reduce_sum(comm, payload)
            count = reduced[config.dim + 1]
            if count != float(global_samples):
                raise ProtocolError(f"pipeline: sample conservation violated ({count} vs {global_samples})")
            for d in range(config.dim):
                model.w[d] -= config.lr_dense * reduced[d] / float(global_samples)
            if rank == 0:
                losses[i] = reduced[config.dim] / float(global_samples)
            if bal:
                bal.report_compute_time(compute_us)
            hooks.fire(B.HookPoint.OptimizerStep, i)
        if config.mode == Mode.Prioritized:
            with torch.cuda.stream(s):
                eng.finalize(stream=s)
        s.synchronize()
        ctx.sync()
        # dense replicas must agree (pipeline.cpp:296-302)
        ws = comm.all_gather_u64(model.w.view(np.uint64))
        if any(not np.array_equal(x, ws[0]) for x in ws):
            raise ProtocolError("pipeline: dense weights diverged across ranks")
        shards[rank] = shard
        if rank == 0:
            dense_out["w"] = model.w.copy()
        eng.close()
        if keep is not None:
            keep[1].close()

    fabric.run(body)
    full = E.gather_full_table(shards)
    tc = E.checkpoint_bytes(geom, full)
    w = dense_out["w"]
    return RunResult(losses, w, tc, tc + np.ascontiguousarray(w, np.float64).tobytes(),
                     num_iters * global_samples)


def batches_from_samples(spec: dict, samples: dict) -> list:
    """Rebuild iterations[i][r] (balancer.Batch) from the flat sample arrays
    the golden fixtures carry (oracle Reference.pipeline_samples)."""
    iters, world, batch = spec["iters"], spec["world"], spec["batch"]
    uih_len, n_cand = samples["uih_len"].astype(np.int64), samples["n_cand"].astype(np.int64)
    ids, cand_len, cand_ids = samples["ids"], samples["cand_len"].astype(np.int64), samples["cand_ids"]
    out, k, at, ca, cia = [], 0, 0, 0, 0
    for i in range(iters):
        row = []
        for r in range(world):
            ss = []
            for _ in range(batch):
                L = int(uih_len[k])
                cands = []
                for _c in range(int(n_cand[k])):
                    cl = int(cand_len[ca])
                    cands.append(cand_ids[cia:cia + cl].astype(np.uint64))
                    cia += cl
                    ca += 1
                ss.append(B.Sample(ids[at:at + L].astype(np.uint64), cands, float(samples["label"][k])))
                at += L
                k += 1
            row.append(B.Batch(ss, r))
        out.append(row)
    return out
