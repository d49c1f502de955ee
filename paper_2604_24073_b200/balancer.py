"""Sequence load balancer, three-stage protocol (proj/include/freescale/
balancer.hpp:12-78, src/balancer.cpp:26-277), over torch.distributed (one
process per GPU; gloo works for CPU-only tests).

  stage 1  all-gather of every rank's UIH lengths, candidate counts and last
           compute time -> global sample metas (rank-major);
  stage 2  all-gather of candidate lengths, then the partition function
           (fbs / vbs + autotune / none / custom:<name>) computed redundantly
           and identically on every rank — fbs and vbs are the libfsx GPU
           kernels, bit-exact with the reference — and validated;
  stage 3  the sample all-to-all. B200 design: instead of the reference's
           per-sample byte records (workload.cpp:391-418) each destination gets
           ONE jagged message of u64 words (per-sample lengths, flat UIH ids,
           candidate counts / lengths / ids, labels as f64 bits), the
           SURVEY §8(f-1) replacement of record serialization;
  take(i)  assembles the balanced batch in the plan's receive order with
           per-source cursors (balancer.cpp:224-252).

Stages must fire in order per batch; violations raise the reference's
ProtocolError messages. Hooks: `install_hooks` wires the stages to a
HookRegistry exactly like balancer.cpp:73-97 (lead batches ahead)."""
from __future__ import annotations

import threading
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

from . import _lib

from . import partition as P
from .errors import ConfigError, ProtocolError


# ---- workload types (workload.hpp:17-35) --------------------------------------------
@dataclass
class Sample:
    uih: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint64))
    candidates: list = field(default_factory=list)  # list of u64 arrays
    label: float = 0.0

    def __eq__(self, o):
        return (isinstance(o, Sample) and np.array_equal(self.uih, o.uih) and self.label == o.label
                and len(self.candidates) == len(o.candidates)
                and all(np.array_equal(a, b) for a, b in zip(self.candidates, o.candidates)))


@dataclass
class Batch:
    samples: list = field(default_factory=list)
    rank: int = 0

    def total_uih_tokens(self) -> int:
        return int(sum(s.uih.size for s in self.samples))

    def uih_ids(self) -> tuple:
        """Batch-major id tensor: (flat ids, per-sample lengths)."""
        if not self.samples:
            return np.zeros(0, np.uint64), np.zeros(0, np.uint64)
        return (np.concatenate([np.asarray(s.uih, np.uint64) for s in self.samples]),
                np.asarray([s.uih.size for s in self.samples], np.uint64))


# ---- hooks (pipeline.hpp:39-59) ----------------------------------------------------------
class HookPoint:
    DataLoad, PreForward, PostForward, OptimizerStep = range(4)


class HookRegistry:
    def __init__(self):
        self._hooks = {}

    def add(self, point: int, fn: Callable) -> None:
        self._hooks.setdefault(point, []).append(fn)

    def fire(self, point: int, iteration: int) -> None:
        for fn in self._hooks.get(point, []):
            fn(iteration)


# ---- custom partitioner registry (pipeline.cpp:16-33) ------------------------------------
_partitioners: dict = {}
_reg_lock = threading.Lock()


def register_partitioner(name: str, fn: Callable) -> None:
    with _reg_lock:
        _partitioners[name] = fn


def find_partitioner(name: str) -> Optional[Callable]:
    with _reg_lock:
        return _partitioners.get(name)


# ---- communicator over torch.distributed ---------------------------------------------
class TorchComm:
    """all_gather / all_to_all of variable-length u64 arrays over a
    torch.distributed group (sizes first, then one padded all_gather or one
    all_to_all_single). `device` = "cpu" for gloo, a cuda device for nccl."""

    def __init__(self, group=None, device="cpu"):
        import torch
        import torch.distributed as dist
        self.torch, self.dist, self.group, self.device = torch, dist, group, torch.device(device)

    def rank(self) -> int:
        return self.dist.get_rank(self.group)

    def world_size(self) -> int:
        return self.dist.get_world_size(self.group)

    def _t(self, a):
        return self.torch.from_numpy(np.ascontiguousarray(a, np.uint64).view(np.int64)).to(self.device)

    def all_gather_u64(self, a: np.ndarray) -> list:
        torch, dist = self.torch, self.dist
        w = self.world_size()
        n = torch.tensor([a.size], dtype=torch.int64, device=self.device)
        ns = [torch.zeros_like(n) for _ in range(w)]
        dist.all_gather(ns, n, group=self.group)
        sizes = [int(x.item()) for x in ns]
        m = max(sizes + [1])
        buf = torch.zeros(m, dtype=torch.int64, device=self.device)
        buf[:a.size] = self._t(a)
        outs = [torch.empty_like(buf) for _ in range(w)]
        dist.all_gather(outs, buf, group=self.group)
        return [o[:s].cpu().numpy().view(np.uint64).copy() for o, s in zip(outs, sizes)]

    def all_to_all_u64(self, parts: list) -> list:
        torch, dist = self.torch, self.dist
        w = self.world_size()
        send_sizes = torch.tensor([p.size for p in parts], dtype=torch.int64, device=self.device)
        recv_sizes = torch.empty_like(send_sizes)
        dist.all_to_all_single(recv_sizes, send_sizes, group=self.group)
        ss, rs = send_sizes.tolist(), recv_sizes.tolist()
        flat = np.concatenate([np.asarray(p, np.uint64) for p in parts]) if parts else np.zeros(0, np.uint64)
        out = torch.empty(sum(rs), dtype=torch.int64, device=self.device)
        dist.all_to_all_single(out, self._t(flat), rs, ss, group=self.group)
        host = out.cpu().numpy().view(np.uint64)
        res, at = [], 0
        for r in range(w):
            res.append(host[at:at + rs[r]].copy())
            at += rs[r]
        return res


def _ce_all_to_all_jagged(comm, parts: list) -> list:
    """Jagged all-to-all on the copy engines: every part's lengths (host, a
    small size round) and its 8-byte values device to device (fsx_a2a_ce)."""
    import ctypes as C
    import torch
    from . import jagged as J
    w, dev = comm.world_size(), comm.dev
    lens = comm.all_to_all_u64([p.lengths() for p in parts])
    nbytes = [8 * p.total_values() for p in parts]
    mat = comm.all_gather_u64(np.asarray(nbytes, np.uint64))
    slot = max([int(x) for row in mat for x in row] + [8])
    vals = [p.values().view(torch.int64) for p in parts]
    send = torch.cat(vals) if any(v.numel() for v in vals) else torch.zeros(1, dtype=torch.int64, device=dev)
    offs = (C.c_uint64 * w)(*np.concatenate([[0], np.cumsum(nbytes)[:-1]]).astype(int))
    recv = torch.empty(w * slot // 8, dtype=torch.int64, device=dev)
    got = (C.c_uint64 * w)()
    _lib.call("fsx_a2a_ce", comm.e.h, C.c_void_p(send.data_ptr()), offs, (C.c_uint64 * w)(*nbytes),
              C.c_void_p(recv.data_ptr()), slot, got, C.c_void_p(comm._stream()))
    return [J.JaggedTensor(recv[d * slot // 8: d * slot // 8 + got[d] // 8].clone(), lens[d], device=dev)
            for d in range(w)]


class LocalComm:
    """world of one (comm.cpp:194-198: every exchange is a local hand-off)."""

    def rank(self) -> int:
        return 0

    def world_size(self) -> int:
        return 1

    def all_gather_u64(self, a):
        return [np.asarray(a, np.uint64).copy()]

    def all_to_all_u64(self, parts):
        return [np.asarray(parts[0], np.uint64).copy()]


class CeComm:
    """The balancer's collectives on the copy engines (0 SMs), over an
    embedding engine's receive windows: all_gather (comm.cpp:185-306; the
    direct schedule, or ring=True for the reference's SmFree ring
    comm.cpp:214-236) through fsx_allgather_ce, all_to_all (comm.cpp:308-365)
    through fsx_a2a_ce. Variable sizes go in a first round (like
    TorchComm); every call synchronizes the engine's device."""

    def __init__(self, engine, ring: bool = False):
        import torch
        self.torch, self.e, self.ring = torch, engine, bool(ring)
        self.dev = engine.shard.ctx.torch_device

    def rank(self) -> int:
        return self.e.comm.rank()

    def world_size(self) -> int:
        return self.e.comm.world_size()

    def _stream(self):
        return self.torch.cuda.current_stream(self.dev).cuda_stream

    def _gather(self, a: np.ndarray, bound: int) -> list:
        import ctypes as C
        torch, w = self.torch, self.world_size()
        a = np.ascontiguousarray(a, np.uint64)
        slot = max(int(bound), 8)
        send = torch.from_numpy(a.view(np.int64).copy()).to(self.dev) if a.size else \
            torch.zeros(1, dtype=torch.int64, device=self.dev)
        recv = torch.zeros(w * slot // 8, dtype=torch.int64, device=self.dev)
        got = (C.c_uint64 * w)()
        _lib.call("fsx_allgather_ce", self.e.h, C.c_void_p(send.data_ptr()), a.nbytes, slot,
                  C.c_void_p(recv.data_ptr()), slot, got, int(self.ring), C.c_void_p(self._stream()))
        host = recv.cpu().numpy().view(np.uint64)
        return [host[d * slot // 8: d * slot // 8 + got[d] // 8].copy() for d in range(w)]

    def all_gather_u64(self, a: np.ndarray) -> list:
        sizes = [int(x[0]) for x in self._gather(np.array([np.asarray(a).size], np.uint64), 8)]
        return self._gather(a, 8 * max(sizes + [1]))

    def all_to_all_u64(self, parts: list) -> list:
        import ctypes as C
        torch, w = self.torch, self.world_size()
        parts = [np.ascontiguousarray(p, np.uint64) for p in parts]
        # size round: every rank's row of the send matrix
        mat = self.all_gather_u64(np.array([p.size for p in parts], np.uint64))
        # one slot size on every rank (the sender checks its payloads against it)
        slot = 8 * max([int(x) for row in mat for x in row] + [1])
        flat = np.concatenate(parts) if parts else np.zeros(0, np.uint64)
        send = torch.from_numpy(flat.view(np.int64).copy()).to(self.dev) if flat.size else \
            torch.zeros(1, dtype=torch.int64, device=self.dev)
        offs = (C.c_uint64 * w)(*np.concatenate([[0], np.cumsum([8 * p.size for p in parts])[:-1]]).astype(int))
        nbytes = (C.c_uint64 * w)(*[8 * p.size for p in parts])
        recv = torch.zeros(w * slot // 8, dtype=torch.int64, device=self.dev)
        got = (C.c_uint64 * w)()
        _lib.call("fsx_a2a_ce", self.e.h, C.c_void_p(send.data_ptr()), offs, nbytes, C.c_void_p(recv.data_ptr()),
                  slot, got, C.c_void_p(self._stream()))
        host = recv.cpu().numpy().view(np.uint64)
        return [host[d * slot // 8: d * slot // 8 + got[d] // 8].copy() for d in range(w)]


CeComm.all_to_all_jagged = _ce_all_to_all_jagged


# ---- balancer ---------------------------------------------------------------------------
@dataclass
class BalancerConfig:
    """balancer.hpp:14-23"""
    partition: str = "fbs"  # fbs | vbs | none | custom:<name>
    alpha: float = 1.0
    autotune_step: int = 1
    autotune_delta: float = 0.05
    autotune_decay: float = 0.9
    lead: int = 1


class Stage:
    Idle, LengthsGathered, CandidatesGathered, Shuffled = range(4)


@dataclass
class _Pending:
    index: int
    raw: Batch
    stage: int = Stage.Idle
    metas: list = field(default_factory=list)
    world_times: list = field(default_factory=list)
    plan: Optional[P.PartitionPlan] = None
    shuffled: Optional[list] = None
    balanced: Optional[Batch] = None


def _f64_bits(x: float) -> int:
    return int(np.array([x], np.float64).view(np.uint64)[0])


def _bits_f64(u) -> float:
    return float(np.array([u], np.uint64).view(np.float64)[0])


def encode_jagged(samples: list) -> np.ndarray:
    """One destination's stage-3 message: [n][len_0..n-1][uih ids][ncand_0..][cand lens][cand ids][labels]."""
    n = len(samples)
    lens = np.asarray([s.uih.size for s in samples], np.uint64)
    nc = np.asarray([len(s.candidates) for s in samples], np.uint64)
    clens = np.asarray([c.size for s in samples for c in s.candidates], np.uint64)
    parts = [np.asarray([n], np.uint64), lens]
    parts += [np.asarray(s.uih, np.uint64) for s in samples]
    parts += [nc, clens]
    parts += [np.asarray(c, np.uint64) for s in samples for c in s.candidates]
    parts.append(np.asarray([_f64_bits(s.label) for s in samples], np.uint64))
    return np.concatenate(parts) if parts else np.zeros(0, np.uint64)


def decode_jagged(msg: np.ndarray) -> list:
    if msg.size == 0:
        raise ProtocolError("balancer: stage-3 payload shorter than the plan")
    n = int(msg[0])
    at = 1
    lens = msg[at:at + n].astype(np.int64)
    at += n
    uih = []
    for L in lens:
        uih.append(msg[at:at + L].copy())
        at += int(L)
    nc = msg[at:at + n].astype(np.int64)
    at += n
    tot_c = int(nc.sum())
    clens = msg[at:at + tot_c].astype(np.int64)
    at += tot_c
    cands, ci = [], 0
    for k in range(n):
        cs = []
        for _ in range(int(nc[k])):
            L = int(clens[ci])
            cs.append(msg[at:at + L].copy())
            at += L
            ci += 1
        cands.append(cs)
    labels = msg[at:at + n]
    at += n
    if at != msg.size:
        raise ProtocolError("balancer: stage-3 record has trailing bytes")
    return [Sample(uih[k], cands[k], _bits_f64(labels[k])) for k in range(n)]


class Balancer:
    """balancer.hpp:32-78"""

    def __init__(self, comm, config: BalancerConfig, raw_batches: Callable[[int], Optional[Batch]],
                 num_iterations: int, ctx=None):
        if config.lead < 1:
            raise ConfigError("balancer: lead must be >= 1")
        self.comm, self.config, self.raw_batches = comm, config, raw_batches
        self.num_iterations = num_iterations
        self.ctx = ctx
        self.pending: list = []
        self.tune = P.AutoTuneState(step=config.autotune_step, delta=config.autotune_delta,
                                    decay=config.autotune_decay)
        self.last_compute_us = 0.0
        self._fires = [0, 0, 0]

    # -- plumbing (balancer.cpp:39-71)
    def _pending_for(self, index: int, create: bool) -> Optional[_Pending]:
        for p in self.pending:
            if p.index == index:
                return p
        if not create or index >= self.num_iterations:
            return None
        raw = self.raw_batches(index)
        if raw is None:
            raise ProtocolError(f"balancer: no raw batch for iteration {index}")
        p = _Pending(index, raw)
        self.pending.append(p)
        return p

    def run_stage_for(self, index: int, stage: int) -> None:
        if index < 0 or index >= self.num_iterations:
            return
        p = self._pending_for(index, stage == 0)
        if p is None:
            return
        self._fires[stage] += 1
        (self._stage1, self._stage2, self._stage3)[stage](p)

    def stage_fires(self, stage: int) -> int:
        return self._fires[stage]

    def report_compute_time(self, us: float) -> None:
        self.last_compute_us = float(us)

    def install_hooks(self, hooks: HookRegistry) -> None:
        """balancer.cpp:73-97"""
        lead = self.config.lead

        def on_load(it):
            if it == 0:
                for j in range(min(lead, self.num_iterations)):
                    for s in range(3):
                        self.run_stage_for(j, s)
                self.run_stage_for(lead, 0)

        hooks.add(HookPoint.DataLoad, on_load)
        hooks.add(HookPoint.PreForward, lambda it: self.run_stage_for(it + lead, 1))
        hooks.add(HookPoint.PostForward, lambda it: self.run_stage_for(it + lead, 2))
        hooks.add(HookPoint.OptimizerStep, lambda it: self.run_stage_for(it + lead + 1, 0))

    # -- stage 1 (balancer.cpp:99-128)
    def _stage1(self, p: _Pending) -> None:
        if p.stage != Stage.Idle:
            raise ProtocolError("balancer: stage 1 fired out of order")
        b = p.raw.samples
        payload = np.concatenate([
            np.asarray([len(b)], np.uint64),
            np.asarray([s.uih.size for s in b], np.uint64),
            np.asarray([len(s.candidates) for s in b], np.uint64),
            np.asarray([_f64_bits(self.last_compute_us)], np.uint64)])
        gathered = self.comm.all_gather_u64(payload)
        p.metas, p.world_times = [], []
        for r, v in enumerate(gathered):
            if v.size < 2:
                raise ProtocolError("balancer: short stage-1 payload")
            B = int(v[0])
            if v.size != 2 + 2 * B:
                raise ProtocolError("balancer: stage-1 payload shape mismatch")
            p.world_times.append(_bits_f64(v[-1]))
            for i in range(B):
                p.metas.append(P.GlobalSampleMeta(r, i, int(v[1 + i]), int(v[1 + B + i])))
        p.stage = Stage.LengthsGathered

    # -- stage 2 (balancer.cpp:130-194)
    def _stage2(self, p: _Pending) -> None:
        if p.stage != Stage.LengthsGathered:
            raise ProtocolError("balancer: stage 2 before stage 1")
        mine = np.asarray([c.size for s in p.raw.samples for c in s.candidates], np.uint64)
        gathered = self.comm.all_gather_u64(mine)
        at_meta = 0
        for r, lens in enumerate(gathered):
            begin = at_meta
            expected = 0
            while at_meta < len(p.metas) and p.metas[at_meta].origin_rank == r:
                expected += p.metas[at_meta].num_candidates
                at_meta += 1
            if lens.size != expected:
                raise ProtocolError(f"balancer: rank {r} sent {lens.size} candidate lengths, "
                                    f"stage 1 announced {expected}")
            off = 0
            for m in range(begin, at_meta):
                k = p.metas[m].num_candidates
                p.metas[m].candidate_lens = [int(x) for x in lens[off:off + k]]
                off += k
        world = self.comm.world_size()
        part = self.config.partition
        if part == "fbs":
            p.plan = P.fbs_partition(p.metas, world, ctx=self.ctx)
        elif part == "vbs":
            if self.tune.initialized and any(t > 0 for t in p.world_times):
                P.autotune_update(self.tune, [max(t, 1e-9) for t in p.world_times])
            p.plan = P.vbs_partition(p.metas, world, self.config.alpha, self.tune, ctx=self.ctx)
        elif part == "none":
            p.plan = P.identity_partition(p.metas, world)
        elif part.startswith("custom:"):
            fn = find_partitioner(part[7:])
            if fn is None:
                raise ConfigError(f"balancer: unknown custom partitioner '{part[7:]}'")
            p.plan = P.custom_partition(fn, p.metas, world)
        else:
            raise ConfigError(f"balancer: unknown partition '{part}'")
        p.plan.validate(len(p.metas), part == "fbs")
        p.stage = Stage.CandidatesGathered

    # -- stage 3 (balancer.cpp:196-222), jagged messages
    def _stage3(self, p: _Pending) -> None:
        if p.stage != Stage.CandidatesGathered:
            raise ProtocolError("balancer: stage 3 before stage 2")
        lists = p.plan.exchange_lists(p.metas)
        mine = lists[self.comm.rank()]
        if hasattr(self.comm, "all_to_all_jagged"):
            p.shuffled = self._stage3_jagged(p, mine)
        else:
            msgs = [encode_jagged([p.raw.samples[int(l)] for l in mine[dst]])
                    for dst in range(self.comm.world_size())]
            p.shuffled = self.comm.all_to_all_u64(msgs)
        p.stage = Stage.Shuffled

    def _stage3_jagged(self, p: _Pending, mine: list) -> list:
        """Stage 3 as jagged device ops instead of per-sample
        record serialization: the UIH and candidate segments go to the device
        once, indexed_permute groups them by destination in exchange order,
        ranged_dispatch cuts one part per destination, and the parts travel by
        copy-engine all-to-all; candidate counts and labels ride a small u64
        message."""
        from . import jagged as J
        dev = self.comm.dev
        samples = p.raw.samples
        w = self.comm.world_size()
        uih = J.IdJagged.from_segments([s.uih for s in samples], device=dev)
        nc = np.asarray([len(s.candidates) for s in samples], np.int64)
        cstart = np.concatenate([[0], np.cumsum(nc)]).astype(np.int64)
        cand = J.IdJagged.from_segments([c for s in samples for c in s.candidates], device=dev)
        order = [int(k) for dst in range(w) for k in mine[dst]]
        counts = [len(mine[dst]) for dst in range(w)]
        ccounts = [int(sum(nc[int(k)] for k in mine[dst])) for dst in range(w)]
        cperm = [int(cstart[k]) + j for k in order for j in range(int(nc[k]))]
        starts = np.concatenate([[0], np.cumsum(counts)]).astype(int)
        cstarts = np.concatenate([[0], np.cumsum(ccounts)]).astype(int)
        uih_parts = J.ranged_dispatch(J.indexed_permute(uih, order), [(starts[d], counts[d]) for d in range(w)])
        cand_parts = J.ranged_dispatch(J.indexed_permute(cand, cperm), [(cstarts[d], ccounts[d]) for d in range(w)])
        meta = [np.concatenate([nc[[int(k) for k in mine[dst]]].astype(np.uint64),
                                np.asarray([_f64_bits(samples[int(k)].label) for k in mine[dst]], np.uint64)])
                for dst in range(w)]
        r_uih = self.comm.all_to_all_jagged(uih_parts)
        r_cand = self.comm.all_to_all_jagged(cand_parts)
        r_meta = self.comm.all_to_all_u64(meta)
        out = []
        for src in range(w):
            segs = r_uih[src].to_segments()
            n = len(segs)
            if r_meta[src].size != 2 * n:
                raise ProtocolError("balancer: stage-3 payload shorter than the plan")
            ncs = r_meta[src][:n].astype(np.int64)
            csegs = r_cand[src].to_segments()
            at, samp = 0, []
            for k in range(n):
                cs = [np.asarray(c, np.uint64) for c in csegs[at:at + int(ncs[k])]]
                at += int(ncs[k])
                samp.append(Sample(np.asarray(segs[k], np.uint64), cs, _bits_f64(r_meta[src][n + k])))
            out.append(samp)
        return out

    # -- consumption (balancer.cpp:224-277)
    def _assemble(self, p: _Pending) -> Batch:
        me = self.comm.rank()
        per_src = ([decode_jagged(m) for m in p.shuffled] if p.shuffled and isinstance(p.shuffled[0], np.ndarray)
                   else p.shuffled)
        cursor = [0] * len(per_src)
        out = Batch(rank=me)
        for g in p.plan.receive_order[me]:
            src = p.metas[int(g)].origin_rank
            if cursor[src] >= len(per_src[src]):
                raise ProtocolError("balancer: stage-3 payload shorter than the plan")
            out.samples.append(per_src[src][cursor[src]])
            cursor[src] += 1
        for src, c in enumerate(cursor):
            if c != len(per_src[src]):
                raise ProtocolError(f"balancer: stage-3 payload from rank {src} longer than the plan")
        return out

    def take(self, iteration: int) -> Batch:
        p = self._pending_for(iteration, False)
        if p is None or p.stage != Stage.Shuffled:
            raise ProtocolError(f"balancer: batch {iteration} consumed before stage 3 completed")
        out = p.balanced if p.balanced is not None else self._assemble(p)
        self.pending = [q for q in self.pending if q.index > iteration]
        return out

    def peek(self, iteration: int) -> Optional[Batch]:
        p = self._pending_for(iteration, False)
        if p is None:
            return None
        if p.stage != Stage.Shuffled:
            raise ProtocolError(f"balancer: peek at batch {iteration} before stage 3 completed")
        if p.balanced is None:
            p.balanced = self._assemble(p)
        return p.balanced
