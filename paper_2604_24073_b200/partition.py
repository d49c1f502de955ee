"""Python mirror of the reference partition API (proj/include/freescale/
partition.hpp) — the sequence load balancer's partition function. The sort,
the FBS snake deal and the VBS min-max DP run as libfsx kernels on the GPU,
bit-exact with the reference; plan bookkeeping (exchange lists, validation,
identity/custom plans) is host logic, as in the reference."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Callable, Sequence

import numpy as np

from . import _lib
from .errors import InvalidArgument, ProtocolError


@dataclass
class GlobalSampleMeta:
    """partition.hpp:14-20"""
    origin_rank: int = 0
    local_index: int = 0
    uih_len: int = 0
    num_candidates: int = 0
    candidate_lens: list = field(default_factory=list)


@dataclass
class PartitionPlan:
    """partition.hpp:25-38"""
    num_ranks: int = 0
    assignment: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    receive_order: list = field(default_factory=list)

    def exchange_lists(self, metas: Sequence[GlobalSampleMeta]):
        """partition.cpp:96-109: [src][dst] -> src-local indices in dst order."""
        lists = [[[] for _ in range(self.num_ranks)] for _ in range(self.num_ranks)]
        for dst in range(self.num_ranks):
            for g in self.receive_order[dst]:
                m = metas[int(g)]
                lists[m.origin_rank][dst].append(m.local_index)
        return lists

    def validate(self, num_samples: int, fixed_batch: bool) -> None:
        """partition.cpp:111-155 (same checks, same messages)."""
        if self.num_ranks < 1:
            raise InvalidArgument("partition plan: num_ranks < 1")
        if len(self.assignment) != num_samples:
            raise InvalidArgument(f"partition plan: assignment covers {len(self.assignment)} samples, "
                                  f"expected {num_samples} (samples lost or duplicated)")
        if len(self.receive_order) != self.num_ranks:
            raise InvalidArgument("partition plan: receive_order must have one list per rank")
        seen = np.zeros(num_samples, np.int64)
        for r in range(self.num_ranks):
            for g in self.receive_order[r]:
                g = int(g)
                if g >= num_samples:
                    raise InvalidArgument(f"partition plan: sample index {g} out of range")
                if self.assignment[g] != r:
                    raise InvalidArgument(f"partition plan: sample {g} listed under rank {r} but assigned "
                                          f"to rank {int(self.assignment[g])}")
                seen[g] += 1
                if seen[g] > 1:
                    raise InvalidArgument(f"partition plan: sample {g} assigned more than once")
        missing = np.nonzero(seen == 0)[0]
        if missing.size:
            raise InvalidArgument(f"partition plan: sample {int(missing[0])} not assigned to any rank")
        if fixed_batch and num_samples % self.num_ranks == 0:
            per = num_samples // self.num_ranks
            for r in range(self.num_ranks):
                if len(self.receive_order[r]) != per:
                    raise InvalidArgument(f"partition plan: rank {r} receives {len(self.receive_order[r])} "
                                          f"samples, expected {per}")


@dataclass
class AutoTuneState:
    """partition.hpp:40-48"""
    local_batch_size: list = field(default_factory=list)
    ema_local: list = field(default_factory=list)
    ema_global: float = 0.0
    step: int = 1
    delta: float = 0.05
    decay: float = 0.9
    initialized: bool = False


def _arrays(metas):
    lens = np.ascontiguousarray([m.uih_len for m in metas], np.uint64)
    origin = np.ascontiguousarray([m.origin_rank for m in metas], np.int32)
    local = np.ascontiguousarray([m.local_index for m in metas], np.int32)
    return lens, origin, local


def _ctx(ctx):
    if ctx is not None:
        return ctx
    from .embedding import default_context
    return default_context()


def _split(order: np.ndarray, sizes) -> list:
    out, at = [], 0
    for s in sizes:
        out.append(order[at:at + int(s)].copy())
        at += int(s)
    return out


def fbs_partition(metas: Sequence[GlobalSampleMeta], num_ranks: int, ctx=None) -> PartitionPlan:
    """partition.cpp:157-176: sort by (uih_len desc, origin, local), snake."""
    return fbs_partition_arrays(*_arrays(metas), num_ranks, ctx=ctx)


def fbs_partition_arrays(lens, origin, local, num_ranks: int, ctx=None) -> PartitionPlan:
    """fbs_partition over the metas' columns (uih_len u64, origin_rank i32,
    local_index i32): the C ABI's own argument form, no per-sample objects."""
    if num_ranks < 1:
        raise InvalidArgument("fbs: num_ranks must be >= 1")
    lens = np.ascontiguousarray(lens, np.uint64)
    origin = np.ascontiguousarray(origin, np.int32)
    local = np.ascontiguousarray(local, np.int32)
    m = lens.size
    if m % num_ranks:
        raise InvalidArgument(f"fbs: {m} samples not divisible by {num_ranks} ranks")
    a = np.zeros(max(m, 1), np.int32)
    o = np.zeros(max(m, 1), np.uint64)
    if m:
        _lib.call("fsx_fbs_partition", _ctx(ctx).h, lens.ctypes.data, origin.ctypes.data, local.ctypes.data,
                  m, num_ranks, a.ctypes.data, o.ctypes.data, None)
    per = m // num_ranks
    return PartitionPlan(num_ranks, a[:m], _split(o[:m], [per] * num_ranks))


def vbs_partition(metas: Sequence[GlobalSampleMeta], num_ranks: int, alpha: float,
                  tune: AutoTuneState | None = None, ctx=None) -> PartitionPlan:
    """partition.cpp:178-209: min-max contiguous cut of the sorted weights
    uih_len^alpha (exact DP on the GPU), or the tuned sizes of an
    initialized autotune state."""
    return vbs_partition_arrays(*_arrays(metas), num_ranks, alpha, tune=tune, ctx=ctx)


def vbs_partition_arrays(lens, origin, local, num_ranks: int, alpha: float,
                         tune: AutoTuneState | None = None, ctx=None) -> PartitionPlan:
    """vbs_partition over the metas' columns (see fbs_partition_arrays)."""
    lens = np.ascontiguousarray(lens, np.uint64)
    origin = np.ascontiguousarray(origin, np.int32)
    local = np.ascontiguousarray(local, np.int32)
    m = lens.size
    a = np.zeros(max(m, 1), np.int32)
    o = np.zeros(max(m, 1), np.uint64)
    sizes = np.zeros(max(num_ranks, 1), np.int32)
    tuned = None
    if tune is not None and tune.initialized and len(tune.local_batch_size) == num_ranks and \
            sum(tune.local_batch_size) == m:
        tuned = np.ascontiguousarray(tune.local_batch_size, np.int32)
    _lib.call("fsx_vbs_partition", _ctx(ctx).h, lens.ctypes.data if m else None,
              origin.ctypes.data if m else None, local.ctypes.data if m else None, m, num_ranks,
              float(alpha), tuned.ctypes.data if tuned is not None else None, sizes.ctypes.data,
              a.ctypes.data, o.ctypes.data, None)
    if tune is not None and tuned is None:
        tune.local_batch_size = [int(x) for x in sizes[:num_ranks]]
        tune.ema_local = [0.0] * num_ranks
        tune.ema_global = 0.0
        tune.initialized = True
    return PartitionPlan(num_ranks, a[:m], _split(o[:m], sizes[:num_ranks]))


def autotune_update(tune: AutoTuneState, local_times) -> None:
    """partition.cpp:211-269 (host f64 via the C ABI)."""
    if not tune.initialized:
        raise ProtocolError("autotune: state not initialized")
    n = len(tune.local_batch_size)
    t = np.ascontiguousarray(local_times, np.float64)
    if t.size != n:
        raise InvalidArgument(f"autotune: expected {n} times, got {t.size}")
    sizes = np.ascontiguousarray(tune.local_batch_size, np.int32)
    ema = np.ascontiguousarray(tune.ema_local, np.float64)
    eg = C.c_double(tune.ema_global)
    _lib.call("fsx_autotune_update", n, sizes.ctypes.data, ema.ctypes.data, C.byref(eg), tune.step,
              tune.delta, tune.decay, t.ctypes.data)
    tune.local_batch_size = [int(x) for x in sizes]
    tune.ema_local = [float(x) for x in ema]
    tune.ema_global = eg.value


def identity_partition(metas: Sequence[GlobalSampleMeta], num_ranks: int) -> PartitionPlan:
    """partition.cpp:271-283"""
    order = [[] for _ in range(num_ranks)]
    for g, m in enumerate(metas):
        order[m.origin_rank].append(g)
    for o in order:
        o.sort(key=lambda g: metas[g].local_index)
    a = np.full(len(metas), -1, np.int32)
    for r, o in enumerate(order):
        a[o] = r
    return PartitionPlan(num_ranks, a, [np.asarray(o, np.uint64) for o in order])


def custom_partition(fn: Callable, metas: Sequence[GlobalSampleMeta], num_ranks: int) -> PartitionPlan:
    """partition.cpp:285-290"""
    plan = fn(metas, num_ranks)
    plan.validate(len(metas), False)
    return plan


def plan_max_weight(plan: PartitionPlan, metas, alpha: float) -> float:
    """partition.cpp:321-330"""
    return max((sum(float(metas[int(g)].uih_len) ** alpha for g in o) for o in plan.receive_order), default=0.0)


def metas_from_lengths(lengths, num_ranks: int) -> list:
    """test_partition.cpp:13-24 helper: rank-major origin / local indices."""
    per = (len(lengths) + num_ranks - 1) // num_ranks if num_ranks > 0 else 1
    return [GlobalSampleMeta(i // per, i % per, int(l)) for i, l in enumerate(lengths)]
