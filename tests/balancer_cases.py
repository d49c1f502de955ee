"""Deterministic raw batches and a test partitioner for the balancer tests."""
import numpy as np

from paper_2604_24073_b200 import balancer as B
from paper_2604_24073_b200 import partition as P
from paper_2604_24073_b200 import workload


def make_raw(i: int, rank: int, world: int, per_rank: int = 6) -> B.Batch:
    """Rank `rank`'s raw batch of iteration i: UIH lengths from the power-law
    generator (clipped small), ids / candidates from splitmix streams."""
    seed = 1000 * i + rank
    lens = (workload.uih_lengths(seed, per_rank) % 23 + 1).astype(np.int64)
    ids = workload.splitmix_stream(seed ^ 0xABCD, int(lens.sum())) % np.uint64(1 << 20)
    ncand = (workload.splitmix_stream(seed ^ 0x77, per_rank) % np.uint64(4)).astype(np.int64)
    out, at, c = [], 0, 0
    for k in range(per_rank):
        cands = []
        for j in range(int(ncand[k])):
            L = 1 + (c * 7 + j) % 5
            cands.append(workload.splitmix_stream(seed ^ (0x1000 + c), L) % np.uint64(1 << 16))
            c += 1
        out.append(B.Sample(ids[at:at + lens[k]].copy(), cands, float(rank) + 0.5 * k))
        at += int(lens[k])
    return B.Batch(out, rank)


def sorted_round_robin(metas, n):
    """Custom partitioner: longest first, dealt round robin (ties by origin, local)."""
    order = sorted(range(len(metas)), key=lambda g: (-metas[g].uih_len, metas[g].origin_rank,
                                                    metas[g].local_index))
    a = np.zeros(len(metas), np.int32)
    ro = [[] for _ in range(n)]
    for k, g in enumerate(order):
        a[g] = k % n
        ro[k % n].append(g)
    return P.PartitionPlan(n, a, [np.asarray(o, np.uint64) for o in ro])


def expected_batches(iters, world, partition):
    """The reference's assemble semantics (balancer.cpp:224-252): rank r's
    balanced batch = the global samples in plan.receive_order[r]."""
    exp = []
    for i in range(iters):
        raws = [make_raw(i, r, world) for r in range(world)]
        metas = [P.GlobalSampleMeta(r, k, int(s.uih.size), len(s.candidates))
                 for r in range(world) for k, s in enumerate(raws[r].samples)]
        glob = [s for r in range(world) for s in raws[r].samples]
        plan = (P.identity_partition(metas, world) if partition == "none"
                else sorted_round_robin(metas, world))
        exp.append([[glob[int(g)] for g in plan.receive_order[r]] for r in range(world)])
    return exp
