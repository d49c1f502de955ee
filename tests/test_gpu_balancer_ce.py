"""The balancer's collectives on the copy engines (CeComm: fsx_allgather_ce
direct and ring schedules, fsx_a2a_ce), ranks as threads on one GPU like the
reference's InProcessFabric (comm.cpp:136-154): the collectives against their
definition (comm.cpp:185-365; a17 all_gather / ring_all_gather, a16
all_to_all), then the whole three-stage balancer (balancer.cpp:99-252) over
them against the plan's expected batches."""
import numpy as np
import pytest

from balancer_cases import expected_batches, make_raw, sorted_round_robin

pytestmark = pytest.mark.gpu


def _with_ranks(world, body, ring):
    from paper_2604_24073_b200 import balancer as B
    from paper_2604_24073_b200 import embedding as E
    from paper_2604_24073_b200.comm import DeviceFabric
    fabric = DeviceFabric(world)
    out = [None] * world

    def rank_body(r):
        ctx = E.Context(fabric.device_of(r), r, world)
        shard = E.ShardView(E.TableGeometry(4 * world, 2, world), r, 0.1, 1, dtype="f32", ctx=ctx)
        eng = E.SynchronizedEmbedding(shard, fabric.communicator(r), max_occurrences=4096)
        try:
            out[r] = body(r, B.CeComm(eng, ring=ring))
        finally:
            eng.close()

    fabric.run(rank_body)
    return out


def _payload(r, k):
    n = (7 * r + 3 * k) % 11  # includes empty chunks
    return (np.arange(n, dtype=np.uint64) * np.uint64(1000003) + np.uint64(r * 97 + k)) ^ np.uint64(1 << 40)


@pytest.mark.parametrize("world", [2, 3, 4])
@pytest.mark.parametrize("ring", [False, True])
def test_all_gather_and_all_to_all(cuda, world, ring):
    def body(r, comm):
        res = []
        for k in range(3):  # repeated calls alternate the window parity
            res.append(comm.all_gather_u64(_payload(r, k)))
            res.append(comm.all_to_all_u64([_payload(r, k + 10 * d) for d in range(world)]))
        return res

    got = _with_ranks(world, body, ring)
    for r in range(world):
        for k in range(3):
            ag, a2a = got[r][2 * k], got[r][2 * k + 1]
            assert len(ag) == world and len(a2a) == world
            for d in range(world):
                assert np.array_equal(ag[d], _payload(d, k))
                assert np.array_equal(a2a[d], _payload(d, k + 10 * r))


@pytest.mark.parametrize("ring", [False, True])
def test_balancer_over_copy_engines(cuda, ring):
    from paper_2604_24073_b200 import balancer as B
    world, iters = 3, 3
    B.register_partitioner("sorted_rr", sorted_round_robin)

    def body(r, comm):
        bal = B.Balancer(comm, B.BalancerConfig(partition="custom:sorted_rr", lead=1),
                         lambda i: make_raw(i, r, world), iters)
        hooks = B.HookRegistry()
        bal.install_hooks(hooks)
        taken = []
        for i in range(iters):
            hooks.fire(B.HookPoint.DataLoad, i)
            taken.append(bal.take(i).samples)
            hooks.fire(B.HookPoint.PreForward, i)
            hooks.fire(B.HookPoint.PostForward, i)
            bal.report_compute_time(100.0 + r)
            hooks.fire(B.HookPoint.OptimizerStep, i)
        return taken

    got = _with_ranks(world, body, ring)
    exp = expected_batches(iters, world, "custom:sorted_rr")
    for r in range(world):
        for i in range(iters):
            assert got[r][i] == exp[i][r]
