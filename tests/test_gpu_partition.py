"""GPU parity of the load-balancer kernels (K12-K14) against the reference's
known answers, the golden plans it produced (tests/golden/partition_cases.npz,
cfg2_partition.npz) and the C oracle: assignments, receive orders and segment
sizes bit-exact, cost-model values bit-exact in f64."""
import os

import numpy as np
import pytest

from golden_io import HERE, partition_cases

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P(cuda):
    from paper_2604_24073_b200 import partition
    return partition


def _metas(P, lens, origin, local):
    return [P.GlobalSampleMeta(int(o), int(l), int(x)) for x, o, l in zip(lens, origin, local)]


def test_fbs_kats(P):
    # test_partition.cpp:38-64
    metas = P.metas_from_lengths([9, 7, 5, 3], 2)
    plan = P.fbs_partition(metas, 2)
    plan.validate(4, True)
    assert [sum(metas[int(g)].uih_len for g in o) for o in plan.receive_order] == [12, 12]
    plan = P.fbs_partition(P.metas_from_lengths([3, 9, 1], 1), 1)
    assert plan.receive_order[0].tolist() == [1, 0, 2]
    metas = P.metas_from_lengths([7] * 12, 3)
    plan = P.fbs_partition(metas, 3)
    assert [sum(metas[int(g)].uih_len for g in o) for o in plan.receive_order] == [28, 28, 28]
    from paper_2604_24073_b200.errors import InvalidArgument
    with pytest.raises(InvalidArgument):
        P.fbs_partition(P.metas_from_lengths([1, 2, 3], 2), 2)


def test_vbs_kats(P):
    # test_partition.cpp:66-95 + derived tie-break KATs
    m = P.metas_from_lengths([4, 3, 2, 1], 2)
    plan = P.vbs_partition(m, 2, 1.0)
    plan.validate(4, False)
    assert P.plan_max_weight(plan, m, 1.0) == pytest.approx(6.0)
    assert [len(o) for o in plan.receive_order] == [1, 3]
    plan = P.vbs_partition(P.metas_from_lengths([3, 3, 3, 3], 2), 2, 2.0)
    assert [len(o) for o in plan.receive_order] == [2, 2]
    assert all(len(o) == 1 for o in P.vbs_partition(P.metas_from_lengths([5, 4, 3], 3), 3, 1.0).receive_order)
    for lens, n, sizes in (([1, 1, 1], 2, [2, 1]), ([2] * 5, 2, [3, 2]), ([2] * 5, 3, [2, 2, 1]),
                           ([4, 2, 2, 2, 2], 2, [2, 3]), ([4, 2, 2, 2, 2], 3, [1, 2, 2])):
        got = P.vbs_partition(P.metas_from_lengths(lens, 1), n, 1.0)
        assert [len(o) for o in got.receive_order] == sizes, (lens, n)
    from paper_2604_24073_b200.errors import InvalidArgument
    with pytest.raises(InvalidArgument):
        P.vbs_partition(P.metas_from_lengths([5, 4], 2), 3, 1.0)
    with pytest.raises(InvalidArgument):
        P.vbs_partition(P.metas_from_lengths([5, 4], 2), 2, 0.0)


def test_golden_cases(P):
    for name, c in partition_cases().items():
        metas = _metas(P, c["lens"], c["origin"], c["local"])
        n = c["n"]
        if c["fbs_assign"].size:
            plan = P.fbs_partition(metas, n)
            assert np.array_equal(plan.assignment, c["fbs_assign"]), name
            assert np.array_equal(np.concatenate(plan.receive_order), c["fbs_order"]), name
        for alpha, (a_ref, o_ref, s_ref) in ((1.0, c["vbs1"]), (2.0, c["vbs2"])):
            if a_ref.size == 0:
                continue
            plan = P.vbs_partition(metas, n, alpha)
            assert np.array_equal(plan.assignment, a_ref), (name, alpha)
            assert np.array_equal(np.concatenate(plan.receive_order), o_ref), (name, alpha)
            assert [len(o) for o in plan.receive_order] == s_ref.tolist(), (name, alpha)


def test_vbs_random_vs_oracle_and_bruteforce(P, oracle):
    from paper_2604_24073_b200.workload import splitmix_stream
    st = splitmix_stream(31337, 300 * 20)
    at = 0
    for _ in range(150):
        m = 2 + int(st[at] % 11)
        n = 1 + int(st[at + 1] % m)
        alpha = [1.0, 2.0, 1.5][int(st[at + 2] % 3)]
        at += 3
        lens = (st[at:at + m] % np.uint64(100)).astype(np.uint64)
        at += m
        metas = P.metas_from_lengths(lens, 1)
        plan = P.vbs_partition(metas, n, alpha)
        a, order, sizes = oracle.vbs(lens, [0] * m, list(range(m)), n, alpha)
        assert np.array_equal(plan.assignment, a)
        w = np.concatenate([lens[o].astype(np.float64) ** alpha for o in order])
        assert P.plan_max_weight(plan, metas, alpha) == pytest.approx(oracle.bruteforce(w, n), rel=1e-12)


def test_vbs_tuned_sizes(P):
    # test_partition.cpp:156-165: an initialized state's sizes are honoured
    metas = P.metas_from_lengths(list(range(1, 17)), 2)
    tune = P.AutoTuneState(local_batch_size=[5, 11], ema_local=[0, 0], initialized=True)
    plan = P.vbs_partition(metas, 2, 1.0, tune)
    assert [len(o) for o in plan.receive_order] == [5, 11]
    fresh = P.AutoTuneState()
    plan = P.vbs_partition(metas, 2, 1.0, fresh)
    assert fresh.initialized and sum(fresh.local_batch_size) == 16


def test_cost_model(cuda, oracle):
    from paper_2604_24073_b200.sim import CostModel
    cm = CostModel(50, 0.01, 0)
    assert cm.compute_time_for_lengths([100, 300]) == pytest.approx(54.0)
    cm = CostModel(50, 0.01, 1e-6)
    assert cm.compute_time_for_lengths([16, 8192, 97, 1000]) == float.fromhex("0x1.a656496ededafp+7")
    rng = np.random.default_rng(1)
    groups = [rng.integers(0, 9000, int(rng.integers(0, 3000))).astype(np.uint64) for _ in range(64)]
    got = cm.compute_times(groups)
    want = np.array([oracle.cost(50, 0.01, 1e-6, g) for g in groups])
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
    big = [np.array([2 ** 27, 3, 2 ** 30], np.uint64)]  # exercises the sequential f64 path
    assert cm.compute_times(big)[0] == oracle.cost(50, 0.01, 1e-6, big[0])


@pytest.mark.skipif(not os.path.exists(os.path.join(HERE, "cfg2_partition.npz")), reason="cfg2 golden absent")
def test_cfg2_full_size(P, cuda):
    """config 2: 65,536 samples over 8 ranks, bit-exact FBS / VBS (alpha 1, 2)
    plans and per-rank costs against the reference's own outputs."""
    import time
    from paper_2604_24073_b200.sim import CostModel
    z = np.load(os.path.join(HERE, "cfg2_partition.npz"))
    metas = _metas(P, z["lens"], z["origin"], z["local"])
    plan = P.fbs_partition(metas, 8)
    assert np.array_equal(plan.assignment, z["fbs_assign"])
    assert np.array_equal(np.concatenate(plan.receive_order), z["fbs_order"])
    for k in (1, 2):
        t = time.time()
        plan = P.vbs_partition(metas, 8, float(k))
        dt = time.time() - t
        assert np.array_equal(plan.assignment, z[f"vbs{k}_assign"]), k
        assert np.array_equal(np.concatenate(plan.receive_order), z[f"vbs{k}_order"]), k
        assert [len(o) for o in plan.receive_order] == z[f"vbs{k}_sizes"].tolist()
        print(f"vbs alpha={k} 65536x8 on GPU: {dt * 1e3:.1f} ms")
    lens = z["lens"]
    for row, c2 in zip(z["cost"], (0.0, 1e-6)):
        got = CostModel(50.0, 0.01, c2).compute_times([lens[r * 8192:(r + 1) * 8192] for r in range(8)])
        assert np.array_equal(got.view(np.uint64), row.view(np.uint64))


@pytest.mark.parametrize("partition,iters", [("fbs", 3), ("vbs", 1)])
def test_balancer_gpu_partition_gloo_world2(cuda, oracle, tmp_path, partition, iters):
    """The three-stage balancer at world size 2 (gloo plumbing) with the GPU
    FBS / VBS partition: every rank's balanced batch equals the plan the C
    oracle computes from the gathered lengths, applied to the global batch."""
    import json
    import socket
    import subprocess
    import sys
    from balancer_cases import make_raw
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    world, out = 2, str(tmp_path / "bal")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(os.path.dirname(os.path.abspath(__file__)), "balancer_worker.py"),
           out, partition, str(iters), "1"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    for i in range(iters):
        raws = [make_raw(i, rr, world) for rr in range(world)]
        lens = np.asarray([x.uih.size for rr in range(world) for x in raws[rr].samples], np.uint64)
        origin = np.repeat(np.arange(world), 6).astype(np.int32)
        local = np.tile(np.arange(6), world).astype(np.int32)
        if partition == "fbs":
            _, order = oracle.fbs(lens, origin, local, world)
        else:
            _, order, _ = oracle.vbs(lens, origin, local, world, 1.0)
        glob = [x for rr in range(world) for x in raws[rr].samples]
        for rank in range(world):
            got = json.load(open(f"{out}.rank{rank}.json"))["taken"][i]
            want = [glob[int(g)] for g in order[rank]]
            assert [g[0] for g in got] == [w.uih.tolist() for w in want]
            assert [g[2] for g in got] == [w.label for w in want]
