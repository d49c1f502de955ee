"""CPU: pin the C restatement (oracle/fsx_oracle.c) to the reference — to its
golden fixtures always, and to the live reference library when oracle/_ref is
built (this container). No GPU involved."""
import numpy as np
import pytest

from golden_io import collision_cases, engine_cases, partition_cases


@pytest.fixture(scope="module")
def ENG():
    return engine_cases()


def test_initial_value_kats(oracle):
    # SURVEY §8(c) derived KATs from the reference
    assert oracle.initial_value(1, 0, 0) == float.fromhex("0x1.7798b6dd7d398p-4")
    assert oracle.initial_value(1, 999999, 127) == float.fromhex("0x1.8dec96a266f52p-4")
    assert oracle.initial_value(42, 12345, 7) == float.fromhex("0x1.4040de7d0e36ap-5")
    assert oracle.initial_value(5, 1023, 7) == float.fromhex("-0x1.3158948c3b7p-8")


def test_cost_model_kat(oracle):
    assert oracle.cost(50, 0.01, 1e-6, [16, 8192, 97, 1000]) == float.fromhex("0x1.a656496ededafp+7")
    assert oracle.cost(50, 0.01, 0, [100, 300]) == pytest.approx(54.0)


def test_engine_cases_bitwise(oracle, ENG):
    for name, c in ENG.items():
        table, stats = oracle.run_engine(c["world"], c["batches"], c["rows"], c["dim"], c["lr"], c["seed"],
                                         with_stats=True)
        assert np.array_equal(table.reshape(-1).view(np.uint64), c["table"].reshape(-1).view(np.uint64)), name
        assert np.array_equal(stats, c["stats"]), name


def test_collision_cases(oracle):
    for name, (a, b, co, exc, exn) in collision_cases().items():
        got = oracle.compute_collision(a, b)
        assert all(np.array_equal(x, y) for x, y in zip(got, (co, exc, exn))), name


def test_partition_cases(oracle):
    for name, c in partition_cases().items():
        if c["fbs_assign"].size:
            a, order = oracle.fbs(c["lens"], c["origin"], c["local"], c["n"])
            assert np.array_equal(a, c["fbs_assign"]), name
            assert np.array_equal(np.concatenate(order), c["fbs_order"]), name
        for alpha, (a_ref, o_ref, s_ref) in ((1.0, c["vbs1"]), (2.0, c["vbs2"])):
            if a_ref.size == 0:
                continue
            a, order, sizes = oracle.vbs(c["lens"], c["origin"], c["local"], c["n"], alpha)
            assert np.array_equal(a, a_ref), (name, alpha)
            assert np.array_equal(np.concatenate(order), o_ref), (name, alpha)
            assert np.array_equal(sizes, s_ref), (name, alpha)


def test_partition_kats(oracle):
    # test_partition.cpp:38-54, 67-75 and the derived VBS tie-break KATs
    lens = [9, 7, 5, 3]
    a, order = oracle.fbs(lens, [0, 0, 1, 1], [0, 1, 0, 1], 2)
    assert [int(sum(np.asarray(lens)[o])) for o in order] == [12, 12]
    a, order = oracle.fbs([3, 9, 1], [0, 0, 0], [0, 1, 2], 1)
    assert order[0].tolist() == [1, 0, 2]
    for lens, n, sizes in (([4, 3, 2, 1], 2, [1, 3]), ([1, 1, 1], 2, [2, 1]), ([2] * 5, 2, [3, 2]),
                           ([2] * 5, 3, [2, 2, 1]), ([4, 2, 2, 2, 2], 2, [2, 3]),
                           ([4, 2, 2, 2, 2], 3, [1, 2, 2])):
        m = len(lens)
        _, order, got = oracle.vbs(lens, [0] * m, list(range(m)), n, 1.0)
        assert got.tolist() == sizes, (lens, n)


def test_autotune_kats(oracle):
    # test_partition.cpp:119-139
    s, _, _ = oracle.autotune([4, 4], [0, 0], 0.0, [10, 10])
    assert s.tolist() == [4, 4]
    s, _, _ = oracle.autotune([4, 4], [0, 0], 0.0, [12, 8])
    assert s.tolist() == [3, 5]
    s, _, _ = oracle.autotune([1, 7], [0, 0], 0.0, [20, 1])
    assert s[0] == 1 and s.sum() == 8


def test_vbs_dp_equals_bruteforce(oracle):
    # test_partition.cpp:97-117 on the restatement
    from paper_2604_24073_b200.workload import splitmix_stream
    st = splitmix_stream(31337, 500 * 20)
    at = 0
    for _ in range(200):
        m = 2 + int(st[at] % 11)
        n = 1 + int(st[at + 1] % m)
        alpha = 1.0 + float(st[at + 2] % 3)
        at += 3
        lens = (st[at:at + m] % np.uint64(100)).astype(np.uint64)
        at += m
        _, order, _ = oracle.vbs(lens, [0] * m, list(range(m)), n, alpha)
        w = np.concatenate([lens[o].astype(np.float64) ** alpha for o in order])
        best = oracle.bruteforce(w, n)
        mx = max(float(np.sum(lens[o].astype(np.float64) ** alpha)) for o in order)
        assert mx == pytest.approx(best, rel=1e-12)


# ---- against the live reference (only where oracle/_ref was built) ----------
def test_restatement_matches_reference_live(oracle, reference):
    from paper_2604_24073_b200 import workload
    for seed in (1, 2, 3):
        b = reference.generate_uniform(3, 5, 20, 0, 20, 200, 0.4, seed, 6)
        t_ref, s_ref = reference.run_engine(True, 3, b, 200, 5, 0.2, seed)
        t_or, s_or = oracle.run_engine(3, b, 200, 5, 0.2, seed, with_stats=True)
        assert np.array_equal(t_ref.view(np.uint64), t_or.view(np.uint64))
        assert np.array_equal(s_ref, s_or)
    ids = workload.zipf_batch(5, 4096, 1_000_000)
    grads = np.random.default_rng(0).standard_normal(4096 * 16)
    v_ref, u_ref, r_ref = reference.apply_gradients(1_000_000, 16, 1, 0, 0.05, 3, ids, grads)
    init = oracle.init_shard(1_000_000, 16, 1, 0, 3)
    v_or, u_or, r_or = oracle.apply_gradients(init, 1_000_000, 16, 1, 0, 0.05, ids, grads)
    assert np.array_equal(u_ref, u_or) and np.array_equal(r_ref, r_or) and np.array_equal(v_ref, v_or)


def _py_engine(world, batches, rows, dim, lr, seed, oracle, chunk, presum, f32):
    """Pure-Python restatement of fso_run_engine_ex2 for small cases: the
    dense synchronized emulation (embedding.cpp:238-297) with the engine's
    chunk and PRESUM associations spelled out loop by loop."""
    import struct

    def r32(x):
        return struct.unpack("f", struct.pack("f", x))[0]

    table = [[oracle.initial_value(seed, g, d) for d in range(dim)] for g in range(rows)]
    if f32:
        table = [[r32(v) for v in row] for row in table]

    def fold(vals):
        if chunk == 0 or len(vals) <= chunk:
            acc = 0.0
            for v in vals:
                acc += v
            return acc
        acc = 0.0
        for c0 in range(0, len(vals), chunk):
            part = 0.0
            for v in vals[c0:c0 + chunk]:
                part += v
            acc += part
        return acc

    iters = len(batches)
    for i in range(iters):
        occ = [(int(g), r, j) for r in range(world) for j, g in enumerate(batches[i][r])]
        served = {(r, j): list(table[g]) for g, r, j in occ}
        nxt = {int(g) for r in range(world) for g in batches[i + 1][r]} if i + 1 < iters else set()
        split = presum and world > 1 and 0 < i < iters - 1
        for g in sorted({o[0] for o in occ}):
            mine = [(r, j) for gg, r, j in occ if gg == g]  # (rank, position) order
            for d in range(dim):
                def grad(rj):
                    v = served[rj][d]
                    return r32(r32(v * 0.125) + 0.0625) if f32 else v * 0.125 + 0.0625
                if split and g in nxt:
                    acc = 0.0
                    for r in range(world):
                        vals = [grad(rj) for rj in mine if rj[0] == r]
                        if vals:
                            ps = fold(vals)
                            acc += r32(ps) if f32 else ps
                else:
                    acc = fold([grad(rj) for rj in mine])
                v = table[g][d] - lr * acc
                table[g][d] = r32(v) if f32 else v
    return np.array(table, np.float64)


@pytest.mark.parametrize("chunk,presum,f32", [(0, False, False), (2, False, False), (3, True, False),
                                              (2, True, True), (0, True, True)])
def test_engine_associations_match_python_restatement(oracle, chunk, presum, f32):
    rng = np.random.default_rng(5)
    world, rows, dim = 3, 12, 3
    batches = [[rng.integers(0, rows // 2 if i % 2 else rows, size=rng.integers(0, 9)).astype(np.uint64)
                for _ in range(world)] for i in range(4)]
    want = _py_engine(world, batches, rows, dim, 0.5, 9, oracle, chunk, presum, f32)
    got, _ = oracle.run_engine(world, batches, rows, dim, 0.5, 9, store_f32=f32, reduce_chunk=chunk,
                               presum=presum)
    assert np.array_equal(got.reshape(-1).view(np.uint64), want.reshape(-1).view(np.uint64))


def test_engine_associations_degenerate_cases(oracle, ENG):
    """chunk >= every row's occurrence count and presum at one rank are the
    reference's single left fold: bit-exact with the reference goldens."""
    for name, c in ENG.items():
        big = max([len(b) for it in c["batches"] for b in it] + [1])
        t, _ = oracle.run_engine(c["world"], c["batches"], c["rows"], c["dim"], c["lr"], c["seed"],
                                 reduce_chunk=big)
        assert np.array_equal(t.reshape(-1).view(np.uint64), c["table"].reshape(-1).view(np.uint64)), name
        if c["world"] == 1:
            t, _ = oracle.run_engine(1, c["batches"], c["rows"], c["dim"], c["lr"], c["seed"], presum=True)
            assert np.array_equal(t.reshape(-1).view(np.uint64), c["table"].reshape(-1).view(np.uint64)), name


@pytest.mark.parametrize("chunk,f32", [(0, False), (2, False), (3, True)])
def test_pooled_oracle_matches_python_restatement(oracle, chunk, f32):
    """fso_pooled_* against a loop-by-loop restatement: bag sums in token
    order, then each row's tokens (row, token order) chunk-folded."""
    import struct

    def r32(x):
        return struct.unpack("f", struct.pack("f", x))[0]

    rng = np.random.default_rng(chunk)
    rows, dim = 10, 3
    lens = [3, 0, 5, 1, 4]
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
    ids = rng.integers(0, 4, int(offs[-1])).astype(np.uint64)
    table = oracle.init_shard(rows, dim, 1, 0, 2)
    if f32:
        table = np.array([[r32(v) for v in row] for row in table])
    def fold(vals):
        if chunk == 0 or len(vals) <= chunk:
            acc = 0.0
            for v in vals:
                acc += v
            return acc
        acc = 0.0
        for c0 in range(0, len(vals), chunk):
            part = 0.0
            for v in vals[c0:c0 + chunk]:
                part += v
            acc += part
        return acc

    want_out = np.zeros((len(lens), dim))
    for b in range(len(lens)):
        for d in range(dim):
            acc = fold([table[int(ids[k]), d] for k in range(int(offs[b]), int(offs[b + 1]))])
            want_out[b, d] = r32(acc) if f32 else acc
    got = oracle.pooled_forward(table, ids, offs, store_f32=f32, reduce_chunk=chunk)
    assert np.array_equal(got.view(np.uint64), want_out.view(np.uint64))
    g = want_out * 0.5 - 0.25
    want_t = table.copy()
    bag_of = np.repeat(np.arange(len(lens)), lens)
    for r in sorted(set(int(x) for x in ids)):
        ks = [k for k in range(ids.size) if int(ids[k]) == r]
        for d in range(dim):
            acc = fold([g[bag_of[k], d] for k in ks])
            v = want_t[r, d] - 0.05 * acc
            want_t[r, d] = r32(v) if f32 else v
    got_t = oracle.pooled_backward(table, ids, offs, g, 0.05, store_f32=f32, reduce_chunk=chunk)
    assert np.array_equal(got_t.view(np.uint64), want_t.view(np.uint64))
