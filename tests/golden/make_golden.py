"""Regenerate the golden fixtures from the reference itself (oracle/_ref,
built from /root/reference/proj/src). Run here (not on the GPU box):

    python tests/golden/make_golden.py

Writes tests/golden/*.npz. Each fixture records the inputs (ids from the
reference's own workload generator) and the reference's outputs (final table
bytes, IterationStats, collision sets, partition plans) for the cases the
reference's tests use (test_embedding.cpp, test_partition.cpp,
acceptance.cpp)."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
sys.path.insert(0, os.path.join(HERE, "..", ".."))
from oracle import Reference, build  # noqa: E402

# (name, world, batch, max_uih, lo, hi, table_rows, ratio, seed, iters, dim, lr, table_seed)
ENGINE_CASES = [
    # test_embedding.cpp:237-251
    ("seeded_2r", 2, 3, 6, 1, 6, 8, None, 1234, 3, 4, 0.25, 42),
]
# test_embedding.cpp:253-272: ranks {1,2,4} x ratio {0, .3, 1}
for ranks in (1, 2, 4):
    for ratio in (0.0, 0.3, 1.0):
        ENGINE_CASES.append((f"ratio_{ranks}r_{int(ratio * 10)}", ranks, 4, 12, 0, 12, 64, ratio,
                             99 + ranks, 7, 3, 0.125, 5))
# acceptance.cpp:44-85 (criterion 1) at reduced iteration count, ranks {1,2,4,8}
for ranks in (1, 2, 4, 8):
    for ratio in (0.0, 0.05, 0.25, 1.0):
        ENGINE_CASES.append((f"accept_{ranks}r_{int(ratio * 100)}", ranks, 4, 16, 1, 16, 1024, ratio,
                             1000 + ranks * 100 + int(ratio * 100), 12, 8, 0.1, 7))


def flat(batches):
    lens = np.array([len(b) for it in batches for b in it], np.uint64)
    ids = np.concatenate([np.asarray(b, np.uint64) for it in batches for b in it]) if lens.sum() else \
        np.zeros(0, np.uint64)
    return ids, lens


def main():
    build(ref=True)
    R = Reference()
    out = {}
    for (name, world, batch, max_uih, lo, hi, rows, ratio, seed, iters, dim, lr, tseed) in ENGINE_CASES:
        b = R.generate_uniform(world, batch, max_uih, lo, hi, rows, ratio, seed, iters)
        ids, lens = flat(b)
        t_sync, _ = R.run_engine(False, world, b, rows, dim, lr, tseed)
        t_prio, st = R.run_engine(True, world, b, rows, dim, lr, tseed)
        assert np.array_equal(t_sync.view(np.uint64), t_prio.view(np.uint64)), name
        out[name] = dict(world=world, iters=iters, rows=rows, dim=dim, lr=lr, seed=tseed, ids=ids,
                         lens=lens, table=t_sync, stats=st)
    np.savez_compressed(os.path.join(HERE, "engine_cases.npz"),
                        **{f"{k}__{f}": np.asarray(v) for k, d in out.items() for f, v in d.items()})

    # collision fuzz (test_embedding.cpp:110-129 / acceptance.cpp:516-528) +
    # cfg1-sized sets, with the reference's split
    from paper_2604_24073_b200.workload import splitmix_stream, zipf_batch
    coll = {}
    st = splitmix_stream(2718, 200 * 130)
    at = 0
    for k in range(200):
        na, nb = int(st[at] % 60), int(st[at + 1] % 60)
        at += 2
        a = st[at:at + na] % np.uint64(80)
        at += na
        bb = st[at:at + nb] % np.uint64(80)
        at += nb
        co, exc, exn, ua, ub = R.compute_collision(a, bb)
        coll[f"f{k}"] = (a, bb, co, exc, exn)
    a = zipf_batch(20261018, 4096, 1_000_000)
    bb = zipf_batch(20261018, 4096, 1_000_000, offset=4096)
    co, exc, exn, ua, ub = R.compute_collision(a, bb)
    coll["cfg1"] = (a, bb, co, exc, exn)
    np.savez_compressed(os.path.join(HERE, "collision_cases.npz"),
                        **{f"{k}__{i}": v for k, tup in coll.items() for i, v in enumerate(tup)})

    # partition plans (test_partition.cpp KATs + random instances + cfg2 sample)
    part = {}
    rng = np.random.default_rng(7)
    cases = [("kat_fbs_9753", [9, 7, 5, 3], 2), ("kat_vbs_4321", [4, 3, 2, 1], 2),
             ("kat_vbs_111", [1, 1, 1], 2), ("kat_vbs_22222", [2, 2, 2, 2, 2], 3),
             ("kat_vbs_42222", [4, 2, 2, 2, 2], 3)]
    for k in range(40):
        n = int(rng.integers(1, 9))
        m = n * int(rng.integers(1, 13))
        cases.append((f"rand{k}", rng.integers(0, 2000, m).tolist(), n))
    hist = np.zeros(8193)
    hist[16:] = np.arange(16, 8193, dtype=np.float64) ** -2.0
    lens_cfg2, _ = R.generate_lengths(hist, 8192, 8, 1024, 20261020)
    cases.append(("cfg2_8k", lens_cfg2.tolist(), 8))
    for name, lens, n in cases:
        lens = np.asarray(lens, np.uint64)
        m = lens.size
        per = (m + n - 1) // n
        origin = (np.arange(m) // per).astype(np.int32)
        local = (np.arange(m) % per).astype(np.int32)
        entry = [lens, origin, local, np.int64(n)]
        if m % n == 0:
            a, order = R.fbs(lens, origin, local, n)
            entry += [a, np.concatenate(order)]
        else:
            entry += [np.zeros(0, np.int32), np.zeros(0, np.uint64)]
        for alpha in (1.0, 2.0):
            if n <= m and (m <= 2048 or alpha == 1.0):
                a, order, sizes = R.vbs(lens, origin, local, n, alpha)
                entry += [a, np.concatenate(order), sizes]
            else:
                entry += [np.zeros(0, np.int32), np.zeros(0, np.uint64), np.zeros(0, np.int32)]
        part[name] = entry
    np.savez_compressed(os.path.join(HERE, "partition_cases.npz"),
                        **{f"{k}__{i}": np.asarray(v) for k, e in part.items() for i, v in enumerate(e)})
    print("wrote", len(out), "engine cases,", len(coll), "collision cases,", len(part), "partition cases")


if __name__ == "__main__":
    main()
