"""GPU parity of the embedding engines (SynchronizedEmbedding /
PrioritizedEmbedding over libfsx) against the reference's golden tables and
the C oracle. f64 tables: bit-exact (same per-row accumulation order);
fp32 tables: bit-exact with the oracle's fp32-storage model, including the
engine's chunk and PRESUM associations. Multi-rank cases run as
threads of one process (several ranks per GPU when the box has fewer GPUs),
exactly like the reference's InProcessFabric tests."""
import numpy as np
import pytest

from golden_io import engine_cases

pytestmark = pytest.mark.gpu


def frel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), 1e-3)))


@pytest.fixture(scope="module")
def ENG():
    return engine_cases()


@pytest.fixture(scope="module")
def drv(cuda):
    import engine_driver
    return engine_driver


def _bits(x):
    return np.ascontiguousarray(x, np.float64).reshape(-1).view(np.uint64)


@pytest.mark.parametrize("prio", [False, True])
def test_seeded_two_ranks_bitwise(drv, ENG, prio):
    from paper_2604_24073_b200.embedding import TableGeometry
    c = ENG["seeded_2r"]
    geom = TableGeometry(c["rows"], c["dim"], c["world"])
    table, stats = drv.run_engine(prio, c["batches"], geom, c["lr"], c["seed"], with_stats=prio)
    assert np.array_equal(_bits(table), _bits(c["table"]))
    if prio:
        got = np.array([[s.collision_rows, s.unique_next_rows, s.blocking_bytes] for s in stats], np.uint64)
        assert np.array_equal(got, c["stats"])


def test_all_golden_cases_bitwise(drv, ENG):
    from paper_2604_24073_b200.embedding import TableGeometry
    for name, c in ENG.items():
        geom = TableGeometry(c["rows"], c["dim"], c["world"])
        for prio in (False, True):
            table, stats = drv.run_engine(prio, c["batches"], geom, c["lr"], c["seed"], with_stats=prio)
            assert np.array_equal(_bits(table), _bits(c["table"])), (name, prio)
            if prio:
                got = np.array([[s.collision_rows, s.unique_next_rows, s.blocking_bytes] for s in stats],
                               np.uint64)
                assert np.array_equal(got, c["stats"]), (name, got, c["stats"])


def test_boundary_runs(drv, oracle):
    # test_embedding.cpp:274-282: one- and two-iteration runs, 2 ranks
    from paper_2604_24073_b200.embedding import TableGeometry
    geom = TableGeometry(16, 2, 2)
    one = [[np.array([1, 2], np.uint64), np.array([3, 1], np.uint64)]]
    two = one + [[np.array([2, 2, 5], np.uint64), np.array([1], np.uint64)]]
    for batches in (one, two):
        want, _ = oracle.run_engine(2, batches, 16, 2, 0.5, 7)
        for prio in (False, True):
            got, _ = drv.run_engine(prio, batches, geom, 0.5, 7)
            assert np.array_equal(_bits(got), _bits(want))


def test_sync_single_rank_dense(drv, oracle):
    # test_embedding.cpp:209-235
    from paper_2604_24073_b200.embedding import TableGeometry
    from paper_2604_24073_b200.workload import splitmix_stream
    st = splitmix_stream(77, 24)
    batches = [[(st[6 * i:6 * i + 6] % np.uint64(8)).astype(np.uint64)] for i in range(4)]
    want, _ = oracle.run_engine(1, batches, 8, 2, 0.5, 11)
    got, _ = drv.run_engine(False, batches, TableGeometry(8, 2, 1), 0.5, 11)
    assert np.array_equal(_bits(got), _bits(want))


@pytest.mark.parametrize("world", [1, 2, 4])
def test_fp32_zipf_bitwise(drv, oracle, world):
    """config-1-like Zipf traffic on fp32 tables, bit-exact with the oracle
    run on an fp32-storage table (store_f32: values rounded to float on store,
    the gradient fixture evaluated in float as the torch op does):
    * reduce_chunk=0: the reference's single left fold per row;
    * reduce_chunk=64 (parallel hot rows): the engine's fixed chunk
      association, restated in the oracle (chunk_fold); both engine modes
      agree bit for bit."""
    from paper_2604_24073_b200 import workload
    from paper_2604_24073_b200.embedding import TableGeometry
    rows, dim, iters = 50_000, 64, 4
    batches = [[workload.zipf_batch(100 + r, 3000, rows, offset=3000 * i) for r in range(world)]
               for i in range(iters)]
    geom = TableGeometry(rows, dim, world)
    exact, _ = drv.run_engine(True, batches, geom, 0.05, 3, dtype="f32", reduce_chunk=0)
    want32, _ = oracle.run_engine(world, batches, rows, dim, 0.05, 3, store_f32=True)
    assert np.array_equal(_bits(exact), _bits(want32))
    got_p, _ = drv.run_engine(True, batches, geom, 0.05, 3, dtype="f32", reduce_chunk=64)
    got_s, _ = drv.run_engine(False, batches, geom, 0.05, 3, dtype="f32", reduce_chunk=64)
    want64, _ = oracle.run_engine(world, batches, rows, dim, 0.05, 3, store_f32=True, reduce_chunk=64)
    assert np.array_equal(_bits(got_p), _bits(want64))
    assert np.array_equal(_bits(got_s), _bits(want64))


def test_f64_chunked_reduce_bitwise(drv, oracle):
    from paper_2604_24073_b200 import workload
    from paper_2604_24073_b200.embedding import TableGeometry
    rows, dim = 20_000, 32
    batches = [[workload.zipf_batch(7, 8000, rows, offset=8000 * i)] for i in range(3)]
    want, _ = oracle.run_engine(1, batches, rows, dim, 0.05, 3, reduce_chunk=16)
    for prio in (True, False):
        got, _ = drv.run_engine(prio, batches, TableGeometry(rows, dim, 1), 0.05, 3, reduce_chunk=16)
        assert np.array_equal(_bits(got), _bits(want)), prio


def test_presum_golden_cases_bitwise(drv, ENG, oracle):
    """FSX_ENGINE_PRESUM on every golden case (1-8 ranks, odd dims, empty
    batches): bit-exact with the oracle's PRESUM association (collision rows
    summed per source, then over sources in rank order), and the
    IterationStats identical to the reference's."""
    from paper_2604_24073_b200.embedding import TableGeometry
    for name, c in ENG.items():
        geom = TableGeometry(c["rows"], c["dim"], c["world"])
        got, stats = drv.run_engine(True, c["batches"], geom, c["lr"], c["seed"], presum=True, with_stats=True)
        want, _ = oracle.run_engine(c["world"], c["batches"], c["rows"], c["dim"], c["lr"], c["seed"],
                                    presum=True)
        assert np.array_equal(_bits(got), _bits(want)), name
        assert frel(got, c["table"]) < 1e-12, name
        st = np.array([[s.collision_rows, s.unique_next_rows, s.blocking_bytes] for s in stats], np.uint64)
        assert np.array_equal(st, c["stats"]), name


@pytest.mark.parametrize("world", [1, 2, 4])
def test_presum_fp32_zipf_bitwise(drv, oracle, world):
    """PRESUM + reduce_chunk 64 on fp32 tables (the bench's numeric path at
    N > 1): bit-exact with the oracle's fp32-storage PRESUM association, and
    the IterationStats (reference accounting) identical to the exact
    protocol's."""
    from paper_2604_24073_b200 import workload
    from paper_2604_24073_b200.embedding import TableGeometry
    rows, dim, iters = 50_000, 64, 4
    batches = [[workload.zipf_batch(200 + r, 3000, rows, offset=3000 * i) for r in range(world)]
               for i in range(iters)]
    geom = TableGeometry(rows, dim, world)
    a, st_a = drv.run_engine(True, batches, geom, 0.05, 3, dtype="f32", reduce_chunk=64, presum=True,
                             with_stats=True)
    want, _ = oracle.run_engine(world, batches, rows, dim, 0.05, 3, store_f32=True, reduce_chunk=64,
                                presum=True)
    assert np.array_equal(_bits(a), _bits(want))
    _, st_x = drv.run_engine(True, batches, geom, 0.05, 3, dtype="f32", reduce_chunk=64, with_stats=True)
    key = lambda st: [(s.collision_rows, s.unique_next_rows, s.blocking_bytes) for s in st]  # noqa: E731
    assert key(st_a) == key(st_x)


def test_protocol_order_errors(cuda):
    # test_embedding.cpp:329-342
    import torch
    from paper_2604_24073_b200 import embedding as E
    from paper_2604_24073_b200.errors import ProtocolError
    shard = E.ShardView(E.TableGeometry(4, 1, 1), 0, 0.1, 1)
    prio = E.PrioritizedEmbedding(shard, max_occurrences=16)
    with pytest.raises(ProtocolError):
        prio.backward(torch.zeros(1, device="cuda"))
    prio.forward([1], None)
    with pytest.raises(ProtocolError):
        prio.forward([1], None)


@pytest.mark.parametrize("dtype,dim,world", [("f64", 256, 1), ("f32", 512, 2), ("f32", 96, 1), ("f64", 16, 2),
                                             ("f32", 256, 3)])
def test_update_row_widths_bitwise(drv, oracle, dtype, dim, world):
    """Every row width the update kernels specialise on (1, 2 or 4 16-byte
    vectors per lane, partial warps, f32 and f64): hot rows split into
    chunks of 16 occurrences, bit-exact with the oracle's chunk association
    in both engine modes."""
    from paper_2604_24073_b200 import workload
    from paper_2604_24073_b200.embedding import TableGeometry
    rows, iters = 4_000, 3
    batches = [[workload.zipf_batch(300 + r, 2500, rows, offset=2500 * i) for r in range(world)]
               for i in range(iters)]
    geom = TableGeometry(rows, dim, world)
    want, _ = oracle.run_engine(world, batches, rows, dim, 0.05, 3, store_f32=dtype == "f32", reduce_chunk=16)
    for prio in (True, False):
        got, _ = drv.run_engine(prio, batches, geom, 0.05, 3, dtype=dtype, reduce_chunk=16)
        assert np.array_equal(_bits(got), _bits(want)), prio
