"""GPU parity of the pooled (bag) lookup and its backward scatter + update
(BASELINE config 3's operator; fsx_pooled_* / PooledEmbedding) against the C
oracle's restatement (oracle/fsx_oracle.c fso_pooled_*): f64 tables bit-exact,
fp32 tables bit-exact against the oracle's fp32-storage model, at the row
widths the kernels specialise on, with empty bags, repeated ids inside a bag,
hot rows split into chunks, and a table-wise shard (config 3's layout:
table t on rank t, gid = row * T + t)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _bits(x):
    return np.ascontiguousarray(x, np.float64).reshape(-1).view(np.uint64)


def _bags(rng, n_bags, rows, max_len, zipf=True, mul=1, add=0):
    lens = rng.integers(0, max_len + 1, n_bags)
    lens[::7] = 0  # empty bags
    lens[5] = 9 * max_len  # a hot bag: split into chunks
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
    n = int(offs[-1])
    if zipf:
        r = np.minimum(rng.zipf(1.3, n) - 1, rows - 1)
    else:
        r = rng.integers(0, rows, n)
    return (r.astype(np.uint64) * np.uint64(mul) + np.uint64(add)), offs


def _run(cuda, geom, shard_id, dtype, ids, offs, grads_fn, chunk, steps=2):
    import torch
    from paper_2604_24073_b200 import embedding as E
    ctx = E.Context(0, 0, 1)
    shard = E.ShardView(geom, shard_id, 0.05, 11, dtype=dtype, ctx=ctx)
    pe = E.PooledEmbedding(shard, max_occurrences=max(ids.size, 1), max_bags=offs.size - 1, reduce_chunk=chunk)
    s = torch.cuda.Stream()
    outs = []
    with torch.cuda.stream(s):
        for _ in range(steps):
            out = pe.forward(ids, offs, stream=s)
            outs.append(out.double().cpu().numpy() if out.numel() else np.zeros((0, geom.dim)))
            pe.backward(grads_fn(out), stream=s)
    s.synchronize()
    ctx.sync()
    vals = shard.values()
    pe.close()
    return outs, vals


@pytest.mark.parametrize("dtype,dim,chunk", [("f64", 16, 0), ("f64", 128, 4), ("f32", 128, 64), ("f32", 256, 16),
                                             ("f32", 12, 0), ("f64", 5, 3)])
def test_pooled_bitwise(cuda, oracle, dtype, dim, chunk):
    from paper_2604_24073_b200 import embedding as E
    rng = np.random.default_rng(dim + chunk)
    rows = 3000
    ids, offs = _bags(rng, 700, rows, 40)
    geom = E.TableGeometry(rows, dim, 1)
    f32 = dtype == "f32"
    outs, vals = _run(cuda, geom, 0, dtype, ids, offs, lambda o: o * 0.125 + 0.0625, chunk)
    table = oracle.init_shard(rows, dim, 1, 0, 11)
    if f32:
        table = table.astype(np.float32).astype(np.float64)
    for out in outs:
        want = oracle.pooled_forward(table, ids, offs, store_f32=f32, reduce_chunk=chunk)
        assert np.array_equal(_bits(out), _bits(want))
        g = want * 0.125 + 0.0625
        if f32:  # the torch fixture in float: fl(fl(x * 0.125) + 0.0625)
            g = ((want.astype(np.float32) * np.float32(0.125)) + np.float32(0.0625)).astype(np.float64)
        table = oracle.pooled_backward(table, ids, offs, g, 0.05, store_f32=f32, reduce_chunk=chunk)
    assert np.array_equal(_bits(vals), _bits(table))


def test_pooled_table_wise_shard(cuda, oracle):
    """Config 3's layout: T tables of R rows table-wise sharded over T ranks
    (in the reference's terms gid = row * T + t under gid mod T, so table t is
    shard t). Shard 3's bags only carry its own gids."""
    from paper_2604_24073_b200 import embedding as E
    T, R, dim, t = 8, 2000, 128, 3
    rng = np.random.default_rng(5)
    ids, offs = _bags(rng, 500, R, 30, mul=T, add=t)
    geom = E.TableGeometry(T * R, dim, T)
    outs, vals = _run(cuda, geom, t, "f32", ids, offs, lambda o: o * 0.125 + 0.0625, 64)
    table = oracle.init_shard(T * R, dim, 1, 0, 11).astype(np.float32).astype(np.float64)
    for out in outs:
        want = oracle.pooled_forward(table, ids, offs, store_f32=True, reduce_chunk=64)
        assert np.array_equal(_bits(out), _bits(want))
        g = ((want.astype(np.float32) * np.float32(0.125)) + np.float32(0.0625)).astype(np.float64)
        table = oracle.pooled_backward(table, ids, offs, g, 0.05, store_f32=True, reduce_chunk=64)
    assert np.array_equal(_bits(vals), _bits(table[t::T]))


def test_pooled_errors(cuda):
    import torch
    from paper_2604_24073_b200 import embedding as E
    from paper_2604_24073_b200.errors import DomainError, InvalidArgument, ProtocolError
    ctx = E.Context(0, 0, 1)
    shard = E.ShardView(E.TableGeometry(16, 4, 2), 0, 0.1, 1, dtype="f64", ctx=ctx)
    pe = E.PooledEmbedding(shard, max_occurrences=8, max_bags=4)
    with pytest.raises(ProtocolError):
        pe.backward(torch.zeros((1, 4), dtype=torch.float64, device="cuda"))
    pe.forward(np.array([2, 4, 5], np.uint64), np.array([0, 2, 3], np.uint64))
    with pytest.raises(DomainError, match="row id 5 is not owned by shard 0"):
        ctx.sync()
    pe.forward(np.array([2, 40], np.uint64), np.array([0, 2], np.uint64))
    with pytest.raises(DomainError, match="row id 40 out of range"):
        ctx.sync()
    with pytest.raises(InvalidArgument):
        pe.forward(np.arange(0, 20, 2, dtype=np.uint64), np.array([0, 10], np.uint64))
    pe.close()
