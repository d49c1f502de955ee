"""Jagged reshuffle kernels against the reference's own test
cases (proj/tests/test_jagged.cpp) and the list-of-lists oracle
(oracle/jagged_oracle.py): bit-exact segment contents, container invariants,
the same exception classes and messages."""
import numpy as np
import pytest

import jagged_oracle as O

pytestmark = pytest.mark.gpu


def _rng(seed):
    s = [seed & 0xFFFFFFFFFFFFFFFF]

    def nxt():
        s[0] = (s[0] + 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF
        z = s[0]
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & 0xFFFFFFFFFFFFFFFF
        return z ^ (z >> 31)
    return nxt


def _random_segs(nxt, max_segments=20, max_len=50):
    return [[nxt() for _ in range(nxt() % (max_len + 1))] for _ in range(nxt() % (max_segments + 1))]


def _invariants(t):
    offs = t.offsets()
    assert offs.size == t.num_segments() + 1 and offs[0] == 0
    assert int(offs[-1]) == t.total_values() == int(t.lengths().sum())
    assert np.array_equal(t.device_offsets().cpu().numpy().view(np.uint64), offs)


def test_construction_and_segments(cuda):
    from paper_2604_24073_b200 import jagged as J
    from paper_2604_24073_b200.errors import InvalidArgument, OutOfRange
    with pytest.raises(InvalidArgument, match="does not match"):
        J.IdJagged([1, 2, 3], [2, 2])
    t = J.IdJagged.from_segments([[1], [], [2, 3]])
    assert t.segment(1).numel() == 0
    with pytest.raises(OutOfRange, match="segment index 3 out of range"):
        t.segment(3)
    _invariants(t)


def test_indexed_permute_cases(cuda):
    from paper_2604_24073_b200 import jagged as J
    from paper_2604_24073_b200.errors import OutOfRange
    segs = [[1, 2], [3], [4, 5, 6]]
    t = J.IdJagged.from_segments(segs)
    out = J.indexed_permute(t, [2, 0, 1])
    assert out.to_segments() == O.permute(segs, [2, 0, 1]) == [[4, 5, 6], [1, 2], [3]]
    assert J.indexed_permute(t, [0, 1, 2]) == t
    assert J.indexed_permute(J.IdJagged.from_segments([[7], [8]]), [0, 0]).to_segments() == [[7], [7]]
    with pytest.raises(OutOfRange, match="index 2"):
        J.indexed_permute(J.IdJagged.from_segments([[1], [2]]), [0, 2])
    # f64 values and an empty permutation
    v = J.JaggedTensor(np.array([0.5, -1.25, 3.0]), [1, 2])
    assert J.indexed_permute(v, [1, 0]).to_segments() == [[-1.25, 3.0], [0.5]]
    assert J.indexed_permute(t, []).num_segments() == 0


def test_indexed_permute_inverse_fuzz(cuda):
    from paper_2604_24073_b200 import jagged as J
    nxt = _rng(2024)
    for _ in range(60):
        segs = _random_segs(nxt)
        t = J.IdJagged.from_segments(segs)
        perm = list(range(len(segs)))
        for i in range(len(perm) - 1, 0, -1):
            j = nxt() % (i + 1)
            perm[i], perm[j] = perm[j], perm[i]
        inv = [0] * len(perm)
        for j, k in enumerate(perm):
            inv[k] = j
        p = J.indexed_permute(t, perm)
        assert p.to_segments() == O.permute(segs, perm)
        back = J.indexed_permute(p, inv)
        assert back == t
        _invariants(back)


def test_ranged_dispatch_and_combine(cuda):
    from paper_2604_24073_b200 import jagged as J
    from paper_2604_24073_b200.errors import InvalidArgument, OutOfRange
    segs = [[1, 2], [3], [4, 5, 6]]
    t = J.IdJagged.from_segments(segs)
    parts = J.ranged_dispatch(t, [(0, 2), (2, 1)])
    assert [p.to_segments() for p in parts] == O.dispatch(segs, [(0, 2), (2, 1)])
    assert J.ranged_dispatch(t, [(0, 3)])[0] == t
    parts = J.ranged_dispatch(t, [(1, 0), (0, 3)])
    assert parts[0].num_segments() == 0 and parts[1] == t
    with pytest.raises(InvalidArgument, match="overlapping"):
        J.ranged_dispatch(t, [(0, 2), (1, 2)])
    with pytest.raises(OutOfRange, match="exceeds segment count"):
        J.ranged_dispatch(t, [(2, 2)])
    a = J.IdJagged.from_segments([[1], [2, 2]])
    b = J.IdJagged.from_segments([[3]])
    assert J.ranged_combine([a, b]).to_segments() == [[1], [2, 2], [3]]
    assert J.ranged_combine([a]) == a
    empty = J.IdJagged.from_segments([])
    assert J.ranged_combine([empty, a, empty]) == a
    nxt = _rng(77)
    for _ in range(60):
        segs = _random_segs(nxt)
        t = J.IdJagged.from_segments(segs)
        ranges, at = [], 0
        while at < len(segs):
            take = 1 + nxt() % (len(segs) - at)
            ranges.append((at, take))
            at += take
        ranges = ranges or [(0, 0)]
        back = J.ranged_combine(J.ranged_dispatch(t, ranges))
        assert back == t
        _invariants(back)


def test_keyed_transpose(cuda):
    from paper_2604_24073_b200 import jagged as J
    from paper_2604_24073_b200.errors import InvalidArgument
    inner = J.IdJagged.from_segments([[10], [11, 11], [20], [21]])
    kt = J.KeyedJaggedTensor(["A", "B"], inner, J.KeyedLayout.FeatureMajor)
    bt = J.keyed_transpose(kt)
    assert bt.layout == J.KeyedLayout.BatchMajor
    assert bt.inner.to_segments() == [[10], [20], [11, 11], [21]]
    for f in range(2):
        for s in range(2):
            assert kt.at(f, s).tolist() == bt.at(f, s).tolist()
    one = J.KeyedJaggedTensor(["only"], J.IdJagged.from_segments([[1], [2], [3]]))
    o = J.keyed_transpose(one)
    assert o.layout == J.KeyedLayout.BatchMajor and o.inner == one.inner
    with pytest.raises(InvalidArgument, match="not divisible"):
        J.KeyedJaggedTensor(["A", "B"], J.IdJagged.from_segments([[1], [2], [3]]))
    nxt = _rng(99)
    for _ in range(40):
        F, S = 1 + nxt() % 4, 1 + nxt() % 6
        segs = [[nxt() for _ in range(nxt() % 5)] for _ in range(F * S)]
        kt = J.KeyedJaggedTensor([f"k{f}" for f in range(F)], J.IdJagged.from_segments(segs))
        tt = J.keyed_transpose(kt)
        assert tt.inner.to_segments() == O.keyed_transpose(segs, F, True)
        assert J.keyed_transpose(tt) == kt


def test_fuzzed_invariants_with_repetition(cuda):
    from paper_2604_24073_b200 import jagged as J
    nxt = _rng(123)
    for _ in range(80):
        segs = _random_segs(nxt, 40, 50)
        if not segs:
            continue
        perm = [nxt() % len(segs) for _ in range(len(segs))]
        out = J.indexed_permute(J.IdJagged.from_segments(segs), perm)
        assert out.to_segments() == O.permute(segs, perm)
        _invariants(out)
