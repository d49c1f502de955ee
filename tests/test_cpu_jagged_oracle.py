"""The jagged oracle (test infrastructure) pinned to the reference's own
expected values (proj/tests/test_jagged.cpp:58-185)."""
import pytest

import jagged_oracle as O


def test_oracle_pins():
    segs = [[1, 2], [3], [4, 5, 6]]
    assert O.permute(segs, [2, 0, 1]) == [[4, 5, 6], [1, 2], [3]]       # test_jagged.cpp:58-64
    assert O.permute([[7], [8]], [0, 0]) == [[7], [7]]                    # :74-78
    with pytest.raises(IndexError, match="index 2"):                      # :80-84
        O.permute([[1], [2]], [0, 2])
    assert O.dispatch(segs, [(0, 2), (2, 1)]) == [[[1, 2], [3]], [[4, 5, 6]]]
    assert O.combine([[[1], [2, 2]], [[3]]]) == [[1], [2, 2], [3]]        # :132-136
    fm = [[10], [11, 11], [20], [21]]
    assert O.keyed_transpose(fm, 2, True) == [[10], [20], [11, 11], [21]]  # :162-168
    assert O.keyed_transpose(O.keyed_transpose(fm, 2, True), 2, False) == fm
