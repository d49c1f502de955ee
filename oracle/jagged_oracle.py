"""Test infrastructure only (never imported by the product): list-of-lists
restatement of the reference's jagged reshuffle ops, the same naive oracles
its own tests use (proj/tests/test_jagged.cpp:18-27) plus keyed_transpose's
index map (proj/include/freescale/jagged.hpp:227-248)."""


def permute(segs, perm):
    """indexed_permute (jagged.hpp:89-111) / oracle_permute (test_jagged.cpp:18-22)"""
    for k in perm:
        if not 0 <= k < len(segs):
            raise IndexError(f"indexed_permute: segment index {k} out of range (have {len(segs)})")
    return [list(segs[k]) for k in perm]


def dispatch(segs, ranges):
    """ranged_dispatch (jagged.hpp:118-155) / oracle_slice (test_jagged.cpp:24-27)"""
    return [[list(s) for s in segs[a:a + c]] for a, c in ranges]


def combine(parts):
    """ranged_combine (jagged.hpp:157-176)"""
    return [list(s) for p in parts for s in p]


def keyed_transpose(segs, num_keys, feature_major=True):
    """keyed_transpose (jagged.hpp:227-248): (f, s) at f*S+s <-> s*F+f"""
    S = len(segs) // num_keys
    out = [None] * len(segs)
    for f in range(num_keys):
        for s in range(S):
            if feature_major:
                out[s * num_keys + f] = list(segs[f * S + s])
            else:
                out[f * S + s] = list(segs[s * num_keys + f])
    return out
