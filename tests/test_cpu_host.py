"""CPU-only checks of the boundary and the host logic (no GPU needed):
libfsx.so loads without a driver and exports every symbol include/fsx.h
declares; host-side pieces (autotune, plan bookkeeping) match the reference."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "fsx.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fsx_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    import ctypes
    from paper_2604_24073_b200 import _lib
    lib = _lib.lib()  # raises if the extension is missing: no fallback
    declared = _declared()
    assert len(declared) >= 30
    for name in declared:
        assert hasattr(lib, name), name
    # the Python binding knows them all too
    assert set(declared) <= set(_lib.EXPORTED), set(declared) - set(_lib.EXPORTED)
    assert lib.fsx_version().startswith(b"libfsx")
    assert isinstance(ctypes.CDLL(_lib.LIB_PATH), ctypes.CDLL)


def test_error_classes_map():
    from paper_2604_24073_b200 import errors
    assert isinstance(errors.from_status(-1, "x"), ValueError)
    assert isinstance(errors.from_status(-4, "x"), errors.ProtocolError)
    assert isinstance(errors.from_status(-5, "x"), errors.CollectiveError)


def test_autotune_kats_via_c_abi(oracle):
    # test_partition.cpp:119-139 through libfsx's host autotune_update
    from paper_2604_24073_b200 import partition as P
    t = P.AutoTuneState([4, 4], [0.0, 0.0], initialized=True)
    P.autotune_update(t, [10, 10])
    assert t.local_batch_size == [4, 4]
    t = P.AutoTuneState([4, 4], [0.0, 0.0], initialized=True)
    P.autotune_update(t, [12, 8])
    assert t.local_batch_size == [3, 5]
    t = P.AutoTuneState([1, 7], [0.0, 0.0], initialized=True)
    P.autotune_update(t, [20, 1])
    assert t.local_batch_size[0] == 1 and sum(t.local_batch_size) == 8
    from paper_2604_24073_b200.errors import ProtocolError
    with pytest.raises(ProtocolError):
        P.autotune_update(P.AutoTuneState(), [1.0])


def test_autotune_matches_oracle_bitwise(oracle):
    # acceptance.cpp:531-545 style: 1500 rounds conserve the batch; f64 EMAs
    # bit-identical to the restatement
    from paper_2604_24073_b200 import partition as P
    from paper_2604_24073_b200.workload import rng_double
    u = rng_double(99, 1500 * 4)
    times = 1.0 + u * 30.0
    t = P.AutoTuneState([8, 8, 8, 8], [0.0] * 4, initialized=True)
    sizes, ema, eg = [8, 8, 8, 8], [0.0] * 4, 0.0
    for k in range(1500):
        P.autotune_update(t, times[4 * k:4 * k + 4])
        assert sum(t.local_batch_size) == 32
    s2, e2, g2 = oracle.autotune(sizes, ema, eg, times)
    assert t.local_batch_size == s2.tolist()
    assert np.array_equal(np.array(t.ema_local).view(np.uint64), e2.view(np.uint64))
    assert np.float64(t.ema_global).view(np.uint64) == np.float64(g2).view(np.uint64)


def test_plan_bookkeeping():
    # validate / exchange_lists / identity (partition.cpp:96-155, 271-290)
    from paper_2604_24073_b200 import partition as P
    from paper_2604_24073_b200.errors import InvalidArgument
    metas = P.metas_from_lengths([5, 1, 4, 2], 2)
    ident = P.identity_partition(metas, 2)
    ident.validate(4, True)
    assert [o.tolist() for o in ident.receive_order] == [[0, 1], [2, 3]]
    lists = ident.exchange_lists(metas)
    assert lists == [[[0, 1], []], [[], [0, 1]]]
    bad = P.PartitionPlan(2, np.array([0, 0, 1, 1], np.int32), [np.array([0, 1]), np.array([2])])
    with pytest.raises(InvalidArgument, match="sample 3 not assigned"):
        bad.validate(4, False)
    dup = P.PartitionPlan(2, np.array([0, 0, 1, 1], np.int32), [np.array([0, 1]), np.array([2, 3, 3])])
    with pytest.raises(InvalidArgument, match="assigned more than once"):
        dup.validate(4, False)
    with pytest.raises(InvalidArgument, match="rank 0 receives 1 samples, expected 2"):
        P.PartitionPlan(2, np.array([0, 1, 1, 1], np.int32), [np.array([0]), np.array([1, 2, 3])]).validate(4, True)
    custom = P.custom_partition(lambda m, n: P.identity_partition(m, n), metas, 2)
    assert custom.num_ranks == 2
