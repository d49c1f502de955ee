"""Workload-file replay, host side — no GPU needed: the
committed fixtures against the reference's Reader, the Python Writer against
the reference's Reader, and the libfsx host scan (fsx_workload_scan, pure C++)
against the reference's record layout and its truncation IoError text."""
import ctypes as C
import os
import shutil

import numpy as np
import pytest

from paper_2604_24073_b200 import _lib, workload_file as W
from paper_2604_24073_b200.errors import IoError

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CASES = ["small_2r", "ragged_4r", "single_1r"]


def _scan(buf: bytes, ranks: int, iteration: int = 0):
    a = np.frombuffer(buf, np.uint8)
    cap = len(buf) // 20 + 1
    off = np.zeros(cap, np.uint64)
    per = np.zeros(ranks, np.uint64)
    n, used = C.c_uint64(), C.c_uint64()
    _lib.call("fsx_workload_scan", C.c_void_p(a.ctypes.data), len(buf), ranks, iteration,
              per.ctypes.data_as(C.c_void_p), off.ctypes.data_as(C.c_void_p), cap, C.byref(n), C.byref(used))
    return per, off[:n.value], used.value


def _body(path):
    raw = open(path, "rb").read()
    hlen = int.from_bytes(raw[8:12], "little")
    return raw, raw[12 + hlen:]


@pytest.mark.parametrize("name", CASES)
def test_fixture_pinned_by_reference_reader(name, reference):
    d = reference.load_workload(os.path.join(GOLD, f"workload_{name}.bin"))
    g = np.load(os.path.join(GOLD, f"workload_{name}.npz"))
    for k in ("ids", "lens", "labels", "counts"):
        assert np.array_equal(d[k], g[k]), k


@pytest.mark.parametrize("name", CASES)
def test_host_scan_walks_every_iteration(name):
    g = np.load(os.path.join(GOLD, f"workload_{name}.npz"))
    ranks, iters = int(g["ranks"]), int(g["iterations"])
    _, body = _body(os.path.join(GOLD, f"workload_{name}.bin"))
    pos, s = 0, 0
    for it in range(iters):
        per, off, used = _scan(body[pos:], ranks, it)
        assert np.array_equal(per, g["counts"][it * ranks:(it + 1) * ranks])
        for k, o in enumerate(off):  # record k's uih count sits at its body start
            assert int.from_bytes(body[pos + int(o):pos + int(o) + 4], "little") == int(g["lens"][s + k])
        s += off.size
        pos += used
    assert pos == len(body)


def test_truncation_message_matches_reference(reference, tmp_path):
    src = os.path.join(GOLD, "workload_small_2r.bin")
    raw, body = _body(src)
    hdr = len(raw) - len(body)
    for cut in (1, 3, 37, len(body) // 2, len(body) - 1):
        p = str(tmp_path / f"cut{cut}.bin")
        open(p, "wb").write(raw[:hdr + cut])
        with pytest.raises(Exception) as ref_e:
            reference.load_workload(p)
        # the reference reads iterations in order; find the one the cut lands in
        pos, it = 0, 0
        while True:
            try:
                _, _, used = _scan(body[pos:cut], 2, it)
            except IoError as e:
                assert str(e) == str(ref_e.value)
                break
            pos += used
            it += 1


def test_python_writer_read_by_reference(reference, tmp_path):
    rng = np.random.default_rng(5)
    spec = {"batch_size": 3, "dist": {"hi": 9, "kind": "uniform", "lo": 0}, "max_uih": 9,
            "num_iterations": 2, "num_ranks": 2, "seed": 1, "table_rows": 100, "target_collision": None}
    its = [[[(rng.integers(0, 2 ** 63, rng.integers(0, 10), dtype=np.uint64),
              [rng.integers(0, 99, 3, dtype=np.uint64)], float(rng.random())) for _ in range(3)]
            for _ in range(2)] for _ in range(2)]
    p = str(tmp_path / "py.bin")
    W.save_workload(p, spec, its)
    d = reference.load_workload(p)
    flat = [s for it in its for b in it for s in b]
    assert np.array_equal(d["lens"], [len(s[0]) for s in flat])
    assert np.array_equal(d["ids"], np.concatenate([s[0] for s in flat]))
    assert np.array_equal(d["labels"], [s[2] for s in flat])
