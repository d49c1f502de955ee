"""C++ drop-in workload.hpp (cpp/src/workload_b200.cpp) against the
reference's own generator and file codec (proj/src/workload.cpp), on the host:
generate_all gives the reference's samples bit for bit (uniform lengths, with
and without the collision-control pool), save_workload writes the reference's
bytes, and load_workload reads the reference's files back."""
import os
import subprocess
import tempfile

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CPP = os.path.join(ROOT, "paper_2604_24073_b200", "cpp")
TOOL = os.path.join(CPP, "build", "workload_tool")

CASES = [
    dict(world=2, batch=4, max_uih=64, lo=0, hi=12, table_rows=5000, target=None, seed=7, iters=3),
    dict(world=3, batch=5, max_uih=10, lo=1, hi=40, table_rows=100000, target=0.3, seed=11, iters=4),
    dict(world=1, batch=8, max_uih=32, lo=16, hi=16, table_rows=1 << 16, target=0.0, seed=3, iters=2),
    dict(world=4, batch=2, max_uih=8, lo=0, hi=8, table_rows=64, target=1.0, seed=5, iters=3),
]


@pytest.fixture(scope="module")
def tool():
    if not os.path.exists(os.path.join(ROOT, "paper_2604_24073_b200", "libfsx.so")):
        pytest.skip("libfsx.so not built")
    r = subprocess.run(["make", "-s", "-C", CPP, "build/workload_tool"], capture_output=True, text=True)
    if r.returncode != 0:
        pytest.fail(r.stdout + r.stderr)
    return TOOL


def _flat(path):
    raw = np.fromfile(path, np.uint64)
    ns, ni, nc, nci = (int(x) for x in raw[:4])
    at = 4
    out = {}
    for k, n in (("uih_len", ns), ("n_cand", ns), ("label", ns), ("ids", ni), ("cand_len", nc), ("cand_ids", nci)):
        out[k] = raw[at:at + n]
        at += n
    out["label"] = out["label"].view(np.float64)
    return out


def _gen(tool, spec, path):
    t = -1.0 if spec["target"] is None else spec["target"]
    args = [tool, "gen"] + [str(spec[k]) for k in ("world", "batch", "max_uih", "lo", "hi", "table_rows")] + \
           [repr(float(t)), str(spec["seed"]), str(spec["iters"]), path]
    r = subprocess.run(args, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return _flat(path + ".flat")


@pytest.mark.parametrize("k", range(len(CASES)))
def test_generator_matches_reference(tool, reference, k):
    spec = CASES[k]
    want = reference.pipeline_samples(spec)
    with tempfile.TemporaryDirectory() as d:
        got = _gen(tool, spec, os.path.join(d, "w.bin"))
    for key in want:
        assert np.array_equal(np.asarray(got[key]).view(np.uint64), np.asarray(want[key]).view(np.uint64)), key


def test_file_bytes_and_reader_match_reference(tool, reference):
    spec = dict(world=2, batch=3, max_uih=20, lo=0, hi=20, table_rows=777, target=None, seed=99, iters=3)
    with tempfile.TemporaryDirectory() as d:
        mine, theirs = os.path.join(d, "mine.bin"), os.path.join(d, "ref.bin")
        _gen(tool, spec, mine)
        reference.save_workload_uniform(theirs, spec["world"], spec["batch"], spec["max_uih"], spec["lo"],
                                        spec["hi"], spec["table_rows"], spec["seed"], spec["iters"])
        assert open(mine, "rb").read() == open(theirs, "rb").read()
        r = subprocess.run([tool, "load", theirs], capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
        got = _flat(theirs + ".flat")
        want = reference.pipeline_samples(spec)
        for key in want:
            assert np.array_equal(np.asarray(got[key]).view(np.uint64), np.asarray(want[key]).view(np.uint64)), key


def test_reader_errors_match_reference_texts(tool, reference):
    spec = dict(world=2, batch=3, max_uih=20, lo=1, hi=20, table_rows=777, target=None, seed=1, iters=2)
    with tempfile.TemporaryDirectory() as d:
        ref = os.path.join(d, "ref.bin")
        reference.save_workload_uniform(ref, spec["world"], spec["batch"], spec["max_uih"], spec["lo"],
                                        spec["hi"], spec["table_rows"], spec["seed"], spec["iters"])
        data = open(ref, "rb").read()
        cut = os.path.join(d, "cut.bin")
        open(cut, "wb").write(data[:-5])
        r = subprocess.run([tool, "load", cut], capture_output=True, text=True)
        assert r.returncode == 1
        assert "workload: file truncated; last complete record is iteration 1, rank 1, sample 1" in r.stderr
        bad = os.path.join(d, "bad.bin")
        open(bad, "wb").write(b"XXXXXXXX" + data[8:])
        r = subprocess.run([tool, "load", bad], capture_output=True, text=True)
        assert r.returncode == 1 and "workload: bad magic in" in r.stderr


@pytest.mark.parametrize("suite", ["workload", "sim"])
def test_reference_host_suites_unchanged(suite):
    """The reference's test_workload.cpp / test_sim.cpp (host-only code: the
    generator, file codec, statistics, Timeline, metric records, cost model)
    compiled unchanged against the drop-in headers (cpp/Makefile)."""
    exe = os.path.join(CPP, "build", f"ref_test_{suite}")
    if not os.path.exists(exe):
        pytest.skip(f"{exe} not built (needs /root/reference at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and " 0 failed" in r.stdout, r.stdout[-3000:] + r.stderr[-2000:]
