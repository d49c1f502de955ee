"""Workload-file replay on the GPU: files written by the
reference's Writer (tests/golden/workload_*.bin) replayed through libfsx
(fsx_workload_scan + fsx_workload_decode) must give exactly the uih ids,
lengths, labels and per-rank sample counts the reference's Reader returned
(tests/golden/workload_*.npz; make_workload_golden.py), with the reference's
IoError / ProtocolError texts on malformed files. At config-2 scale (8 ranks x
8,192 power-law samples) the Python Writer → GPU Reader round trip is checked
sample for sample."""
import os
import struct

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _flatten(its):
    ids, lens, labels, counts = [], [], [], []
    for it in its:
        for b in it:
            counts.append(b.num_samples())
            lens.append(b.uih.lengths())
            ids.append(b.uih.values().cpu().numpy().view(np.uint64))
            labels.append(b.labels.cpu().numpy())
    cat = lambda xs, dt: np.concatenate(xs).astype(dt) if xs else np.zeros(0, dt)  # noqa: E731
    return cat(ids, np.uint64), cat(lens, np.uint64), cat(labels, np.float64), np.asarray(counts, np.uint64)


@pytest.mark.parametrize("name", ["small_2r", "ragged_4r", "single_1r"])
def test_replay_matches_reference_reader(name, cuda):
    from paper_2604_24073_b200 import workload_file as W
    g = np.load(os.path.join(GOLD, f"workload_{name}.npz"))
    spec, its = W.load_workload(os.path.join(GOLD, f"workload_{name}.bin"), cuda)
    assert spec["num_ranks"] == int(g["ranks"]) and len(its) == int(g["iterations"])
    ids, lens, labels, counts = _flatten(its)
    assert np.array_equal(ids, g["ids"])
    assert np.array_equal(lens, g["lens"])
    assert np.array_equal(labels.view(np.uint64), g["labels"].view(np.uint64))  # bit-exact f64
    assert np.array_equal(counts, g["counts"])
    for it in its:
        for b in it:  # device offsets agree with the host lengths
            offs = b.uih.device_offsets().cpu().numpy().view(np.uint64)
            assert np.array_equal(offs, b.uih.offsets())


def test_reader_errors(cuda, tmp_path):
    from paper_2604_24073_b200 import workload_file as W
    from paper_2604_24073_b200.errors import IoError, ProtocolError
    raw = open(os.path.join(GOLD, "workload_small_2r.bin"), "rb").read()
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"NOTMAGIC" + raw[8:])
    with pytest.raises(IoError, match="bad magic"):
        W.Reader(str(bad), cuda)
    with pytest.raises(IoError, match="cannot open"):
        W.Reader(str(tmp_path / "missing.bin"), cuda)
    cut = tmp_path / "cut.bin"
    cut.write_bytes(raw[:2000])  # reference: iteration 0, rank 1, sample 1
    r = W.Reader(str(cut), cuda)
    with pytest.raises(IoError, match=r"^workload: file truncated; last complete record is iteration 0, rank 1, sample 1$"):
        r.next_iteration()
    r = W.Reader(os.path.join(GOLD, "workload_single_1r.bin"), cuda)
    r.next_iteration()
    with pytest.raises(ProtocolError, match="no more iterations"):
        r.next_iteration()


def test_trailing_bytes_in_record(cuda, tmp_path):
    from paper_2604_24073_b200 import workload_file as W
    from paper_2604_24073_b200.errors import IoError
    spec = {"batch_size": 2, "dist": {"hi": 4, "kind": "uniform", "lo": 0}, "max_uih": 4,
            "num_iterations": 1, "num_ranks": 2, "seed": 1, "table_rows": 10, "target_collision": None}
    p = tmp_path / "trail.bin"
    w = W.Writer(str(p), spec)
    w.close()
    recs = [W.encode_sample([1, 2], [[3]], 0.5), W.encode_sample([4], [], 0.25),
            W.encode_sample([5], [], 0.75) + b"\0\0\0\0", W.encode_sample([], [], 1.0)]
    with open(p, "ab") as f:
        for r in range(2):
            f.write(struct.pack("<I", 2))
            for rec in recs[2 * r:2 * r + 2]:
                f.write(struct.pack("<I", len(rec)) + rec)
    with pytest.raises(IoError, match=r"^workload: record has trailing bytes at iteration 0, rank 1, sample 0$"):
        W.Reader(str(p), cuda).next_iteration()


def test_cfg2_scale_round_trip(cuda, tmp_path):
    """8 ranks x 8,192 samples, power-law UIH lengths 16..8192 (config 2's
    shape): every id, length and label survives Writer → GPU Reader."""
    from paper_2604_24073_b200 import workload as G, workload_file as W
    ranks, per = 8, 8192
    lens = G.uih_lengths(20261020, ranks * per).astype(np.int64)
    rng = np.random.default_rng(3)
    ids = rng.integers(0, 2 ** 63, int(lens.sum()), dtype=np.uint64)
    labels = rng.random(ranks * per)
    offs = np.concatenate([[0], np.cumsum(lens)])
    samples = [(ids[offs[s]:offs[s + 1]], [], labels[s]) for s in range(ranks * per)]
    spec = {"batch_size": per, "dist": {"kind": "empirical", "histogram": []}, "max_uih": 8192,
            "num_iterations": 1, "num_ranks": ranks, "seed": 1, "table_rows": 2 ** 63, "target_collision": None}
    p = str(tmp_path / "cfg2.bin")
    W.save_workload(p, spec, [[samples[r * per:(r + 1) * per] for r in range(ranks)]])
    _, its = W.load_workload(p, cuda)
    got_ids, got_lens, got_labels, counts = _flatten(its)
    assert np.array_equal(counts, [per] * ranks)
    assert np.array_equal(got_lens, lens.astype(np.uint64))
    assert np.array_equal(got_ids, ids)
    assert np.array_equal(got_labels, labels)


def _write_records(p, W, per_rank_recs, truncate=0):
    spec = {"batch_size": 2, "dist": {"hi": 4, "kind": "uniform", "lo": 0}, "max_uih": 4,
            "num_iterations": 1, "num_ranks": len(per_rank_recs), "seed": 1, "table_rows": 10,
            "target_collision": None}
    w = W.Writer(str(p), spec)
    w.close()
    body = b""
    for recs in per_rank_recs:
        body += struct.pack("<I", len(recs))
        for rec in recs:
            body += struct.pack("<I", len(rec)) + rec
    with open(p, "ab") as f:
        f.write(body[:len(body) - truncate])


def test_misaligned_record_is_an_io_error_not_a_fault(cuda, tmp_path):
    """A record whose length is not a multiple of 4 (1 trailing byte) shifts
    every later record off 4-byte alignment. The reference raises its
    trailing-bytes IoError at that record; the GPU decode must do the same
    (no misaligned-address fault poisoning the context) and stay usable."""
    from paper_2604_24073_b200 import workload_file as W
    from paper_2604_24073_b200.errors import IoError
    good = [W.encode_sample([1, 2], [[3]], 0.5), W.encode_sample([4], [], 0.25)]
    p = tmp_path / "misaligned.bin"
    _write_records(p, W, [[good[0], W.encode_sample([5], [], 0.75) + b"\0"], [good[1], good[0]]])
    with pytest.raises(IoError, match=r"^workload: record has trailing bytes at iteration 0, rank 0, sample 1$"):
        W.Reader(str(p), cuda).next_iteration()
    # the context is intact: a good file decodes afterwards
    q = tmp_path / "good.bin"
    _write_records(q, W, [good, good])
    out = W.Reader(str(q), cuda).next_iteration()
    assert len(out) == 2


def test_first_bad_record_in_file_order_wins(cuda, tmp_path):
    """Several malformed records: the reference decodes in file order and
    names the first; a malformed record also beats a later file truncation."""
    from paper_2604_24073_b200 import workload_file as W
    from paper_2604_24073_b200.errors import IoError
    ok = W.encode_sample([1], [], 0.5)
    trail = W.encode_sample([2], [], 0.5) + b"\0\0\0\0"
    recs = [[ok] * 40 + [trail] + [ok] * 300 + [trail], [ok] * 5 + [trail]]
    p = tmp_path / "multi.bin"
    _write_records(p, W, recs)
    with pytest.raises(IoError, match=r"^workload: record has trailing bytes at iteration 0, rank 0, sample 40$"):
        W.Reader(str(p), cuda).next_iteration()
    q = tmp_path / "trail_then_cut.bin"
    _write_records(q, W, [[ok, trail, ok], [ok, ok]], truncate=3)
    with pytest.raises(IoError, match=r"^workload: record has trailing bytes at iteration 0, rank 0, sample 1$"):
        W.Reader(str(q), cuda).next_iteration()


def test_empty_records_reach_the_decode_error(cuda, tmp_path):
    """Many zero-length records: the record table must hold them all, so the
    decode reports the reference's 'record truncated', not a capacity error."""
    from paper_2604_24073_b200 import workload_file as W
    from paper_2604_24073_b200.errors import IoError
    p = tmp_path / "empty.bin"
    _write_records(p, W, [[b""] * 64, [b""] * 64])
    with pytest.raises(IoError, match=r"^workload: record truncated$"):
        W.Reader(str(p), cuda).next_iteration()
