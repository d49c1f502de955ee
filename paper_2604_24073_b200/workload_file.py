"""Workload-file replay onto the GPU.

Reads the reference's binary workload stream — 8-byte magic ``FSCLWKL1``, u32
header length, JSON WorkloadSpec header, then per (iteration, rank) a u32
sample count and one u32-length-prefixed record per sample
(include/freescale/workload.hpp:111-144, src/workload.cpp:391-418, 478-549) —
and hands the engine what it consumes: per rank the batch-major UIH ids as a
device JaggedTensor (one segment per sample, ``Batch::uih_ids``,
workload.hpp:31-32) plus the labels, resident in HBM.

Same names, argument meaning and exceptions as the reference's Reader
(``spec()``, ``has_next()``, ``next_iteration()``; IoError / ProtocolError with
the reference's texts). The file is memory-mapped; each iteration is one pinned
host → device copy of its raw bytes. The host walks only the length prefixes
(``fsx_workload_scan``, C++ in libfsx); records are parsed and validated and
the ids moved by libfsx kernels (``fsx_workload_decode``). Candidates stay in
the raw bytes (the embedding path does not consume them); ``Writer`` /
``save_workload`` write the same format (workload.cpp:441-476, 551-557).
"""
from __future__ import annotations

import ctypes as C
import json
import mmap
import os
import struct

import numpy as np
import torch

from . import _lib
from .errors import InvalidArgument, IoError, ProtocolError
from .jagged import JaggedTensor, _ctx, _stream

MAGIC = b"FSCLWKL1"  # workload.cpp:328


class DeviceBatch:
    """One rank's share of an iteration on the device (the parts of
    workload::Batch the embedding path reads, workload.hpp:25-35)."""

    def __init__(self, rank: int, uih: JaggedTensor, labels: torch.Tensor):
        self.rank = rank
        self.uih = uih          # JaggedTensor of u64 ids (int64 bits), one segment per sample
        self.labels = labels    # f64 [samples] on the device

    def num_samples(self) -> int:
        return self.uih.num_segments()

    def uih_ids(self) -> JaggedTensor:
        return self.uih

    def total_uih_tokens(self) -> int:
        return self.uih.total_values()

    def max_uih_len(self) -> int:
        ln = self.uih.lengths()
        return int(ln.max()) if ln.size else 0


class Reader:
    """workload::Reader (workload.hpp:129-140, workload.cpp:478-549)."""

    def __init__(self, path: str, device=None):
        self.path = path
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        try:
            self._f = open(path, "rb")
        except OSError:
            raise IoError(f"workload: cannot open '{path}'") from None
        size = os.fstat(self._f.fileno()).st_size
        self._mm = mmap.mmap(self._f.fileno(), 0, access=mmap.ACCESS_READ) if size else b""
        self._buf = np.frombuffer(self._mm, dtype=np.uint8) if size else np.zeros(0, np.uint8)
        if size < 8 or bytes(self._buf[:8]) != MAGIC:
            raise IoError(f"workload: bad magic in '{path}'")
        if size < 12:
            raise IoError("workload: truncated header length")
        (hlen,) = struct.unpack_from("<I", self._mm, 8)
        if 12 + hlen > size:
            raise IoError("workload: truncated header")
        try:
            self._spec = json.loads(bytes(self._buf[12:12 + hlen]).decode())
            self._ranks = int(self._spec["num_ranks"])
            self._iters = int(self._spec["num_iterations"])
        except (ValueError, KeyError, TypeError) as e:
            raise IoError(f"workload: malformed header: {e}") from None
        self._pos = 12 + hlen
        self._iteration = 0
        self._pinned = None

    def spec(self) -> dict:
        return dict(self._spec)

    def has_next(self) -> bool:
        return self._iteration < self._iters

    def next_iteration(self) -> list:
        """One DeviceBatch per rank (workload.cpp:500-549)."""
        if not self.has_next():
            raise ProtocolError("workload: no more iterations in file")
        view = self._buf[self._pos:]
        nbytes = int(view.size)
        # every record carries at least its u32 length prefix (a short or empty
        # record must reach the decode's IoError, not a capacity error)
        cap = nbytes // 4 + 1
        rec_off = np.empty(cap, np.uint64)
        per_rank = np.zeros(self._ranks, np.uint64)
        n, used = C.c_uint64(), C.c_uint64()
        _lib.call("fsx_workload_scan", C.c_void_p(view.ctypes.data if nbytes else 0), nbytes, self._ranks,
                  self._iteration, per_rank.ctypes.data_as(C.c_void_p), rec_off.ctypes.data_as(C.c_void_p), cap,
                  C.byref(n), C.byref(used))
        n, used = int(n.value), int(used.value)
        dev = self.device
        # one pinned H2D of the iteration's raw bytes (padded to 8 for the u64 id loads)
        padded = (used + 7) & ~7
        if self._pinned is None or self._pinned.numel() < padded:
            self._pinned = torch.empty(max(padded, 1 << 20), dtype=torch.uint8, pin_memory=True)
            self._pinned_np = self._pinned.numpy()
        np.copyto(self._pinned_np[:used], view[:used])
        d_bytes = torch.empty(max(padded, 8), dtype=torch.uint8, device=dev)
        d_bytes[:used].copy_(self._pinned[:used], non_blocking=True)
        d_off = torch.from_numpy(rec_off[:n].view(np.int64)).to(dev, non_blocking=False)
        d_len = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
        d_offs = torch.empty(n + 1, dtype=torch.int64, device=dev)
        d_lab = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
        id_cap = used // 8
        d_vals = torch.empty(max(id_cap, 1), dtype=torch.int64, device=dev)
        tot = C.c_uint64()
        _lib.call("fsx_workload_decode", _ctx(dev).h, C.c_void_p(d_bytes.data_ptr()), used,
                  C.c_void_p(d_off.data_ptr()), n, self._iteration, per_rank.ctypes.data_as(C.c_void_p),
                  self._ranks, C.c_void_p(d_len.data_ptr()), C.c_void_p(d_offs.data_ptr()),
                  C.c_void_p(d_lab.data_ptr()), C.c_void_p(d_vals.data_ptr()), id_cap, C.byref(tot),
                  C.c_void_p(_stream(dev)))
        lens = d_len[:n].cpu().numpy().view(np.uint64)
        offs = np.concatenate([[0], np.cumsum(lens, dtype=np.uint64)]).astype(np.uint64)
        out, s0 = [], 0
        for r in range(self._ranks):
            s1 = s0 + int(per_rank[r])
            vals = d_vals[int(offs[s0]):int(offs[s1])]
            out.append(DeviceBatch(r, JaggedTensor(vals, lens[s0:s1], device=dev), d_lab[s0:s1]))
            s0 = s1
        self._pos += used
        self._iteration += 1
        return out

    def close(self) -> None:
        self._buf = None
        if isinstance(self._mm, mmap.mmap):
            self._mm.close()
        self._f.close()


def load_workload(path: str, device=None):
    """workload::load_workload (workload.cpp:559-564): (spec, [iteration][rank] DeviceBatch)."""
    r = Reader(path, device)
    its = []
    while r.has_next():
        its.append(r.next_iteration())
    return r.spec(), its


# ---- writing (host side; the format's producer) -----------------------------

def encode_sample(uih, candidates=(), label: float = 0.0) -> bytes:
    """encode_sample (workload.cpp:391-403)."""
    uih = np.asarray(uih, dtype="<u8").reshape(-1)
    parts = [struct.pack("<I", uih.size), uih.tobytes(), struct.pack("<I", len(candidates))]
    for c in candidates:
        c = np.asarray(c, dtype="<u8").reshape(-1)
        parts += [struct.pack("<I", c.size), c.tobytes()]
    parts.append(struct.pack("<d", float(label)))
    return b"".join(parts)


class Writer:
    """workload::Writer (workload.cpp:441-476). An iteration is a list of one
    batch per rank; a batch is a list of (uih, candidates, label) samples."""

    def __init__(self, path: str, spec: dict):
        self.spec = dict(spec)
        self._closed = False
        try:
            self._f = open(path, "wb")
        except OSError:
            raise IoError(f"workload: cannot open '{path}' for writing") from None
        header = json.dumps(self.spec, separators=(",", ":"), sort_keys=True).encode()
        self._f.write(MAGIC + struct.pack("<I", len(header)) + header)

    def write_iteration(self, batches) -> None:
        if self._closed:
            raise IoError("workload: writer already closed")
        if len(batches) != int(self.spec["num_ranks"]):
            raise InvalidArgument("workload: iteration must carry one batch per rank")
        for b in batches:
            buf = [struct.pack("<I", len(b))]
            for s in b:
                rec = encode_sample(*s)
                buf += [struct.pack("<I", len(rec)), rec]
            self._f.write(b"".join(buf))

    def close(self) -> None:
        if not self._closed:
            self._f.close()
            self._closed = True


def save_workload(path: str, spec: dict, iterations) -> None:
    """save_workload (workload.cpp:551-557)."""
    s = dict(spec)
    s["num_iterations"] = len(iterations)
    w = Writer(path, s)
    for it in iterations:
        w.write_iteration(it)
    w.close()
