"""Jagged tensors on the GPU (include/freescale/jagged.hpp).

Mirror of the reference's JaggedTensor / KeyedJaggedTensor and its reshuffle
ops with the same names, argument meaning and exceptions. Values live on the
device (a 1-D torch tensor of any 1/2/4/8/16-byte dtype); lengths are kept on
the host as well (the reference's constructor validates them there), offsets
on the device come from fsx_jagged_offsets. Segment moves run on libfsx
kernels: indexed_permute / keyed_transpose through fsx_jagged_permute and
fsx_keyed_transpose_perm, ranged_dispatch / ranged_combine as contiguous device
slices / concatenations (jagged.hpp:120-199 moves whole ranges).
"""
from __future__ import annotations

import ctypes as C
import enum
import threading

import numpy as np
import torch

from . import _lib
from .errors import InvalidArgument, OutOfRange

def _stream(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _ctx(device: torch.device):
    """One libfsx context per device for the jagged ops, created once under a
    lock (a context that lost a creation race would be destroyed while a
    caller still holds its handle)."""
    from .embedding import Context
    idx = device.index if device.index is not None else torch.cuda.current_device()
    with _CTX_LOCK:
        c = _CTX.get(idx)
        if c is None:
            c = _CTX[idx] = Context(idx, 0, 1)
    return c


_CTX: dict = {}
_CTX_LOCK = threading.Lock()


class JaggedTensor:
    """jagged.hpp:18-80. `values`: 1-D device tensor (or array-like: moved to
    cuda:0 as u64/i64 bits); `lengths`: per-segment counts."""

    def __init__(self, values=None, lengths=None, device=None):
        if values is None:
            values, lengths = np.zeros(0, np.uint64), []
        if not isinstance(values, torch.Tensor):
            a = np.ascontiguousarray(np.asarray(values))
            if a.dtype == np.uint64:
                a = a.view(np.int64)
            values = torch.from_numpy(a.reshape(-1).copy())
        dev = torch.device(device) if device is not None else (
            values.device if values.is_cuda else torch.device("cuda", torch.cuda.current_device()))
        self._v = values.reshape(-1).to(dev).contiguous()
        self._len = np.asarray(lengths if lengths is not None else [], dtype=np.uint64).reshape(-1)
        tot = int(self._len.sum()) if self._len.size else 0
        if tot != self._v.numel():
            raise InvalidArgument(f"jagged: sum(lengths)={tot} does not match len(values)={self._v.numel()}")
        self._offs = np.concatenate([[0], np.cumsum(self._len, dtype=np.uint64)]).astype(np.uint64)
        self._d_offs = None

    @staticmethod
    def from_segments(segments, dtype=np.uint64, device=None) -> "JaggedTensor":
        vals = [np.asarray(s, dtype=dtype).reshape(-1) for s in segments]
        flat = np.concatenate(vals) if vals else np.zeros(0, dtype)
        return JaggedTensor(flat, [v.size for v in vals], device=device)

    # ---- accessors (jagged.hpp:45-78)
    def num_segments(self) -> int:
        return int(self._len.size)

    def total_values(self) -> int:
        return int(self._v.numel())

    def length(self, k: int) -> int:
        self._check(k)
        return int(self._len[k])

    def offset(self, k: int) -> int:
        if not 0 <= k <= self.num_segments():
            raise OutOfRange(f"jagged: offset index {k} out of range")
        return int(self._offs[k])

    def _check(self, k: int) -> None:
        if not 0 <= k < self.num_segments():
            raise OutOfRange(f"jagged: segment index {k} out of range (have {self.num_segments()})")

    def segment(self, k: int) -> torch.Tensor:
        self._check(k)
        return self._v[int(self._offs[k]):int(self._offs[k + 1])]

    def values(self) -> torch.Tensor:
        return self._v

    def lengths(self) -> np.ndarray:
        return self._len.copy()

    def offsets(self) -> np.ndarray:
        return self._offs.copy()

    def device_offsets(self) -> torch.Tensor:
        """u64 [n+1] on the device, computed by the libfsx scan (fsx_jagged_offsets)."""
        if self._d_offs is None:
            dev = self._v.device
            d_len = torch.from_numpy(self._len.view(np.int64).copy()).to(dev)
            d_offs = torch.empty(self.num_segments() + 1, dtype=torch.int64, device=dev)
            tot = C.c_uint64()
            _lib.call("fsx_jagged_offsets", _ctx(dev).h, C.c_void_p(d_len.data_ptr()), self.num_segments(),
                      C.c_void_p(d_offs.data_ptr()), C.byref(tot), C.c_void_p(_stream(dev)))
            self._d_offs = d_offs
        return self._d_offs

    def to_segments(self) -> list:
        host = self._v.cpu().numpy()
        if host.dtype == np.int64:
            host = host.view(np.uint64)
        return [host[int(self._offs[k]):int(self._offs[k + 1])].tolist() for k in range(self.num_segments())]

    def __eq__(self, o) -> bool:
        return (isinstance(o, JaggedTensor) and np.array_equal(self._len, o._len)
                and self._v.dtype == o._v.dtype and torch.equal(self._v.cpu(), o._v.cpu()))

    def __repr__(self) -> str:
        return f"JaggedTensor(segments={self.num_segments()}, values={self.total_values()})"


IdJagged = JaggedTensor
ValueJagged = JaggedTensor


def indexed_permute(t: JaggedTensor, perm) -> JaggedTensor:
    """jagged.hpp:89-111: segment j of the result is segment perm[j] of t
    (repetition allowed); out_of_range names the bad index."""
    dev = t.values().device
    if isinstance(perm, torch.Tensor) and perm.is_cuda:
        d_perm = perm.reshape(-1).to(device=dev, dtype=torch.int64).contiguous()
    else:
        p = np.asarray(perm, dtype=np.uint64).reshape(-1)
        d_perm = torch.from_numpy(p.view(np.int64).copy()).to(dev)
    n = d_perm.numel()
    d_len = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    d_offs = torch.empty(n + 1, dtype=torch.int64, device=dev)
    tot = C.c_uint64()
    ctx, s = _ctx(dev).h, _stream(dev)
    args = (C.c_void_p(t.values().data_ptr()), t.values().element_size(),
            C.c_void_p(t.device_offsets().data_ptr()), t.num_segments(), C.c_void_p(d_perm.data_ptr()), n)
    _lib.call("fsx_jagged_permute", ctx, *args, None, 0, C.c_void_p(d_len.data_ptr()),
              C.c_void_p(d_offs.data_ptr()), C.byref(tot), C.c_void_p(s))
    out = torch.empty(max(tot.value, 1), dtype=t.values().dtype, device=dev)
    _lib.call("fsx_jagged_permute", ctx, *args, C.c_void_p(out.data_ptr()), tot.value,
              C.c_void_p(d_len.data_ptr()), C.c_void_p(d_offs.data_ptr()), C.byref(tot), C.c_void_p(s))
    lengths = d_len[:n].cpu().numpy().view(np.uint64)
    r = JaggedTensor(out[:tot.value], lengths, device=dev)
    r._d_offs = d_offs
    return r


class SegmentRange:
    """jagged.hpp:113-116"""

    def __init__(self, start: int = 0, count: int = 0):
        self.start, self.count = int(start), int(count)


def _ranges(ranges) -> list:
    return [r if isinstance(r, SegmentRange) else SegmentRange(*r) for r in ranges]


def ranged_dispatch(t: JaggedTensor, ranges) -> list:
    """jagged.hpp:118-155: one part per range, each a contiguous run of t's
    segments; out_of_range for a range past the end, invalid_argument for
    overlapping non-empty ranges."""
    rs = _ranges(ranges)
    for d, r in enumerate(rs):
        if r.start + r.count > t.num_segments():
            raise OutOfRange(f"ranged_dispatch: range {d} = ({r.start},{r.count}) exceeds segment count "
                             f"{t.num_segments()}")
    spans = sorted((r.start, r.start + r.count) for r in rs if r.count > 0)
    for i in range(1, len(spans)):
        if spans[i][0] < spans[i - 1][1]:
            raise InvalidArgument(f"ranged_dispatch: overlapping ranges at segment {spans[i][0]}")
    offs, lens = t.offsets(), t.lengths()
    out = []
    for r in rs:
        b = int(offs[r.start]) if r.start <= t.num_segments() else 0
        e = int(offs[r.start + r.count])
        out.append(JaggedTensor(t.values()[b:e].clone(), lens[r.start:r.start + r.count], device=t.values().device))
    return out


def ranged_combine(parts) -> JaggedTensor:
    """jagged.hpp:157-176: concatenation of the parts' segments in order."""
    parts = list(parts)
    if not parts:
        return JaggedTensor()
    dev = parts[0].values().device
    vals = torch.cat([p.values().to(dev) for p in parts]) if parts else None
    lens = np.concatenate([p.lengths() for p in parts]) if parts else np.zeros(0, np.uint64)
    return JaggedTensor(vals, lens, device=dev)


class KeyedLayout(enum.Enum):
    FeatureMajor = 0
    BatchMajor = 1


class KeyedJaggedTensor:
    """jagged.hpp:196-225: segments of (feature, sample) in one of two orders."""

    def __init__(self, keys, inner: JaggedTensor, layout: KeyedLayout = KeyedLayout.FeatureMajor):
        self.keys = list(keys)
        self.inner = inner
        self.layout = layout
        if not self.keys:
            raise InvalidArgument("keyed jagged: no keys")
        if inner.num_segments() % len(self.keys) != 0:
            raise InvalidArgument(f"keyed jagged: segment count {inner.num_segments()} not divisible by key "
                                  f"count {len(self.keys)}")
        self.num_samples = inner.num_segments() // len(self.keys)

    def at(self, f: int, s: int) -> torch.Tensor:
        F, S = len(self.keys), self.num_samples
        return self.inner.segment(f * S + s if self.layout == KeyedLayout.FeatureMajor else s * F + f)

    def __eq__(self, o) -> bool:
        return (isinstance(o, KeyedJaggedTensor) and self.keys == o.keys and self.layout == o.layout
                and self.num_samples == o.num_samples and self.inner == o.inner)


def keyed_transpose(kt: KeyedJaggedTensor) -> KeyedJaggedTensor:
    """jagged.hpp:227-248: flip feature-major <-> batch-major; the (f, s)
    segment is unchanged. The permutation is built on the device."""
    dev = kt.inner.values().device
    F, S = len(kt.keys), kt.num_samples
    d_perm = torch.empty(max(F * S, 1), dtype=torch.int64, device=dev)
    _lib.call("fsx_keyed_transpose_perm", _ctx(dev).h, F, S, int(kt.layout == KeyedLayout.FeatureMajor),
              C.c_void_p(d_perm.data_ptr()), C.c_void_p(_stream(dev)))
    out = KeyedJaggedTensor.__new__(KeyedJaggedTensor)
    out.keys = list(kt.keys)
    out.inner = indexed_permute(kt.inner, d_perm[:F * S])
    out.layout = KeyedLayout.BatchMajor if kt.layout == KeyedLayout.FeatureMajor else KeyedLayout.FeatureMajor
    out.num_samples = S
    return out
