"""Python mirror of the reference embedding API (proj/include/freescale/
embedding.hpp) over libfsx's C ABI. Same names, argument meaning and error
classes as the C++ reference, so the parity tests read like its own tests
(tests/test_embedding.cpp). All computation runs in libfsx's CUDA kernels;
torch is only used for device memory and streams.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .errors import InvalidArgument, ProtocolError

_DTYPES = {"f32": (_lib.FSX_F32, torch.float32), "f64": (_lib.FSX_F64, torch.float64)}


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _stream(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _dev_u64(x, device) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        t = x.to(device=device, dtype=torch.int64)
    else:
        a = np.ascontiguousarray(np.asarray(x, dtype=np.uint64).reshape(-1))
        t = torch.from_numpy(a.view(np.int64)).to(device)
    return t.contiguous()


def _np_u64(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy().view(np.uint64).copy()


@dataclass(frozen=True)
class TableGeometry:
    """embedding.hpp:13-26: row g lives on shard g mod p at local index g div p."""
    total_rows: int = 0
    dim: int = 1
    num_shards: int = 1

    def owner(self, g: int) -> int:
        return int(g % self.num_shards)

    def local_index(self, g: int) -> int:
        return int(g // self.num_shards)

    def local_rows(self, shard: int) -> int:
        return (self.total_rows - 1 - shard) // self.num_shards + 1 if self.total_rows > shard else 0


class Context:
    """One libfsx context (= one rank on one GPU)."""

    def __init__(self, device: int = 0, rank: int = 0, world: int = 1):
        self.device = device
        self.rank = rank
        self.world = world
        h = C.c_void_p()
        _lib.call("fsx_ctx_create", device, rank, world, C.byref(h))
        self.h = h

    @property
    def torch_device(self) -> torch.device:
        return torch.device("cuda", self.device)

    def sync(self) -> None:
        _lib.call("fsx_ctx_sync", self.h)

    def launches(self) -> int:
        return int(_lib.lib().fsx_ctx_launches(self.h))

    def kernel_span(self, on: bool) -> tuple[float, int]:
        """Mean own span (us) and count of the row-update kernel's launches
        since the last call, then switch recording on / off (measurement)."""
        m, n = C.c_double(), C.c_uint64()
        _lib.call("fsx_ctx_kernel_span", self.h, int(on), C.byref(m), C.byref(n))
        return m.value, n.value

    def close(self) -> None:
        if self.h:
            _lib.lib().fsx_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_ctx: dict[int, Context] = {}


def default_context(device: int | None = None) -> Context:
    dev = torch.cuda.current_device() if device is None else device
    if dev not in _default_ctx:
        _default_ctx[dev] = Context(dev)
    return _default_ctx[dev]


@dataclass
class CollisionSplit:
    """embedding.hpp:45-49"""
    collision: np.ndarray
    exclusive_cur: np.ndarray
    exclusive_next: np.ndarray


def sorted_unique(ids, ctx: Context | None = None) -> tuple[np.ndarray, np.ndarray]:
    """sorted_unique (embedding.cpp:12-16) on the device; also each input's slot."""
    ctx = ctx or default_context()
    d = _dev_u64(ids, ctx.torch_device)
    n = d.numel()
    out = torch.empty(max(n, 1), dtype=torch.int64, device=d.device)
    inv = torch.empty(max(n, 1), dtype=torch.int32, device=d.device)
    nu = C.c_uint64()
    _lib.call("fsx_sort_unique_u64", ctx.h, _ptr(d), n, _ptr(out), _ptr(inv), C.byref(nu), _stream())
    return _np_u64(out[:nu.value]), inv[:n].cpu().numpy().astype(np.uint32)


def compute_collision(cur, nxt, ctx: Context | None = None) -> CollisionSplit:
    """compute_collision (embedding.cpp:82-93) on two shard-major id lists."""
    ctx = ctx or default_context()
    a = _dev_u64(cur, ctx.torch_device)
    b = _dev_u64(nxt, ctx.torch_device)
    co = torch.empty(max(a.numel(), 1), dtype=torch.int64, device=a.device)
    exc = torch.empty(max(a.numel(), 1), dtype=torch.int64, device=a.device)
    exn = torch.empty(max(b.numel(), 1), dtype=torch.int64, device=a.device)
    cnt = (C.c_uint64 * 5)()
    _lib.call("fsx_collision_split", ctx.h, _ptr(a), a.numel(), _ptr(b), b.numel(), _ptr(co),
              _ptr(exc), _ptr(exn), cnt, _stream())
    return CollisionSplit(_np_u64(co[:cnt[0]]), _np_u64(exc[:cnt[1]]), _np_u64(exn[:cnt[2]]))


def collision_pct(cur, nxt, ctx: Context | None = None) -> float:
    """collision_pct (embedding.cpp:95-104)."""
    ctx = ctx or default_context()
    a = _dev_u64(cur, ctx.torch_device)
    b = _dev_u64(nxt, ctx.torch_device)
    co = torch.empty(max(a.numel(), 1), dtype=torch.int64, device=a.device)
    exc = torch.empty(max(a.numel(), 1), dtype=torch.int64, device=a.device)
    exn = torch.empty(max(b.numel(), 1), dtype=torch.int64, device=a.device)
    cnt = (C.c_uint64 * 5)()
    _lib.call("fsx_collision_split", ctx.h, _ptr(a), a.numel(), _ptr(b), b.numel(), _ptr(co),
              _ptr(exc), _ptr(exn), cnt, _stream())
    if cnt[4] == 0:
        raise InvalidArgument("collision_pct: next iteration uses no rows")
    return cnt[0] / cnt[4]


def route_by_owner(ids, total_rows: int, num_shards: int, ctx: Context | None = None):
    """Requester half of route_to_shard_major (embedding.cpp:194-204): per owner,
    the ids and their flat positions in original order."""
    ctx = ctx or default_context()
    d = _dev_u64(ids, ctx.torch_device)
    n = d.numel()
    sid = torch.empty(max(n, 1), dtype=torch.int64, device=d.device)
    spos = torch.empty(max(n, 1), dtype=torch.int32, device=d.device)
    cnt = (C.c_uint64 * num_shards)()
    _lib.call("fsx_route_by_owner", ctx.h, _ptr(d), n, total_rows, num_shards, _ptr(sid),
              _ptr(spos), cnt, _stream())
    ids_np, pos_np = _np_u64(sid[:n]), spos[:n].cpu().numpy().astype(np.uint32)
    out, at = [], 0
    for s in range(num_shards):
        k = int(cnt[s])
        out.append((ids_np[at:at + k], pos_np[at:at + k]))
        at += k
    return out


@dataclass
class UpdateResult:
    """ShardView::UpdateResult (embedding.hpp:77-80)."""
    unique_ids: np.ndarray
    rows: torch.Tensor  # |unique_ids| x dim, on the device


class ShardView:
    """One rank's shard (embedding.hpp:59-90), resident in HBM."""

    def __init__(self, geom: TableGeometry, shard_id: int, learning_rate: float, seed: int,
                 dtype: str = "f32", ctx: Context | None = None):
        self.geom = geom
        self.shard_id = shard_id
        self.learning_rate = learning_rate
        self.seed = seed
        self.ctx = ctx or default_context()
        self.dtype_code, self.torch_dtype = _DTYPES[dtype]
        h = C.c_void_p()
        _lib.call("fsx_table_create", self.ctx.h, geom.total_rows, geom.dim, geom.num_shards,
                  shard_id, learning_rate, seed, self.dtype_code, C.byref(h))
        self.h = h

    def geometry(self) -> TableGeometry:
        return self.geom

    def local_rows(self) -> int:
        return int(_lib.lib().fsx_table_local_rows(self.h))

    def values(self) -> np.ndarray:
        """f64 host mirror [local_rows x dim] (lazy D2H)."""
        n = self.local_rows() * self.geom.dim
        out = np.zeros(max(n, 1), np.float64)
        _lib.call("fsx_table_download", self.h, out.ctypes.data)
        return out[:n].reshape(self.local_rows(), self.geom.dim)

    def device_values(self) -> torch.Tensor:
        """Zero-copy view of the shard in HBM."""
        ptr = _lib.lib().fsx_table_values(self.h)
        n = self.local_rows() * self.geom.dim
        return _wrap_device(ptr, n, self.torch_dtype, self.ctx.device).view(self.local_rows(), self.geom.dim)

    def upload(self, values: np.ndarray) -> None:
        v = np.ascontiguousarray(np.asarray(values, np.float64).reshape(-1))
        if v.size != self.local_rows() * self.geom.dim:
            raise InvalidArgument("embedding: upload shape mismatch")
        _lib.call("fsx_table_upload", self.h, v.ctypes.data)

    def row(self, global_id: int) -> np.ndarray:
        return self.lookup([global_id]).double().cpu().numpy()[0]

    def lookup(self, ids) -> torch.Tensor:
        """embedding.cpp:139-146: rows in id order, duplicates duplicated."""
        d = _dev_u64(ids, self.ctx.torch_device)
        out = torch.empty((d.numel(), self.geom.dim), dtype=self.torch_dtype, device=d.device)
        if d.numel():
            _lib.call("fsx_table_gather", self.h, _ptr(d), d.numel(), _ptr(out), _stream(), 1)
        return out

    def apply_gradients(self, ids, grads) -> UpdateResult:
        """embedding.cpp:148-181."""
        d = _dev_u64(ids, self.ctx.torch_device)
        g = grads if isinstance(grads, torch.Tensor) else torch.as_tensor(np.asarray(grads, np.float64))
        g = g.to(device=d.device, dtype=self.torch_dtype).contiguous().reshape(-1)
        dim = self.geom.dim
        if g.numel() != d.numel() * dim:
            raise InvalidArgument(f"embedding: gradient shape {g.numel()} misaligned with "
                                  f"{d.numel()} ids x dim {dim}")
        n = d.numel()
        uq = torch.empty(max(n, 1), dtype=torch.int64, device=d.device)
        rows = torch.empty((max(n, 1), dim), dtype=self.torch_dtype, device=d.device)
        nu = C.c_uint64()
        _lib.call("fsx_table_sgd_update", self.h, _ptr(d), n, _ptr(g), _ptr(uq), _ptr(rows),
                  C.byref(nu), _stream())
        return UpdateResult(_np_u64(uq[:nu.value]), rows[:nu.value])

    def close(self) -> None:
        if getattr(self, "h", None):
            _lib.lib().fsx_table_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _wrap_device(ptr: int, n: int, dtype: torch.dtype, device: int) -> torch.Tensor:
    """A torch view of libfsx-owned device memory (no copy, no ownership)."""

    class _CAI:
        def __init__(self):
            typestr = {torch.float32: "<f4", torch.float64: "<f8", torch.int64: "<i8",
                       torch.int32: "<i4", torch.uint8: "|u1"}[dtype]
            self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr,
                                             "data": (ptr, False), "version": 2}

    with torch.cuda.device(device):
        return torch.as_tensor(_CAI(), device=torch.device("cuda", device))


# ---- engines (embedding.hpp:126-189) -------------------------------------------
@dataclass
class IterationStats:
    """embedding.hpp:119-124 (blocking_bytes in the reference's 8-byte-value
    accounting, whatever the table dtype)."""
    collision_rows: int = 0
    unique_next_rows: int = 0
    blocking_bytes: int = 0

    @property
    def collision_fraction(self) -> float:
        return self.collision_rows / self.unique_next_rows if self.unique_next_rows else 0.0


class _Engine:
    _mode = _lib.FSX_MODE_SYNC

    def __init__(self, shard: ShardView, comm=None, max_occurrences: int = 1 << 16,
                 reduce_chunk: int = 0, transport: str = "ce", presum: bool = False):
        from .comm import DeviceFabric
        self.shard = shard
        if comm is None:
            comm = DeviceFabric(1, [shard.ctx.device]).communicator(0)
        self.comm = comm
        if comm.world_size() != shard.geom.num_shards or comm.rank() != shard.shard_id:
            raise InvalidArgument("embedding: shard geometry does not match the communicator")
        tr = {"ce": _lib.FSX_TRANSPORT_CE, "nccl": _lib.FSX_TRANSPORT_NCCL}[transport]
        cfg = _lib.EngineConfig(self._mode, tr, max_occurrences, reduce_chunk,
                                _lib.FSX_ENGINE_PRESUM if presum else 0)
        h = C.c_void_p()
        _lib.call("fsx_engine_create", shard.ctx.h, shard.h, C.byref(cfg), C.byref(h))
        self.h = h
        self.transport = transport
        self.max_occurrences = max_occurrences
        self._n_cur = None
        if transport == "nccl":
            comm.connect_nccl(h)
        else:
            comm.connect(h)

    def _ids(self, ids) -> torch.Tensor:
        return _dev_u64(ids, self.shard.ctx.torch_device)

    def set_ids_ready(self, ready: bool = True) -> None:
        """Device id tensors passed to forward are complete when passed."""
        _lib.call("fsx_engine_set_ids_ready", self.h, int(ready))

    def set_eco_direct(self, on, cog: bool = False) -> None:
        """Collision chain transfers by direct NVLink stores from the compute
        kernels (SM-issued) instead of the copy engines: E_co from the
        collision update (`on`), and with `cog` (PRESUM) the collision
        gradients from the pre-sum; between iterations, on every rank."""
        _lib.call("fsx_engine_set_eco_direct", self.h, (1 if on else 0) | (2 if cog else 0))

    def join(self, stream=None) -> None:
        """Order every lane's issued work before `stream` (timing regions)."""
        _lib.call("fsx_engine_join", self.h, _stream(stream))

    def set_profiling(self, on: bool = True) -> None:
        _lib.call("fsx_engine_set_profiling", self.h, int(on))

    def phase_ms(self) -> dict:
        """{phase: (total ms, spans)} since the last call (synchronizes)."""
        out = {}
        for k, name in enumerate(_lib.PHASES):
            t, n = C.c_double(), C.c_uint64()
            _lib.call("fsx_engine_phase_ms", self.h, k, C.byref(t), C.byref(n))
            out[name] = (t.value, n.value)
        return out

    def spans(self, max_spans: int = 100000):
        """[(phase, start_ms, end_ms)] of every recorded span (synchronizes)."""
        buf = np.zeros(3 * max_spans, np.float64)
        n = C.c_uint64()
        _lib.call("fsx_engine_spans", self.h, buf.ctypes.data, max_spans, C.byref(n))
        return [(_lib.PHASES[int(buf[3 * k])], buf[3 * k + 1], buf[3 * k + 2]) for k in range(n.value)]

    def trace(self, max_spans: int = 100000):
        """[(phase, lane, channel, gpu_start_ms, gpu_end_ms, host_issue_ms)] of every
        recorded span (synchronizes; consumes them). Lanes: C L H X S, K = a copy
        stream (its channel = 1000 + 16 * all-to-all channel + destination),
        M = the side lane's part 2 (L2)."""
        buf = np.zeros(6 * max_spans, np.float64)
        n = C.c_uint64()
        _lib.call("fsx_engine_trace", self.h, buf.ctypes.data, max_spans, C.byref(n))
        return [(_lib.PHASES[int(buf[6 * k])], "CLHXSKM"[int(buf[6 * k + 1])], int(buf[6 * k + 2]),
                 buf[6 * k + 3], buf[6 * k + 4], buf[6 * k + 5]) for k in range(n.value)]

    def exposed_ms(self) -> float:
        v = C.c_double()
        _lib.call("fsx_engine_exposed_ms", self.h, C.byref(v))
        return v.value

    def close(self) -> None:
        if getattr(self, "h", None):
            _lib.lib().fsx_engine_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class SynchronizedEmbedding(_Engine):
    """Blocking baseline (embedding.cpp:235-297)."""
    _mode = _lib.FSX_MODE_SYNC

    def forward(self, ids, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        d = self._ids(ids)
        n = d.numel()
        if out is None:
            out = torch.empty((n, self.shard.geom.dim), dtype=self.shard.torch_dtype, device=d.device)
        _lib.call("fsx_engine_forward", self.h, _ptr(d), n, None, 0, _ptr(out), _stream(stream))
        self._keep = d
        self._n_cur = n
        return out

    def backward(self, grads: torch.Tensor, stream=None) -> None:
        if self._n_cur is None:
            raise ProtocolError("embedding: backward before forward")
        g = grads.to(dtype=self.shard.torch_dtype).contiguous()
        if g.numel() != self._n_cur * self.shard.geom.dim:
            raise InvalidArgument("embedding: gradient count does not match forward occurrences")
        _lib.call("fsx_engine_backward", self.h, _ptr(g), _stream(stream))
        self._keep_g = g
        self._n_cur = None


class PrioritizedEmbedding(_Engine):
    """Collision-first protocol (embedding.cpp:301-607)."""
    _mode = _lib.FSX_MODE_PRIO

    def __init__(self, *a, **kw):
        super().__init__(*a, **kw)
        self._iters = 0
        self._keep = []

    def forward(self, ids_cur, ids_next=None, out: torch.Tensor | None = None,
                stream=None) -> torch.Tensor:
        # pinned host tensors go to the engine as host pointers (side-lane H2D)
        c = ids_cur.contiguous() if isinstance(ids_cur, torch.Tensor) and not ids_cur.is_cuda and \
            ids_cur.is_pinned() else self._ids(ids_cur)
        if isinstance(ids_next, torch.Tensor) and not ids_next.is_cuda and ids_next.is_pinned():
            nx = ids_next.contiguous()
        else:
            nx = None if ids_next is None else self._ids(ids_next)
        n = c.numel()
        if out is None:
            out = torch.empty((n, self.shard.geom.dim), dtype=self.shard.torch_dtype,
                              device=self.shard.ctx.torch_device)
        _lib.call("fsx_engine_forward", self.h, _ptr(c), n, _ptr(nx),
                  0 if nx is None else nx.numel(), _ptr(out), _stream(stream))
        self._keep = [c, nx, out]
        self._n_cur = n
        self._iters += 1
        return out

    def backward(self, grads: torch.Tensor, stream=None) -> None:
        if self._n_cur is None:
            raise ProtocolError("embedding: backward before forward")
        g = grads.to(dtype=self.shard.torch_dtype).contiguous()
        if g.numel() != self._n_cur * self.shard.geom.dim:
            raise InvalidArgument("embedding: gradient count does not match forward occurrences")
        _lib.call("fsx_engine_backward", self.h, _ptr(g), _stream(stream))
        self._keep.append(g)
        self._n_cur = None

    def finalize(self, stream=None) -> None:
        _lib.call("fsx_engine_finalize", self.h, _stream(stream))

    def stats(self) -> list[IterationStats]:
        out = []
        buf = (C.c_uint64 * 3)()
        for i in range(self._iters):
            _lib.call("fsx_engine_stats", self.h, i, buf)
            out.append(IterationStats(buf[0], buf[1], buf[2]))
        return out


def gather_full_table(shards: list[ShardView]) -> np.ndarray:
    """gather_full_table (embedding.cpp:611-631) from every rank's shard:
    the full table in global row-major order (f64)."""
    geom = shards[0].geom
    full = np.zeros((geom.total_rows, geom.dim), np.float64)
    for s in shards:
        full[s.shard_id::geom.num_shards] = s.values()
    return full


def checkpoint_bytes(geom: TableGeometry, full_table: np.ndarray) -> bytes:
    """embedding.cpp:633-640: u64 rows, u64 dim, u64 shards, row-major f64."""
    hdr = np.array([geom.total_rows, geom.dim, geom.num_shards], np.uint64).tobytes()
    return hdr + np.ascontiguousarray(full_table, np.float64).tobytes()


class PooledEmbedding:
    """Pooled (bag) lookup on one shard — BASELINE config 3's operator (a
    sum per (sample, table) bag; the reference has only a toy mean-pool over
    whole samples, pipeline.cpp:59-67). forward(ids, offsets) returns one row
    per bag: the sum of its tokens' rows in token order (f64 accumulate, one
    rounding); backward(bag_grads) gives every token its bag's gradient row
    and updates the rows as ShardView.apply_gradients (embedding.cpp:148-181)
    with the engine's fixed chunk association. Oracle: fso_pooled_*."""

    def __init__(self, shard: ShardView, max_occurrences: int, max_bags: int, reduce_chunk: int = 64):
        self.shard = shard
        h = C.c_void_p()
        _lib.call("fsx_pooled_create", shard.h, int(max_occurrences), int(max_bags), int(reduce_chunk), C.byref(h))
        self.h = h
        self._nb = 0

    def forward(self, ids, offsets, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        dev = self.shard.ctx.torch_device
        ids = _dev_u64(ids, dev)
        offsets = _dev_u64(offsets, dev)
        nb = int(offsets.numel()) - 1
        if out is None:
            out = torch.empty((max(nb, 0), self.shard.geom.dim), dtype=self.shard.torch_dtype, device=dev)
        self._nb = nb
        _lib.call("fsx_pooled_forward", self.h, C.c_void_p(ids.data_ptr()), C.c_void_p(offsets.data_ptr()), nb,
                  int(ids.numel()), C.c_void_p(out.data_ptr()), _stream(stream))
        self._keep = (ids, offsets)  # alive until the backward's plan has run
        return out

    def backward(self, bag_grads: torch.Tensor, stream=None) -> None:
        g = bag_grads.to(self.shard.torch_dtype).contiguous()
        _lib.call("fsx_pooled_backward", self.h, C.c_void_p(g.data_ptr()), _stream(stream))
        self._keep_g = g

    def close(self) -> None:
        if getattr(self, "h", None):
            _lib.call("fsx_pooled_destroy", self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass
