"""Rank fabrics for the embedding engines (the comm.hpp layer).

The reference runs ranks as threads of one process over mailboxes
(InProcessFabric, comm.cpp:30-154). On a B200 box the ranks are GPUs and the
engines move bytes with copy-engine peer copies into each other's receive
windows; what a fabric provides is only the wiring (who can write where):

* ``DeviceFabric`` — ranks are threads of one process (the reference's
  shape, used by the parity tests and the C++ drop-in); peers are connected
  with direct device pointers. Several ranks may share one GPU.
* ``ProcessGroupFabric`` — one process per GPU under torchrun; the receive
  windows are exchanged once as CUDA IPC handles over torch.distributed.

``run(body)`` keeps InProcessFabric's contract: one thread per rank, the
lowest failing rank's exception is rethrown after all ranks finish.
"""
from __future__ import annotations

import ctypes as C
import threading

from . import _lib
from .errors import CollectiveError


class Communicator:
    """Per-rank handle: rank, world size, device and the fabric that wires
    this rank's engines to its peers (comm.hpp:105-164)."""

    def __init__(self, fabric, rank: int):
        self.fabric = fabric
        self._rank = rank

    def rank(self) -> int:
        return self._rank

    def world_size(self) -> int:
        return self.fabric.world_size

    @property
    def device(self) -> int:
        return self.fabric.device_of(self._rank)

    def connect(self, engine_handle) -> None:
        self.fabric.connect(self._rank, engine_handle)

    def connect_nccl(self, engine_handle) -> None:
        self.fabric.connect_nccl(self._rank, engine_handle)


def _nccl_id() -> bytes:
    buf = (C.c_ubyte * 128)()
    _lib.call("fsx_nccl_unique_id", buf)
    return bytes(buf)


class DeviceFabric:
    def __init__(self, world_size: int, devices: list[int] | None = None):
        if world_size < 1:
            raise ValueError("fabric: world_size must be >= 1")
        import torch
        ndev = max(torch.cuda.device_count(), 1)
        self.world_size = world_size
        self.devices = devices or [r % ndev for r in range(world_size)]
        self._lock = threading.Lock()
        self._engines: dict[int, list] = {}
        self._barrier = threading.Barrier(world_size)
        self._poisoned: str | None = None

    def device_of(self, rank: int) -> int:
        return self.devices[rank]

    def communicator(self, rank: int) -> Communicator:
        return Communicator(self, rank)

    def connect(self, rank: int, engine_handle) -> None:
        """Register this rank's engine, wait for every rank's, then wire all
        peers. Collective: every rank creates its engines in the same order."""
        with self._lock:
            self._engines.setdefault(rank, []).append(engine_handle)
            k = len(self._engines[rank]) - 1
        self._wait()
        for peer in range(self.world_size):
            if peer != rank:
                _lib.call("fsx_engine_connect_local", engine_handle, peer, self._engines[peer][k])
        self._wait()

    def connect_nccl(self, rank: int, engine_handle) -> None:
        """NCCL baseline: rank 0 makes the unique id, every rank joins."""
        if rank == 0:
            self._nccl_uid = _nccl_id()
        self._wait()
        buf = (C.c_ubyte * 128).from_buffer_copy(self._nccl_uid)
        _lib.call("fsx_engine_connect_nccl", engine_handle, buf)
        self._wait()

    def _wait(self) -> None:
        try:
            self._barrier.wait(timeout=600)
        except threading.BrokenBarrierError:
            raise CollectiveError(f"collective aborted: {self._poisoned or 'barrier broken'}")

    def poison(self, why: str) -> None:
        self._poisoned = why
        self._barrier.abort()

    def run(self, body) -> None:
        import torch
        errors: list[BaseException | None] = [None] * self.world_size

        def worker(r: int) -> None:
            try:
                torch.cuda.set_device(self.devices[r])
                body(r)
            except BaseException as e:  # noqa: BLE001
                errors[r] = e
                self.poison(f"rank {r} failed")

        threads = [threading.Thread(target=worker, args=(r,)) for r in range(self.world_size)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        for e in errors:
            if e is not None:
                raise e


class ProcessGroupFabric:
    """One rank per process (torchrun). Window handles are exchanged with
    torch.distributed.all_gather_object (gloo or nccl both work)."""

    def __init__(self, rank: int, world_size: int, device: int):
        self.rank = rank
        self.world_size = world_size
        self.device = device

    def device_of(self, rank: int) -> int:
        return self.device

    def communicator(self, rank: int | None = None) -> Communicator:
        return Communicator(self, self.rank if rank is None else rank)

    def connect(self, rank: int, engine_handle) -> None:
        import torch.distributed as dist
        blob = (C.c_ubyte * 4096)()
        n = C.c_uint64()
        _lib.call("fsx_engine_export", engine_handle, blob, C.byref(n))
        mine = bytes(blob[:n.value])
        blobs: list = [None] * self.world_size
        dist.all_gather_object(blobs, mine)
        for peer, b in enumerate(blobs):
            if peer != rank:
                buf = (C.c_ubyte * len(b)).from_buffer_copy(b)
                _lib.call("fsx_engine_connect_ipc", engine_handle, peer, buf, len(b))
        dist.barrier()

    def connect_nccl(self, rank: int, engine_handle) -> None:
        import torch.distributed as dist
        obj = [_nccl_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        buf = (C.c_ubyte * 128).from_buffer_copy(obj[0])
        _lib.call("fsx_engine_connect_nccl", engine_handle, buf)
        dist.barrier()
