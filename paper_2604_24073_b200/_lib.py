"""ctypes binding of libfsx.so (include/fsx.h).

The shared library is built in-tree by ``__graft_entry__.build()`` /
``make -C paper_2604_24073_b200/csrc``. There is no fallback: if the library
is missing or cannot be loaded, importing the product API raises.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

from . import errors

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FSX_LIB") or os.path.join(HERE, "libfsx.so")
CSRC = os.path.join(HERE, "csrc")

FSX_F32, FSX_F64 = 0, 1
FSX_MODE_SYNC, FSX_MODE_PRIO = 0, 1
FSX_TRANSPORT_CE, FSX_TRANSPORT_NCCL = 0, 1
PHASES = ["merge", "split", "co_update", "ex_update", "prefetch", "eco", "route", "dedup",
          "collide", "masks", "serve", "update", "a2a", "exposed"]

_lock = threading.Lock()
_lib = None

vp = C.c_void_p
u64 = C.c_uint64
u32 = C.c_uint32
i32 = C.c_int
dbl = C.c_double
P = C.POINTER


FSX_ENGINE_PRESUM = 1


class EngineConfig(C.Structure):
    _fields_ = [("mode", C.c_int), ("transport", C.c_int), ("max_occurrences", C.c_uint64),
                ("reduce_chunk", C.c_uint32), ("flags", C.c_uint32)]


# name -> (argtypes, restype)
_SIGS = {
    "fsx_last_error": ([], C.c_char_p),
    "fsx_version": ([], C.c_char_p),
    "fsx_ctx_create": ([i32, i32, i32, P(vp)], i32),
    "fsx_ctx_destroy": ([vp], i32),
    "fsx_ctx_sync": ([vp], i32),
    "fsx_ctx_launches": ([vp], u64),
    "fsx_ctx_kernel_span": ([vp, i32, P(C.c_double), P(u64)], i32),
    "fsx_sort_unique_u64": ([vp, vp, u64, vp, vp, P(u64), vp], i32),
    "fsx_collision_split": ([vp, vp, u64, vp, u64, vp, vp, vp, P(u64), vp], i32),
    "fsx_route_by_owner": ([vp, vp, u64, u64, i32, vp, vp, P(u64), vp], i32),
    "fsx_table_create": ([vp, u64, u32, i32, i32, dbl, u64, i32, P(vp)], i32),
    "fsx_table_destroy": ([vp], i32),
    "fsx_table_local_rows": ([vp], u64),
    "fsx_table_values": ([vp], vp),
    "fsx_table_gather": ([vp, vp, u64, vp, vp, i32], i32),
    "fsx_table_sgd_update": ([vp, vp, u64, vp, vp, vp, P(u64), vp], i32),
    "fsx_table_download": ([vp, vp], i32),
    "fsx_table_upload": ([vp, vp], i32),
    "fsx_engine_create": ([vp, vp, P(EngineConfig), P(vp)], i32),
    "fsx_engine_destroy": ([vp], i32),
    "fsx_engine_connect_local": ([vp, i32, vp], i32),
    "fsx_engine_export": ([vp, vp, P(u64)], i32),
    "fsx_engine_connect_ipc": ([vp, i32, vp, u64], i32),
    "fsx_nccl_unique_id": ([vp], i32),
    "fsx_engine_connect_nccl": ([vp, vp], i32),
    "fsx_engine_forward": ([vp, vp, u64, vp, u64, vp, vp], i32),
    "fsx_engine_backward": ([vp, vp, vp], i32),
    "fsx_engine_finalize": ([vp, vp], i32),
    "fsx_engine_stats": ([vp, i32, P(u64)], i32),
    "fsx_engine_exposed_ms": ([vp, P(dbl)], i32),
    "fsx_engine_set_profiling": ([vp, i32], i32),
    "fsx_engine_set_ids_ready": ([vp, i32], i32),
    "fsx_engine_join": ([vp, vp], i32),
    "fsx_engine_set_eco_direct": ([vp, i32], i32),
    "fsx_pooled_create": ([vp, u64, u64, u32, P(vp)], i32),
    "fsx_pooled_destroy": ([vp], i32),
    "fsx_pooled_forward": ([vp, vp, vp, u64, u64, vp, vp], i32),
    "fsx_pooled_backward": ([vp, vp, vp], i32),
    "fsx_engine_spans": ([vp, vp, u64, P(u64)], i32),
    "fsx_engine_trace": ([vp, vp, u64, P(u64)], i32),
    "fsx_engine_a2a_staged": ([vp, u64, vp], i32),
    "fsx_engine_phase_ms": ([vp, i32, P(dbl), P(u64)], i32),
    "fsx_cost_estimate": ([vp, vp, vp, i32, dbl, dbl, dbl, vp, vp], i32),
    "fsx_fbs_partition": ([vp, vp, vp, vp, u64, i32, vp, vp, vp], i32),
    "fsx_vbs_partition": ([vp, vp, vp, vp, u64, i32, dbl, vp, vp, vp, vp, vp], i32),
    "fsx_autotune_update": ([i32, vp, vp, P(dbl), i32, dbl, dbl, vp], i32),
    "fsx_engine_slot_bytes": ([vp], u64),
    "fsx_a2a_ce": ([vp, vp, vp, vp, vp, u64, vp, vp], i32),
    "fsx_allgather_ce": ([vp, vp, u64, u64, vp, u64, vp, i32, vp], i32),
    "fsx_jagged_offsets": ([vp, vp, u64, vp, P(u64), vp], i32),
    "fsx_jagged_permute": ([vp, vp, u32, vp, u64, vp, u64, vp, u64, vp, vp, P(u64), vp], i32),
    "fsx_keyed_transpose_perm": ([vp, u64, u64, i32, vp, vp], i32),
    "fsx_workload_scan": ([vp, u64, i32, i32, vp, vp, u64, P(u64), P(u64)], i32),
    "fsx_workload_decode": ([vp, vp, u64, vp, u64, i32, vp, i32, vp, vp, vp, vp, u64, P(u64), vp], i32),
}

EXPORTED = sorted(_SIGS)


def lib():
    """Load libfsx.so once; raise (never fall back) when it is unavailable."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(
                    f"libfsx.so not built at {LIB_PATH}; run `make -C {CSRC}` "
                    "(or __graft_entry__.build())")
            L = C.CDLL(LIB_PATH)
            for name, (args, res) in _SIGS.items():
                f = getattr(L, name)
                f.argtypes = args
                f.restype = res
            _lib = L
        return _lib


def check(rc: int) -> None:
    if rc != 0:
        msg = lib().fsx_last_error().decode()
        raise errors.from_status(rc, msg)


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args))
