"""TEST INFRASTRUCTURE — NOT PRODUCT CODE.

ctypes bindings for the two parity checkers built by ``oracle/Makefile``:

* ``Oracle``    — ``oracle/liboracle.so``, the plain-C restatement
  (``oracle/fsx_oracle.c``) of the reference hot path;
* ``Reference`` — ``oracle/_ref/libfsref.so``, the unmodified reference
  library (/root/reference/proj/src) behind ``oracle/ref_shim.cpp``. Present
  only where it was built from /root/reference (it travels to the GPU box as
  a prebuilt file; it is never rebuilt there).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
legs import this module. The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libfsref.so")

u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def build(ref: bool = True) -> None:
    """Compile the checkers (gcc/g++ only; reference only if its tree exists)."""
    targets = ["liboracle.so"]
    if ref and os.path.isdir("/root/reference/proj/src"):
        targets.append("_ref/libfsref.so")
    subprocess.run(["make", "-s", "-C", HERE, "-j8", *targets], check=True)


def _u64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint64).reshape(-1))


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64).reshape(-1))


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32).reshape(-1))


class _Lib:
    prefix = ""

    def __init__(self, path: str):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.lib = C.CDLL(path)
        err = getattr(self.lib, self.prefix + "last_error")
        err.restype = C.c_char_p
        self._err = err

    def _check(self, rc: int) -> None:
        if rc != 0:
            raise OracleError(rc, self._err().decode())

    def _fn(self, name, argtypes, restype=C.c_int):
        f = getattr(self.lib, self.prefix + name)
        f.argtypes = argtypes
        f.restype = restype
        return f

    # -- shared entry points (same signatures in both libraries) -------------
    def initial_value(self, seed: int, row: int, d: int) -> float:
        f = self._fn("initial_value", [C.c_uint64, C.c_uint64, C.c_uint32], C.c_double)
        return f(seed, row, d)

    def fbs(self, lens, origin, local, n):
        lens, origin, local = _u64(lens), _i32(origin), _i32(local)
        m = lens.size
        a = np.zeros(m, np.int32)
        o = np.zeros(m, np.uint64)
        ol = np.zeros(max(n, 1), np.uint64)
        f = self._fn("fbs", [u64p, i32p, i32p, C.c_uint64, C.c_int, i32p, u64p, u64p])
        self._check(f(lens, origin, local, m, n, a, o, ol))
        return a, _split(o, ol[:n])

    def cost(self, c0, c1, c2, lens) -> float:
        lens = _u64(lens)
        f = self._fn("cost", [C.c_double, C.c_double, C.c_double, u64p, C.c_uint64], C.c_double)
        return f(c0, c1, c2, lens, lens.size)

    def bruteforce(self, w, segments) -> float:
        w = _f64(w)
        f = self._fn("bruteforce", [f64p, C.c_uint64, C.c_int], C.c_double)
        return f(w, w.size, segments)

    def route(self, world: int, total_rows: int, batches):
        """batches: list of per-rank id arrays -> per shard (recv_ids, recv_lens, uniq), occ_shard."""
        lens = _u64([len(b) for b in batches])
        ids = _u64(np.concatenate([_u64(b) for b in batches]) if batches else [])
        tot = int(lens.sum())
        occ = np.zeros(max(tot, 1), np.int32)
        recv = np.zeros(max(tot, 1), np.uint64)
        rl = np.zeros(world * world, np.uint64)
        uq = np.zeros(max(tot, 1), np.uint64)
        nu = np.zeros(world, np.uint64)
        f = self._fn("route", [C.c_int, C.c_uint64, u64p, u64p, i32p, u64p, u64p, u64p, u64p])
        self._check(f(world, total_rows, ids, lens, occ, recv, rl, uq, nu))
        out, at, uat = [], 0, 0
        rl = rl.reshape(world, world)
        for s in range(world):
            n = int(rl[s].sum())
            out.append((recv[at:at + n].copy(), rl[s].copy(), uq[uat:uat + int(nu[s])].copy()))
            at += n
            uat += int(nu[s])
        return out, occ[:tot].copy()


def _split(flat: np.ndarray, lens: np.ndarray):
    out, at = [], 0
    for n in lens:
        out.append(flat[at:at + int(n)].copy())
        at += int(n)
    return out


class Oracle(_Lib):
    """The plain-C restatement (always buildable, travels with the repo)."""

    prefix = "fso_"

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build(ref=False)
        super().__init__(path)

    def sorted_unique(self, v) -> np.ndarray:
        v = _u64(v).copy()
        f = self._fn("sorted_unique", [u64p, C.c_uint64], C.c_uint64)
        n = f(v, v.size) if v.size else 0
        return v[:n]

    def compute_collision(self, cur, nxt):
        cur, nxt = _u64(cur), _u64(nxt)
        co = np.zeros(max(cur.size, 1), np.uint64)
        exc = np.zeros(max(cur.size, 1), np.uint64)
        exn = np.zeros(max(nxt.size, 1), np.uint64)
        n = [C.c_uint64() for _ in range(3)]
        f = self._fn("compute_collision", [u64p, C.c_uint64, u64p, C.c_uint64, u64p, C.c_void_p,
                                           u64p, C.c_void_p, u64p, C.c_void_p])
        self._check(f(cur, cur.size, nxt, nxt.size, co, C.byref(n[0]), exc, C.byref(n[1]), exn,
                      C.byref(n[2])))
        return co[:n[0].value], exc[:n[1].value], exn[:n[2].value]

    def init_shard(self, total_rows, dim, num_shards, shard, seed) -> np.ndarray:
        rows = self.local_rows(total_rows, num_shards, shard)
        v = np.zeros(max(rows * dim, 1), np.float64)
        f = self._fn("init_shard", [C.c_uint64, C.c_uint32, C.c_int, C.c_int, C.c_uint64, f64p])
        self._check(f(total_rows, dim, num_shards, shard, seed, v))
        return v[:rows * dim].reshape(rows, dim)

    def local_rows(self, total_rows, num_shards, shard) -> int:
        f = self._fn("local_rows", [C.c_uint64, C.c_int, C.c_int], C.c_uint64)
        return int(f(total_rows, num_shards, shard))

    def lookup(self, values, total_rows, dim, num_shards, shard, ids):
        values, ids = _f64(values), _u64(ids)
        out = np.zeros(max(ids.size * dim, 1), np.float64)
        f = self._fn("lookup", [f64p, C.c_uint64, C.c_uint32, C.c_int, C.c_int, u64p, C.c_uint64, f64p])
        self._check(f(values, total_rows, dim, num_shards, shard, ids, ids.size, out))
        return out[:ids.size * dim].reshape(ids.size, dim)

    def apply_gradients(self, values, total_rows, dim, num_shards, shard, lr, ids, grads):
        """Returns (new_values, unique_ids, post-update rows)."""
        values, ids, grads = _f64(values).copy(), _u64(ids), _f64(grads)
        if grads.size != ids.size * dim:
            raise OracleError(-1, f"embedding: gradient shape {grads.size} misaligned with "
                                  f"{ids.size} ids x dim {dim}")
        uq = np.zeros(max(ids.size, 1), np.uint64)
        rows = np.zeros(max(ids.size * dim, 1), np.float64)
        nu = C.c_uint64()
        f = self._fn("apply_gradients", [f64p, C.c_uint64, C.c_uint32, C.c_int, C.c_int, C.c_double,
                                         u64p, C.c_uint64, f64p, u64p, C.c_void_p, f64p])
        self._check(f(values, total_rows, dim, num_shards, shard, lr, ids, ids.size,
                      grads if grads.size else np.zeros(1), uq, C.byref(nu), rows))
        u = nu.value
        return values.reshape(-1, dim) if dim else values, uq[:u], rows[:u * dim].reshape(u, dim)

    def run_engine(self, world, batches_per_iter, total_rows, dim, lr, seed,
                   grad_scale=0.125, grad_shift=0.0625, with_stats=False, store_f32=False,
                   reduce_chunk=0, presum=False):
        """batches_per_iter[i][r] = id array. Returns (table [rows x dim], stats or None).
        store_f32: model an fp32 table; reduce_chunk / presum: the engine's
        fixed chunk association and PRESUM two-level association
        (fso_run_engine_ex2)."""
        iters = len(batches_per_iter)
        lens = _u64([len(b) for it in batches_per_iter for b in it])
        flat = [_u64(b) for it in batches_per_iter for b in it]
        ids = _u64(np.concatenate(flat)) if flat else _u64([])
        table = np.zeros(max(total_rows * dim, 1), np.float64)
        stats = np.zeros(max(3 * iters, 1), np.uint64)
        f = self._fn("run_engine_ex2", [C.c_int, C.c_int, u64p, u64p, C.c_uint64, C.c_uint32, C.c_double,
                                        C.c_uint64, C.c_double, C.c_double, f64p, C.c_void_p, C.c_int,
                                        C.c_uint32, C.c_int])
        self._check(f(world, iters, ids if ids.size else np.zeros(1, np.uint64), lens if lens.size else
                      np.zeros(1, np.uint64), total_rows, dim, lr, seed, grad_scale, grad_shift, table,
                      stats.ctypes.data if with_stats else None, int(store_f32), int(reduce_chunk),
                      int(presum)))
        return table[:total_rows * dim].reshape(total_rows, dim), (stats[:3 * iters].reshape(iters, 3)
                                                                    if with_stats else None)

    def pooled_forward(self, table, ids, offs, store_f32=False, reduce_chunk=0):
        """Sum-pooled bags of a one-shard table [rows x dim] (fso_pooled_forward)."""
        table = np.ascontiguousarray(table, np.float64)
        rows, dim = table.shape
        ids, offs = _u64(ids), _u64(offs)
        nb = offs.size - 1
        out = np.zeros(max(nb * dim, 1), np.float64)
        f = self._fn("pooled_forward", [f64p, C.c_uint64, C.c_uint32, u64p, u64p, C.c_uint64, C.c_int,
                                        C.c_uint32, f64p])
        self._check(f(table, rows, dim, ids if ids.size else np.zeros(1, np.uint64), offs, nb, int(store_f32),
                      int(reduce_chunk), out))
        return out[:nb * dim].reshape(nb, dim)

    def pooled_backward(self, table, ids, offs, bag_grads, lr, store_f32=False, reduce_chunk=0):
        """Bag gradients scattered to their tokens, then the row update
        (fso_pooled_backward); returns the updated table."""
        table = np.ascontiguousarray(table, np.float64).copy()
        rows, dim = table.shape
        ids, offs = _u64(ids), _u64(offs)
        g = _f64(bag_grads)
        f = self._fn("pooled_backward", [f64p, C.c_uint64, C.c_uint32, C.c_double, u64p, u64p, C.c_uint64, f64p,
                                         C.c_int, C.c_uint32])
        self._check(f(table, rows, dim, lr, ids if ids.size else np.zeros(1, np.uint64), offs, offs.size - 1,
                      g if g.size else np.zeros(1), int(store_f32), int(reduce_chunk)))
        return table

    def vbs(self, lens, origin, local, n, alpha, tuned_sizes=None):
        lens, origin, local = _u64(lens), _i32(origin), _i32(local)
        m = lens.size
        a = np.zeros(max(m, 1), np.int32)
        o = np.zeros(max(m, 1), np.uint64)
        ol = np.zeros(max(n, 1), np.uint64)
        sz = np.zeros(max(n, 1), np.int32)
        ts = _i32(tuned_sizes) if tuned_sizes is not None else None
        f = self._fn("vbs", [u64p, i32p, i32p, C.c_uint64, C.c_int, C.c_double, C.c_void_p, i32p,
                             i32p, u64p, u64p])
        self._check(f(lens if m else np.zeros(1, np.uint64), origin if m else np.zeros(1, np.int32),
                      local if m else np.zeros(1, np.int32), m, n, alpha,
                      ts.ctypes.data if ts is not None else None, sz, a, o, ol))
        return a[:m], _split(o, ol[:n]), sz[:n]

    def autotune(self, sizes, ema_local, ema_global, times, step=1, delta=0.05, decay=0.9):
        n = len(sizes)
        sizes, ema_local = _i32(sizes).copy(), _f64(ema_local).copy()
        eg = C.c_double(ema_global)
        times = _f64(times)
        f = self._fn("autotune", [C.c_int, i32p, f64p, C.c_void_p, C.c_int, C.c_double, C.c_double,
                                  f64p, C.c_int])
        self._check(f(n, sizes, ema_local, C.byref(eg), step, delta, decay, times, times.size // n))
        return sizes, ema_local, eg.value


class Reference(_Lib):
    """The reference library itself (oracle/_ref/libfsref.so)."""

    prefix = "fsref_"

    def __init__(self, path: str = REF_SO):
        super().__init__(path)

    @staticmethod
    def available() -> bool:
        return os.path.exists(REF_SO)

    def compute_collision(self, cur, nxt):
        cur, nxt = _u64(cur), _u64(nxt)
        bufs = [np.zeros(max(k, 1), np.uint64) for k in (cur.size, cur.size, nxt.size, cur.size, nxt.size)]
        n = [C.c_uint64() for _ in range(5)]
        f = self._fn("compute_collision", [u64p, C.c_uint64, u64p, C.c_uint64] + [u64p, C.c_void_p] * 5)
        self._check(f(cur if cur.size else np.zeros(1, np.uint64), cur.size,
                      nxt if nxt.size else np.zeros(1, np.uint64), nxt.size,
                      bufs[0], C.byref(n[0]), bufs[1], C.byref(n[1]), bufs[2], C.byref(n[2]),
                      bufs[3], C.byref(n[3]), bufs[4], C.byref(n[4])))
        return tuple(b[:k.value].copy() for b, k in zip(bufs, n))

    def apply_gradients(self, total_rows, dim, num_shards, shard, lr, seed, ids, grads):
        ids, grads = _u64(ids), _f64(grads)
        rows_local = Oracle().local_rows(total_rows, num_shards, shard)
        uq = np.zeros(max(ids.size, 1), np.uint64)
        rows = np.zeros(max(ids.size * dim, 1), np.float64)
        vals = np.zeros(max(rows_local * dim, 1), np.float64)
        nu = C.c_uint64()
        f = self._fn("apply_gradients", [C.c_uint64, C.c_uint32, C.c_int, C.c_int, C.c_double,
                                         C.c_uint64, u64p, C.c_uint64, f64p, C.c_uint64, u64p,
                                         C.c_void_p, f64p, f64p])
        self._check(f(total_rows, dim, num_shards, shard, lr, seed,
                      ids if ids.size else np.zeros(1, np.uint64), ids.size,
                      grads if grads.size else np.zeros(1), grads.size, uq, C.byref(nu), rows, vals))
        u = nu.value
        return vals[:rows_local * dim].reshape(rows_local, dim), uq[:u], rows[:u * dim].reshape(u, dim)

    def lookup(self, total_rows, dim, num_shards, shard, seed, ids):
        ids = _u64(ids)
        out = np.zeros(max(ids.size * dim, 1), np.float64)
        f = self._fn("lookup", [C.c_uint64, C.c_uint32, C.c_int, C.c_int, C.c_uint64, u64p,
                                C.c_uint64, f64p])
        self._check(f(total_rows, dim, num_shards, shard, seed,
                      ids if ids.size else np.zeros(1, np.uint64), ids.size, out))
        return out[:ids.size * dim].reshape(ids.size, dim)

    def run_engine(self, prioritized, world, batches_per_iter, total_rows, dim, lr, seed,
                   grad_scale=0.125, grad_shift=0.0625):
        iters = len(batches_per_iter)
        lens = _u64([len(b) for it in batches_per_iter for b in it])
        flat = [_u64(b) for it in batches_per_iter for b in it]
        ids = _u64(np.concatenate(flat)) if flat else _u64([])
        table = np.zeros(max(total_rows * dim, 1), np.float64)
        stats = np.zeros(max(3 * iters, 1), np.uint64)
        f = self._fn("run_engine", [C.c_int, C.c_int, C.c_int, u64p, u64p, C.c_uint64, C.c_uint32,
                                    C.c_double, C.c_uint64, C.c_double, C.c_double, f64p, u64p])
        self._check(f(int(prioritized), world, iters, ids if ids.size else np.zeros(1, np.uint64),
                      lens if lens.size else np.zeros(1, np.uint64), total_rows, dim, lr, seed,
                      grad_scale, grad_shift, table, stats))
        return table[:total_rows * dim].reshape(total_rows, dim), stats[:3 * iters].reshape(iters, 3)

    def save_workload_uniform(self, path, world, batch, max_uih, lo, hi, table_rows, seed, iters):
        """workload::save_workload of generate_all (workload.cpp:551-557)."""
        f = self._fn("save_workload_uniform", [C.c_char_p, C.c_int, C.c_int, C.c_uint64, C.c_uint64,
                                               C.c_uint64, C.c_uint64, C.c_uint64, C.c_int])
        self._check(f(path.encode(), world, batch, max_uih, lo, hi, table_rows, seed, iters))

    def load_workload(self, path):
        """workload::load_workload (workload.cpp:559-564), flattened: dict of
        ids, lens / labels per sample, counts per (iteration, rank), ranks, iterations."""
        f = self._fn("load_workload", [C.c_char_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                       C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.POINTER(C.c_int)])
        ni, ns, dims = C.c_uint64(), C.c_uint64(), (C.c_int * 2)()
        self._check(f(path.encode(), None, None, None, None, C.byref(ni), C.byref(ns), dims))
        ids = np.zeros(max(ni.value, 1), np.uint64)
        lens = np.zeros(max(ns.value, 1), np.uint64)
        labels = np.zeros(max(ns.value, 1), np.float64)
        counts = np.zeros(max(dims[0] * dims[1], 1), np.uint64)
        self._check(f(path.encode(), ids.ctypes.data, lens.ctypes.data, labels.ctypes.data, counts.ctypes.data,
                      C.byref(ni), C.byref(ns), dims))
        return {"ids": ids[:ni.value], "lens": lens[:ns.value], "labels": labels[:ns.value],
                "counts": counts[:dims[0] * dims[1]], "ranks": dims[0], "iterations": dims[1]}

    def generate_uniform(self, world, batch, max_uih, lo, hi, table_rows, target_collision, seed,
                         iters):
        cap = iters * world * batch * max(max_uih, 1)
        ids = np.zeros(max(cap, 1), np.uint64)
        lens = np.zeros(max(iters * world, 1), np.uint64)
        f = self._fn("generate_uniform", [C.c_int, C.c_int, C.c_uint64, C.c_uint64, C.c_uint64,
                                          C.c_uint64, C.c_double, C.c_int, C.c_uint64, C.c_int,
                                          u64p, u64p])
        has = target_collision is not None
        self._check(f(world, batch, max_uih, lo, hi, table_rows, target_collision if has else 0.0,
                      int(has), seed, iters, ids, lens))
        out, at = [], 0
        for i in range(iters):
            row = []
            for r in range(world):
                n = int(lens[i * world + r])
                row.append(ids[at:at + n].copy())
                at += n
            out.append(row)
        return out

    def generate_lengths(self, hist, max_uih, world, batch, seed):
        hist = _f64(hist)
        lens = np.zeros(world * batch, np.uint64)
        nc = np.zeros(world * batch, np.uint64)
        f = self._fn("generate_lengths", [f64p, C.c_uint64, C.c_uint64, C.c_int, C.c_int, C.c_uint64,
                                          u64p, u64p])
        self._check(f(hist, hist.size, max_uih, world, batch, seed, lens, nc))
        return lens, nc

    def vbs(self, lens, origin, local, n, alpha, tuned_sizes=None):
        lens, origin, local = _u64(lens), _i32(origin), _i32(local)
        m = lens.size
        a = np.zeros(max(m, 1), np.int32)
        o = np.zeros(max(m, 1), np.uint64)
        ol = np.zeros(max(n, 1), np.uint64)
        ts = np.zeros(max(n, 1), np.int32)
        if tuned_sizes is not None:
            ts[:n] = tuned_sizes
        f = self._fn("vbs", [u64p, i32p, i32p, C.c_uint64, C.c_int, C.c_double, C.c_int, C.c_int,
                             i32p, i32p, u64p, u64p])
        self._check(f(lens if m else np.zeros(1, np.uint64), origin if m else np.zeros(1, np.int32),
                      local if m else np.zeros(1, np.int32), m, n, alpha, 1,
                      int(tuned_sizes is not None), ts, a, o, ol))
        return a[:m], _split(o, ol[:n]), ts[:n]

    def autotune(self, sizes, ema_local, ema_global, times, step=1, delta=0.05, decay=0.9):
        n = len(sizes)
        sizes, ema_local = _i32(sizes).copy(), _f64(ema_local).copy()
        eg = C.c_double(ema_global)
        times = _f64(times)
        f = self._fn("autotune", [C.c_int, i32p, f64p, C.c_void_p, C.c_int, C.c_double, C.c_double,
                                  f64p, C.c_int])
        self._check(f(n, sizes, ema_local, C.byref(eg), step, delta, decay, times, times.size // n))
        return sizes, ema_local, eg.value

    def pipeline_samples(self, spec):
        """generate_all of a uniform-length WorkloadSpec (dict: world, batch,
        max_uih, lo, hi, table_rows, target (None or float), seed, iters), sample
        by sample: dict of per-sample uih_len / n_cand / label and the flat uih
        ids, candidate lengths, candidate ids (iteration, rank, sample order)."""
        args = [spec["world"], spec["batch"], spec["max_uih"], spec["lo"], spec["hi"], spec["table_rows"],
                float(spec["target"] or 0.0), int(spec["target"] is not None), spec["seed"], spec["iters"]]
        n = np.zeros(4, np.uint64)
        vp = C.c_void_p
        f = self._fn("pipeline_samples", [C.c_int, C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64,
                                          C.c_double, C.c_int, C.c_uint64, C.c_int, vp, vp, vp, vp, vp, vp, u64p])
        self._check(f(*args, None, None, None, None, None, None, n))
        ns, ni, nc, nci = (int(x) for x in n)
        out = {"uih_len": np.zeros(max(ns, 1), np.uint64), "n_cand": np.zeros(max(ns, 1), np.uint64),
               "label": np.zeros(max(ns, 1), np.float64), "ids": np.zeros(max(ni, 1), np.uint64),
               "cand_len": np.zeros(max(nc, 1), np.uint64), "cand_ids": np.zeros(max(nci, 1), np.uint64)}
        self._check(f(*args, out["uih_len"].ctypes.data, out["n_cand"].ctypes.data, out["label"].ctypes.data,
                      out["ids"].ctypes.data, out["cand_len"].ctypes.data, out["cand_ids"].ctypes.data, n))
        return {"uih_len": out["uih_len"][:ns], "n_cand": out["n_cand"][:ns], "label": out["label"][:ns],
                "ids": out["ids"][:ni], "cand_len": out["cand_len"][:nc], "cand_ids": out["cand_ids"][:nci]}

    def pipeline_run(self, spec, cfg):
        """pipeline::run (pipeline.cpp:118-323) on the spec's workload; cfg keys:
        prioritized, balancer, partition ('fbs'|'vbs'|'none'), alpha, dim,
        table_rows, lr_emb, lr_dense, model_seed, c0, c1, c2. Returns
        (full_checkpoint bytes, losses, final dense weights)."""
        args = [spec["world"], spec["batch"], spec["max_uih"], spec["lo"], spec["hi"], spec["table_rows"],
                float(spec["target"] or 0.0), int(spec["target"] is not None), spec["seed"], spec["iters"],
                int(cfg["prioritized"]), int(cfg["balancer"]), {"fbs": 0, "vbs": 1, "none": 2}[cfg["partition"]],
                float(cfg["alpha"]), int(cfg["dim"]), int(cfg["table_rows"]), float(cfg["lr_emb"]),
                float(cfg["lr_dense"]), int(cfg["model_seed"]), float(cfg["c0"]), float(cfg["c1"]), float(cfg["c2"])]
        cap = 64 + int(cfg["table_rows"]) * int(cfg["dim"]) * 8 + int(cfg["dim"]) * 8
        ckpt = np.zeros(cap, np.uint8)
        n = C.c_uint64()
        losses = np.zeros(max(spec["iters"], 1), np.float64)
        dense = np.zeros(max(int(cfg["dim"]), 1), np.float64)
        f = self._fn("pipeline_run", [C.c_int, C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, C.c_double,
                                      C.c_int, C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_uint32,
                                      C.c_uint64, C.c_double, C.c_double, C.c_uint64, C.c_double, C.c_double,
                                      C.c_double, C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64), f64p, f64p])
        self._check(f(*args, ckpt.ctypes.data, cap, C.byref(n), losses, dense))
        return ckpt[:n.value].tobytes(), losses[:spec["iters"]], dense[:int(cfg["dim"])]

    def bench_engine(self, prioritized, world, batches_per_iter, total_rows, dim, lr, seed):
        iters = len(batches_per_iter)
        lens = _u64([len(b) for it in batches_per_iter for b in it])
        ids = _u64(np.concatenate([_u64(b) for it in batches_per_iter for b in it]))
        us = np.zeros(iters, np.float64)
        f = self._fn("bench_engine", [C.c_int, C.c_int, C.c_int, u64p, u64p, C.c_uint64, C.c_uint32,
                                      C.c_double, C.c_uint64, f64p])
        self._check(f(int(prioritized), world, iters, ids, lens, total_rows, dim, lr, seed, us))
        return us
