"""Time the workload-file replay at config-2 shape: 8 ranks x
8,192 power-law UIH samples per iteration (~50 MB of records). Reports the
device decode (fsx_workload_decode: parse + offsets scan + id mover) in GB/s of
record bytes, timed with CUDA events on the launching stream, and the whole
next_iteration() (host scan + pinned H2D + decode + per-rank split) in ms."""
import ctypes as C
import json
import os
import sys
import tempfile
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_24073_b200 import _lib, workload as G, workload_file as W  # noqa: E402
from paper_2604_24073_b200.jagged import _ctx  # noqa: E402

ranks, per = 8, 8192
lens = G.uih_lengths(20261020, ranks * per).astype(np.int64)
rng = np.random.default_rng(3)
ids = rng.integers(0, 2 ** 63, int(lens.sum()), dtype=np.uint64)
offs = np.concatenate([[0], np.cumsum(lens)])
samples = [(ids[offs[s]:offs[s + 1]], [], 0.5) for s in range(ranks * per)]
spec = {"batch_size": per, "dist": {"kind": "empirical", "histogram": []}, "max_uih": 8192,
        "num_iterations": 8, "num_ranks": ranks, "seed": 1, "table_rows": 2 ** 63, "target_collision": None}
path = os.path.join(tempfile.mkdtemp(), "cfg2.bin")
it = [samples[r * per:(r + 1) * per] for r in range(ranks)]
W.save_workload(path, spec, [it] * 8)
dev = torch.device("cuda", 0)
r = W.Reader(path, dev)
torch.cuda.synchronize()
t = []
for i in range(8):
    t0 = time.perf_counter()
    r.next_iteration()
    torch.cuda.synchronize()
    t.append(time.perf_counter() - t0)
# device decode alone on resident bytes
raw = open(path, "rb").read()
hlen = int.from_bytes(raw[8:12], "little")
body = np.frombuffer(raw, np.uint8)[12 + hlen:]
cap = body.size // 20 + 1
roff = np.zeros(cap, np.uint64)
per_rank = np.zeros(ranks, np.uint64)
n, used = C.c_uint64(), C.c_uint64()
_lib.call("fsx_workload_scan", C.c_void_p(body.ctypes.data), body.size, ranks, 0, per_rank.ctypes.data_as(C.c_void_p),
          roff.ctypes.data_as(C.c_void_p), cap, C.byref(n), C.byref(used))
n, used = n.value, used.value
d_bytes = torch.from_numpy(body[:used].copy()).to(dev)
d_off = torch.from_numpy(roff[:n].view(np.int64)).to(dev)
d_len = torch.empty(n, dtype=torch.int64, device=dev)
d_offs = torch.empty(n + 1, dtype=torch.int64, device=dev)
d_lab = torch.empty(n, dtype=torch.float64, device=dev)
d_vals = torch.empty(used // 8, dtype=torch.int64, device=dev)
tot = C.c_uint64()
st = torch.cuda.current_stream(dev)
ctx = _ctx(dev).h


def dec():
    _lib.call("fsx_workload_decode", ctx, C.c_void_p(d_bytes.data_ptr()), used, C.c_void_p(d_off.data_ptr()), n, 0,
              per_rank.ctypes.data_as(C.c_void_p), ranks, C.c_void_p(d_len.data_ptr()), C.c_void_p(d_offs.data_ptr()),
              C.c_void_p(d_lab.data_ptr()), C.c_void_p(d_vals.data_ptr()), used // 8, C.byref(tot),
              C.c_void_p(st.cuda_stream))


for _ in range(3):
    dec()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ms = []
for _ in range(10):
    e0.record(st)
    dec()
    e1.record(st)
    e1.synchronize()
    ms.append(e0.elapsed_time(e1))
assert np.array_equal(d_vals[:tot.value].cpu().numpy().view(np.uint64), ids)
med = float(np.median(ms))
# the reference's own Reader on the same file (oracle/_ref, one host thread), per iteration
cpu = None
try:
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
    from oracle import Reference
    if Reference.available():
        R = Reference()
        t0 = time.perf_counter()
        R.load_workload(path)
        cpu = {"kind": "reference", "cores": 1, "ms_per_iteration": round(1e3 * (time.perf_counter() - t0) / 8, 3),
               "sample": "workload::load_workload of the same 8-iteration file"}
except Exception as e:  # noqa: BLE001 — a reported baseline, not the measured path
    cpu = {"unavailable": str(e)}
print(json.dumps({"what": "workload replay, cfg2 shape (8 ranks x 8192 samples)", "record_bytes": used,
                  "ids": int(tot.value), "decode_ms": round(med, 4),
                  "decode_GBps_record_bytes": round(used / med / 1e6, 1),
                  "decode_GBps_moved": round((used + 8 * tot.value) / med / 1e6, 1),
                  "next_iteration_ms_median": round(1e3 * float(np.median(t[2:])), 3),
                  "note": "decode includes one host sync (error word + id total)", "cpu_baseline": cpu}))
