"""debug: smoke scenario, which rows differ from the oracle"""
import os, sys
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np, torch
from oracle import Oracle
from paper_2604_24073_b200 import embedding as E, workload
rows, dim = 100_000, 64
for iters in (1, 2, 3):
    batches = [[workload.zipf_batch(11, 4096, rows, offset=4096 * i)] for i in range(iters)]
    ctx = E.Context(0, 0, 1)
    shard = E.ShardView(E.TableGeometry(rows, dim, 1), 0, 0.05, 3, dtype="f64", ctx=ctx)
    eng = E.PrioritizedEmbedding(shard, max_occurrences=4096)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for i in range(iters):
            nxt = batches[i + 1][0] if i + 1 < iters else None
            out = eng.forward(batches[i][0], nxt, stream=s)
            eng.backward(out * 0.125 + 0.0625, stream=s)
        eng.finalize(stream=s)
    s.synchronize(); ctx.sync()
    got = shard.values()
    want, _ = Oracle().run_engine(1, batches, rows, dim, 0.05, 3)
    bad = np.where(np.any(got != want, axis=1))[0]
    cnt = np.bincount(np.concatenate([b[0] for b in batches]).astype(np.int64), minlength=rows)
    print(f"iters={iters} bad rows {bad.size}; occ counts of bad rows: {np.bincount(cnt[bad])[:10]} max {cnt[bad].max() if bad.size else 0}")
    if bad.size:
        r = bad[0]; print(" row", r, "got", got[r][:4], "want", want[r][:4])
    eng.close()
