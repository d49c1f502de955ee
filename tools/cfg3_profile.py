"""Config 3's pooled lookup + scatter alone (the bench's cfg3 section as a
standalone program): for launch lists / ncu captures of its kernels.
usage: python tools/cfg3_profile.py [iters]"""
import os
import sys
import types

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2604_24073_b200 import embedding as E  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 3
args = types.SimpleNamespace(rows_per_table=10_000_000, samples=2048, seed=20261018, reduce_chunk=64)
ctx = E.Context(0, 0, 1)
print(bench.run_cfg3(args, ctx, torch.device("cuda", 0), 3, iters))
