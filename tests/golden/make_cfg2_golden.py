"""Config-2 golden (65,536 UIH samples over 8 ranks, power-law lengths
16..8192 drawn by the reference's own empirical generator): FBS and VBS
(alpha 1 and 2) plans and per-rank CostModel values from the reference
library (oracle/_ref). The exact VBS DP takes ~1 min per alpha on one CPU
core. Run here:  python tests/golden/make_cfg2_golden.py"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
from oracle import Reference, build  # noqa: E402


def main():
    build(ref=True)
    R = Reference()
    hist = np.zeros(8193)
    hist[16:] = np.arange(16, 8193, dtype=np.float64) ** -2.0
    lens, ncand = R.generate_lengths(hist, 8192, 8, 8192, 20261020)
    m, n = lens.size, 8
    origin = (np.arange(m) // 8192).astype(np.int32)
    local = (np.arange(m) % 8192).astype(np.int32)
    out = dict(lens=lens, origin=origin, local=local)
    a, order = R.fbs(lens, origin, local, n)
    out["fbs_assign"], out["fbs_order"] = a, np.concatenate(order)
    for alpha in (1.0, 2.0):
        a, order, sizes = R.vbs(lens, origin, local, n, alpha)
        k = int(alpha)
        out[f"vbs{k}_assign"], out[f"vbs{k}_order"], out[f"vbs{k}_sizes"] = a, np.concatenate(order), sizes
    costs = []
    for c2 in (0.0, 1e-6):
        costs.append([R.cost(50.0, 0.01, c2, lens[r * 8192:(r + 1) * 8192]) for r in range(n)])
    out["cost"] = np.array(costs, np.float64)
    np.savez_compressed(os.path.join(HERE, "cfg2_partition.npz"), **out)
    print("wrote cfg2_partition.npz", {k: v.shape for k, v in out.items()})


if __name__ == "__main__":
    main()
