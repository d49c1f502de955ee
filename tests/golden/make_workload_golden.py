"""Regenerate the workload-file replay fixtures from the
reference itself (oracle/_ref). Run here (not on the GPU box):

    python tests/golden/make_workload_golden.py

For each case the reference's own Writer (workload::save_workload of
generate_all, workload.cpp:142-241, 551-557) writes `workload_<name>.bin`, and
the reference's Reader (load_workload, workload.cpp:478-564) reads it back into
`workload_<name>.npz` (uih ids, per-sample lengths and labels, samples per
(iteration, rank)). The GPU tests replay the .bin through libfsx and compare
with the .npz; no reference code runs on the GPU box."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
from oracle import Reference  # noqa: E402

# (name, world, batch, max_uih, lo, hi, table_rows, seed, iters)
CASES = [
    ("small_2r", 2, 5, 40, 0, 40, 1000, 7, 3),      # lengths from 0: empty samples included
    ("ragged_4r", 4, 33, 300, 1, 300, 10 ** 6, 20261018, 2),
    ("single_1r", 1, 1, 1, 1, 1, 2, 1, 1),           # one sample of one id
]


def main():
    R = Reference()
    for name, *args in CASES:
        path = os.path.join(HERE, f"workload_{name}.bin")
        R.save_workload_uniform(path, *args)
        d = R.load_workload(path)
        np.savez(os.path.join(HERE, f"workload_{name}.npz"), **{k: np.asarray(v) for k, v in d.items()})
        print(name, os.path.getsize(path), "bytes,", d["lens"].size, "samples,", d["ids"].size, "ids")


if __name__ == "__main__":
    main()
