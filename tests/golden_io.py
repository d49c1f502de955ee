"""Readers for the committed golden fixtures (tests/golden/*.npz, produced by
tests/golden/make_golden.py from the reference library)."""
import os

import numpy as np

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _group(path):
    z = np.load(os.path.join(HERE, path))
    out = {}
    for key in z.files:
        name, field = key.split("__", 1)
        out.setdefault(name, {})[field] = z[key]
    return out


def engine_cases():
    cases = {}
    for name, d in _group("engine_cases.npz").items():
        world, iters = int(d["world"]), int(d["iters"])
        ids, lens = d["ids"], d["lens"]
        batches, at = [], 0
        for i in range(iters):
            row = []
            for r in range(world):
                n = int(lens[i * world + r])
                row.append(ids[at:at + n].copy())
                at += n
            batches.append(row)
        cases[name] = dict(world=world, iters=iters, rows=int(d["rows"]), dim=int(d["dim"]),
                           lr=float(d["lr"]), seed=int(d["seed"]), batches=batches,
                           table=d["table"], stats=d["stats"])
    return cases


def collision_cases():
    return {k: tuple(v[str(i)] for i in range(5)) for k, v in _group("collision_cases.npz").items()}


def partition_cases():
    out = {}
    for k, v in _group("partition_cases.npz").items():
        e = [v[str(i)] for i in range(len(v))]
        out[k] = dict(lens=e[0], origin=e[1], local=e[2], n=int(e[3]), fbs_assign=e[4],
                      fbs_order=e[5], vbs1=(e[6], e[7], e[8]), vbs2=(e[9], e[10], e[11]))
    return out
