"""Golden fixtures for the pipeline harness: the reference's
own pipeline::run (pipeline.cpp:118-323, oracle/_ref/libfsref.so) on
workloads from its own generator (generate_all of a uniform-length spec),
sync and prioritized, 1 / 2 / 4 ranks, balancer off and on (FBS, VBS).
Stores each case's workload sample by sample and the run's full_checkpoint,
losses and final dense weights. Run here (the container with
/root/reference): python tests/golden/make_pipeline_golden.py"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
from oracle import Reference  # noqa: E402

CFG = dict(balancer=0, partition="fbs", alpha=1.0, dim=8, table_rows=64, lr_emb=0.05, lr_dense=0.05,
           model_seed=1, c0=50.0, c1=0.01, c2=0.0)


def cases():
    for world in (1, 2, 4):
        for prio in (0, 1):
            yield f"w{world}_{'prio' if prio else 'sync'}", world, dict(CFG, prioritized=prio)
    for world, prio, part in ((2, 0, "fbs"), (2, 1, "fbs"), (4, 1, "fbs"), (2, 1, "vbs")):
        yield f"w{world}_{'prio' if prio else 'sync'}_bal_{part}", world, dict(CFG, prioritized=prio, balancer=1,
                                                                              partition=part)


def main():
    R = Reference()
    out = {}
    for name, world, cfg in cases():
        spec = dict(world=world, batch=6, max_uih=8, lo=0, hi=8, table_rows=64, target=0.3, seed=11 + world,
                    iters=5)
        smp = R.pipeline_samples(spec)
        ckpt, losses, dense = R.pipeline_run(spec, cfg)
        for k, v in smp.items():
            out[f"{name}/samples/{k}"] = v
        out[f"{name}/spec"] = np.array([spec["world"], spec["batch"], spec["iters"]], np.int64)
        out[f"{name}/cfg"] = np.array([cfg["prioritized"], cfg["balancer"], {"fbs": 0, "vbs": 1}[cfg["partition"]]],
                                      np.int64)
        out[f"{name}/ckpt"] = np.frombuffer(ckpt, np.uint8)
        out[f"{name}/losses"] = losses
        out[f"{name}/dense"] = dense
        print(name, len(ckpt), losses)
    np.savez_compressed(os.path.join(HERE, "pipeline_cases.npz"), **out)


if __name__ == "__main__":
    main()
