"""The five-stage pipeline harness (paper_2604_24073_b200/pipeline.py, SURVEY
§8 f-2) against the reference's own pipeline::run (pipeline.cpp:118-323):
same workload (the reference's generator), sync and prioritized engines on
the GPU, 1 / 2 / 4 ranks, balancer off and on (FBS, VBS) — the
full_checkpoint (table + dense weights), the per-iteration losses and the
final dense weights byte for byte (test_pipeline.cpp:143-207 checks sync ==
prio the same way). Goldens: tests/golden/make_pipeline_golden.py."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "pipeline_cases.npz")


def _cases():
    if not os.path.exists(GOLD):
        return []
    z = np.load(GOLD)
    return sorted({k.split("/")[0] for k in z.files})


@pytest.mark.parametrize("name", _cases())
def test_pipeline_full_checkpoint_bitwise(cuda, name):
    from paper_2604_24073_b200 import pipeline as PL
    z = np.load(GOLD)
    world, batch, iters = (int(x) for x in z[f"{name}/spec"])
    prio, bal, part = (int(x) for x in z[f"{name}/cfg"])
    samples = {k.split("/")[-1]: z[k] for k in z.files if k.startswith(f"{name}/samples/")}
    its = PL.batches_from_samples({"iters": iters, "world": world, "batch": batch}, samples)
    cfg = PL.RunConfig(mode=PL.Mode.Prioritized if prio else PL.Mode.Synchronized, balancer_enabled=bool(bal),
                       partition=("fbs", "vbs")[part], table_rows=64, dim=8, lr_embedding=0.05, lr_dense=0.05,
                       model_seed=1)
    res = PL.run(its, world, batch, cfg)
    assert np.array_equal(np.asarray(res.losses).view(np.uint64), z[f"{name}/losses"].view(np.uint64))
    assert np.array_equal(np.asarray(res.final_dense).view(np.uint64), z[f"{name}/dense"].view(np.uint64))
    assert res.full_checkpoint == z[f"{name}/ckpt"].tobytes()
