"""Multi-GPU parity: one process per GPU over CUDA IPC + copy engines
(tests/mp_engine_check.py under torchrun). Needs >= 2 GPUs on the box
(`gpurun --gpus 2`); skipped otherwise."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpus():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_multiprocess_engine_parity(dtype):
    n = _ngpus()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    world = min(n, 4)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", "--master-port=29533", os.path.join(ROOT, "tests", "mp_engine_check.py"),
           dtype]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    print(r.stdout[-3000:], r.stderr[-3000:])
    assert r.returncode == 0 and "MP_OK" in r.stdout
