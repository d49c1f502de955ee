"""The reference's own C++ test cases run against the drop-in headers
(paper_2604_24073_b200/cpp): a reference user's code, unchanged, executing
on libfsx's GPU kernels."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CPP = os.path.join(ROOT, "paper_2604_24073_b200", "cpp")


def test_reference_cases_through_cpp_dropin(cuda):
    subprocess.run(["make", "-s", "-C", CPP], check=True)
    env = dict(os.environ, CUDA_MODULE_LOADING="EAGER", CUDA_DEVICE_MAX_CONNECTIONS="32")
    r = subprocess.run([os.path.join(CPP, "build", "test_dropin")], capture_output=True, text=True,
                       timeout=600, env=env)
    print(r.stdout[-4000:], r.stderr[-2000:])
    assert r.returncode == 0, r.stdout[-2000:]
    assert "0 failed" in r.stdout
