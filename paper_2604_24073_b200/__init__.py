"""B200-native FreeScale embedding hot path (arxiv 2604.24073).

Collision detection, sharded gather/scatter with the collision-first SGD
update, the copy-engine all-to-all and the sequence load balancer, as
hand-written sm_100a CUDA behind the C ABI in include/fsx.h (libfsx.so).
This package is the Python mirror of the reference's C++ API.
"""
import os as _os

# The copy-engine transport parks streams on peer flags (cuStreamWaitValue32).
# Lazy module loading may then block a host thread on a kernel's first launch
# until those streams drain, which can need that very thread: load modules
# eagerly, and give every stream its own hardware queue. Effective only if
# set before the CUDA context is created (import this package first).
_os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
_os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

from . import errors  # noqa: E402,F401

__all__ = ["errors", "embedding", "partition", "sim", "comm"]
