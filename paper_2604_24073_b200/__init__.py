"""B200-native FreeScale embedding hot path (arxiv 2604.24073).

Collision detection, sharded gather/scatter with the collision-first SGD
update, the copy-engine all-to-all and the sequence load balancer, as
hand-written sm_100a CUDA behind the C ABI in include/fsx.h (libfsx.so).
This package is the Python mirror of the reference's C++ API.
"""
from . import errors  # noqa: F401

__all__ = ["errors", "embedding", "partition", "sim", "comm"]
