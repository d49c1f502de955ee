"""Python mirror of sim::CostModel (proj/include/freescale/sim.hpp:16-36).
compute_time_for_lengths runs the libfsx cost kernel (K12), bit-exact with
the reference's f64 formula; compute_times evaluates many groups (e.g. every
rank's batch) in one launch."""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib


@dataclass
class CostModel:
    c0: float = 50.0   # µs per iteration
    c1: float = 0.01   # µs per UIH token
    c2: float = 0.0    # µs per squared token per sample

    def compute_time(self, tokens: int, sq_tokens: float) -> float:
        """sim.hpp:21-23 (host arithmetic, for reference)."""
        return self.c0 + self.c1 * float(tokens) + self.c2 * sq_tokens

    def compute_times(self, groups, ctx=None) -> np.ndarray:
        """One cost per group of lengths (one launch, one CTA per group)."""
        from .embedding import default_context
        ctx = ctx or default_context()
        groups = [np.asarray(g, np.uint64).reshape(-1) for g in groups]
        offs = np.zeros(len(groups) + 1, np.uint64)
        offs[1:] = np.cumsum([g.size for g in groups])
        flat = np.concatenate(groups) if groups else np.zeros(0, np.uint64)
        d = torch.from_numpy(flat.view(np.int64)).to(ctx.torch_device) if flat.size else \
            torch.zeros(1, dtype=torch.int64, device=ctx.torch_device)
        out = np.zeros(max(len(groups), 1), np.float64)
        if groups:
            _lib.call("fsx_cost_estimate", ctx.h, d.data_ptr(), offs.ctypes.data, len(groups), self.c0, self.c1,
                      self.c2, out.ctypes.data, torch.cuda.current_stream().cuda_stream)
        return out[:len(groups)]

    def compute_time_for_lengths(self, lengths, ctx=None) -> float:
        """sim.hpp:27-35"""
        return float(self.compute_times([lengths], ctx)[0])
