"""Worker for tests/test_cpu_balancer.py: one rank of the three-stage balancer
over gloo (torchrun, CPU). Drives the stages through the hook registry like the
reference pipeline (balancer.cpp:73-97), takes every balanced batch and writes
them to <out>.rank<r>.json."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

import numpy as np  # noqa: E402
import torch.distributed as dist  # noqa: E402

from balancer_cases import make_raw, sorted_round_robin  # noqa: E402
from paper_2604_24073_b200 import balancer as B  # noqa: E402


def main():
    out, partition, iters, lead = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    B.register_partitioner("sorted_rr", sorted_round_robin)
    comm = B.TorchComm(device="cpu")
    bal = B.Balancer(comm, B.BalancerConfig(partition=partition, lead=lead),
                     lambda i: make_raw(i, rank, world), iters)
    hooks = B.HookRegistry()
    bal.install_hooks(hooks)
    taken = []
    for i in range(iters):
        hooks.fire(B.HookPoint.DataLoad, i)
        batch = bal.take(i)
        taken.append([[s.uih.tolist(), [c.tolist() for c in s.candidates], s.label] for s in batch.samples])
        hooks.fire(B.HookPoint.PreForward, i)
        hooks.fire(B.HookPoint.PostForward, i)
        bal.report_compute_time(100.0 + rank)
        hooks.fire(B.HookPoint.OptimizerStep, i)
    fires = [bal.stage_fires(s) for s in range(3)]
    with open(f"{out}.rank{rank}.json", "w") as f:
        json.dump({"taken": taken, "fires": fires}, f)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
