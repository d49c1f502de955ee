"""Host-side N>1 logic on CPU: the three-stage load balancer
(balancer.cpp:99-277) over gloo at world size 2, and its jagged stage-3 codec.
The expected balanced batches are computed here from the global sample list
and the plan (the reference's assemble semantics: receive order, per-source
cursors)."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from balancer_cases import expected_batches, make_raw

HERE = os.path.dirname(os.path.abspath(__file__))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _expected(iters, world, partition):
    return expected_batches(iters, world, partition)


@pytest.mark.parametrize("partition,lead", [("none", 1), ("custom:sorted_rr", 1), ("custom:sorted_rr", 2)])
def test_balancer_gloo_world2(tmp_path, partition, lead):
    world, iters = 2, 4
    out = str(tmp_path / "bal")
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", CUDA_VISIBLE_DEVICES="")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(HERE, "balancer_worker.py"), out, partition, str(iters), str(lead)]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=240)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    exp = _expected(iters, world, partition)
    total = 0
    for rank in range(world):
        got = json.load(open(f"{out}.rank{rank}.json"))
        assert got["fires"] == [iters, iters, iters]
        for i in range(iters):
            want = exp[i][rank]
            assert len(got["taken"][i]) == len(want)
            for (uih, cands, label), s in zip(got["taken"][i], want):
                assert uih == s.uih.tolist() and label == s.label
                assert cands == [c.tolist() for c in s.candidates]
            total += len(want)
    assert total == iters * world * 6  # conservation: every sample exactly once


def test_jagged_codec_roundtrip():
    from paper_2604_24073_b200 import balancer as B
    samples = make_raw(3, 1, 2).samples + [B.Sample(np.zeros(0, np.uint64), [], -1.25)]
    msg = B.encode_jagged(samples)
    back = B.decode_jagged(msg)
    assert back == samples
    assert B.decode_jagged(B.encode_jagged([])) == []
    from paper_2604_24073_b200.errors import ProtocolError
    with pytest.raises(ProtocolError, match="trailing"):
        B.decode_jagged(np.concatenate([msg, np.zeros(1, np.uint64)]))


def test_stage_order_and_config_errors():
    from paper_2604_24073_b200 import balancer as B
    from paper_2604_24073_b200.errors import ConfigError, ProtocolError
    with pytest.raises(ConfigError, match="lead must be >= 1"):
        B.Balancer(B.LocalComm(), B.BalancerConfig(lead=0), lambda i: make_raw(i, 0, 1), 3)
    bal = B.Balancer(B.LocalComm(), B.BalancerConfig(partition="none"), lambda i: make_raw(i, 0, 1), 3)
    bal.run_stage_for(0, 0)
    with pytest.raises(ProtocolError, match="stage 1 fired out of order"):
        bal.run_stage_for(0, 0)
    with pytest.raises(ProtocolError, match="consumed before stage 3 completed"):
        bal.take(0)
    bal.run_stage_for(0, 1)
    with pytest.raises(ProtocolError, match="peek at batch 0 before stage 3 completed"):
        bal.peek(0)
    bal.run_stage_for(0, 2)
    assert bal.peek(0).samples == make_raw(0, 0, 1).samples
    assert bal.take(0).samples == make_raw(0, 0, 1).samples
    bad = B.Balancer(B.LocalComm(), B.BalancerConfig(partition="nope"), lambda i: make_raw(i, 0, 1), 1)
    bad.run_stage_for(0, 0)
    with pytest.raises(ConfigError, match="unknown partition 'nope'"):
        bad.run_stage_for(0, 1)
    none = B.Balancer(B.LocalComm(), B.BalancerConfig(partition="custom:missing"),
                      lambda i: make_raw(i, 0, 1), 1)
    none.run_stage_for(0, 0)
    with pytest.raises(ConfigError, match="unknown custom partitioner 'missing'"):
        none.run_stage_for(0, 1)
    nob = B.Balancer(B.LocalComm(), B.BalancerConfig(), lambda i: None, 2)
    with pytest.raises(ProtocolError, match="no raw batch for iteration 0"):
        nob.run_stage_for(0, 0)
