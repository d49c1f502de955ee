"""The committed profile artefacts the bench line cites stay reproducible on
the host: profiles/traffic.json (the roofline line's `traffic`) is what
tools/traffic.py derives from the committed launch list, and the launch-list
summary parses (tools/launches.py)."""
import json
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSV = os.path.join(ROOT, "profiles", "r2_launches_dram_n1.csv")


def test_traffic_json_matches_the_launch_list():
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "traffic.json")
        r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "traffic.py"), CSV, out], capture_output=True,
                           text=True)
        assert r.returncode == 0, r.stderr
        got = json.load(open(out))["n1"]
    want = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))["n1"]
    assert got == want
    # the update moves about its algorithmic bytes (no wasted re-reads): 345 MB of DRAM for
    # ~364 MB algorithmic per launch (profiles/r2_bench_n1.json)
    bench = json.load(open(os.path.join(ROOT, "profiles", "r2_bench_n1.json")))
    algo = bench["roofline"]["algorithmic_bytes_per_launch"]
    assert 0.8 * algo < got["co_update"] < 1.1 * algo


def test_launch_list_summary_parses():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "launches.py"), CSV], capture_output=True,
                       text=True)
    assert r.returncode == 0, r.stderr
    assert "k_sgd_stream" in r.stdout and "MergeMap" in r.stdout
