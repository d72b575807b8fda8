"""The per-instance flow cores K6 runs on the device (csrc/flow_core.hpp),
host-compiled against the reference's flow::max_flow / extract_assignment
on 20k random graphs and 20k instances (oracle/flow_core_check.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "flow_core_check")


def test_flow_core_matches_reference():
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/flow_core_check not built (needs /root/reference at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "FLOW CORE CHECK OK" in r.stdout
