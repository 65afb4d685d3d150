"""A short run of tools/fuzz_parity.py inside the GPU suite: random SimConfigs x
random strategies, step kernels, split points and uploaded hand-built schools,
and random shardings through the host exchange, each against the CPU oracle
(bit-exact school and trace, barycentre within 1e-12).  The long runs are in
profiles/round2_s6_fuzz_parity.jsonl and round2_s10_fuzz_parity_final_sources.jsonl (31,000 cases, 0 mismatches)."""
import json
import os
import subprocess
import sys

import pytest

import paper_2507_20173_b200 as fsb
from conftest import ROOT

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("extra", [["--cases", "300", "--seed", "11", "--max-fish", "100000"],
                                   ["--sharded", "--cases", "100", "--seed", "12", "--max-fish", "50000"]])
def test_random_configurations_match_the_oracle(extra):
    if fsb.device_count() == 0:
        pytest.fail("no CUDA device: the GPU tests must run on a B200")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "fuzz_parity.py"), *extra],
                       capture_output=True, text=True, timeout=900)
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert lines, r.stderr[-2000:]
    assert r.returncode == 0 and lines[-1]["mismatches"] == 0, lines[:5]
