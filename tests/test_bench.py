"""bench.py keeps the driver's contract: one JSON line with the required keys,
for our arm (GPU; plain and under torchrun with the NCCL exchange) and for the
reference arm (CPU: the reference headers compiled, oracle/_ref)."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config"}


def run(args, timeout=900):
    r = subprocess.run([sys.executable, *args], cwd=ROOT, capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_reference_arm_line():
    if not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libfsbref.so")):
        pytest.skip("oracle/_ref not built")
    d = run(["bench.py", "--impl", "reference", "--steps", "3", "--warmup", "3", "--fish", "20000"])
    assert KEYS <= d.keys() and d["impl"] == "reference"
    assert d["value"] > 0 and d["e2e"]["value"] == d["value"]
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1


@pytest.mark.gpu
def test_bench_line():
    d = run(["bench.py", "--steps", "4", "--warmup", "3", "--fish", "400000", "--cpu-steps", "2"])
    assert KEYS <= d.keys()
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["gpu_launches"] >= 1  # one cluster-grid launch here
    for k in ("roofline", "cpu_baseline", "e2e", "clocks"):
        assert d[k], k
    assert d["roofline"]["bound"] == "hbm" and d["roofline"]["frac"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0


@pytest.mark.gpu
def test_bench_torchrun_nccl_path():
    """The multi-GPU launch (torchrun, NCCL uid broadcast, allgather in the
    graph) on one rank; the claimed-tile kernel at 4e6 fish per GPU."""
    d = run(["-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1", "--master-addr", "127.0.0.1",
             "--master-port", str(free_port()), "bench.py", "--gpus", "1", "--steps", "4", "--warmup", "3",
             "--fish", "4000000", "--force-nccl", "--no-cpu-baseline"])
    assert d["value"] > 0 and d["roofline"]["kernel"] == "step_kernel_dyn"


def test_reference_arm_under_torchrun():
    """N>1 launch of the reference arm: rank 0 alone prints the line, the other
    ranks exit 0 without work."""
    if not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libfsbref.so")):
        pytest.skip("oracle/_ref not built")
    d = run(["-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
             "--master-port", str(free_port()), "bench.py", "--impl", "reference", "--gpus", "2", "--steps", "3",
             "--warmup", "3", "--fish", "20000"])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
