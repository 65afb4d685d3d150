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


def _bench_module():
    import importlib.util

    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def test_multi_gpu_branch_picks_c3_share():
    """N > 1 (or --scaling) benches BASELINE configs[3]'s weak-scaling share,
    1.25e8 fish per GPU (1e9 at N=8); N = 1 benches configs[1] (1e7)."""
    import argparse

    m = _bench_module()
    ns = lambda **kw: argparse.Namespace(**{"fish": 0, "scaling": False, **kw})  # noqa: E731
    assert m.fish_per_gpu(ns(), 1) == 10_000_000
    for world in (2, 4, 8):
        assert m.fish_per_gpu(ns(), world) == 125_000_000
    assert m.fish_per_gpu(ns(scaling=True), 1) == 125_000_000
    assert m.fish_per_gpu(ns(fish=777), 8) == 777
    assert "configs[3]" in m.workload(125_000_000, 8) and "1000000000 fish total" in m.workload(125_000_000, 8)
    assert "configs[1]" in m.workload(10_000_000, 1)


def test_both_arms_print_the_same_config():
    """The driver pairs the two arms by config: both print common_config(),
    arm-specific details live under "arm"."""
    src = open(os.path.join(ROOT, "bench.py")).read()
    assert src.count('"config": common_config(') == 2


@pytest.mark.gpu
def test_bench_scaling_workload_under_torchrun():
    """torchrun --nproc-per-node 1 bench.py --scaling: the configs[3] share
    (1.25e8 fish per GPU), with the N=1 point and the one-rank exchange costs."""
    d = run(["-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1", "--master-addr", "127.0.0.1",
             "--master-port", str(free_port()), "bench.py", "--gpus", "1", "--steps", "3", "--warmup", "3",
             "--scaling", "--no-cpu-baseline", "--no-e2e"])
    assert d["config"]["fish_per_gpu"] == 125_000_000 and "configs[3]" in d["config"]["workload"]
    sp = d["scaling_points"]
    assert sp["n1_fish"] == 125_000_000 and sp["n1_value"] > 0
    assert set(sp["exchange_us_per_step_one_rank"]) == {"nccl_allgather", "peer_window"}
