"""C-ABI boundary checks that need no GPU: the library loads, exports every
symbol include/fsb_b200.h declares, and its host-only functions behave."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import oracle
import paper_2507_20173_b200 as fsb
from paper_2507_20173_b200 import _native as N
from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "fsb_b200.h")


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fsb_\w+)\s*\(", src)))


def has_gpu():
    return fsb.device_count() > 0


def test_library_exports_every_declared_symbol():
    L = fsb.lib()
    names = header_functions()
    assert len(names) >= 20
    for n in names:
        assert hasattr(L, n), n
    out = subprocess.run(["nm", "-D", "--defined-only", fsb.lib_path()], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (fsb_\w+)", out))
    assert set(names) <= exported
    # the ctypes binding covers exactly the header
    assert sorted(n for n, _, _ in N.SIGNATURES) == names


def test_built_for_sm100a_only():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", fsb.lib_path()],
                         capture_output=True, text=True, check=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_flag_constants_match_header():
    """Every FSB_FLAG_* / FSB_STRATEGY_* value the Python layer passes equals the header's."""
    src = open(HEADER).read()
    flags = {m.group(1): int(m.group(2), 16) for m in re.finditer(r"#define FSB_(FLAG_\w+)\s+(0x[0-9a-fA-F]+)u", src)}
    assert len(flags) >= 11 and "FLAG_HOST_EXCHANGE" in flags
    for name, value in flags.items():
        assert getattr(N, name) == value, name
    assert len(set(flags.values())) == len(flags), "two flags share a bit"


def test_abi_version():
    assert fsb.lib().fsb_abi_version() == N.ABI_VERSION == 2


def test_config_validation_matches_reference():
    # sim.hpp:44-49, same order and messages
    with pytest.raises(ValueError, match="pond_size must be > 0"):
        fsb.SimConfig(pond_size=0.0).validate()
    with pytest.raises(ValueError, match="weight_scale must be >= 1"):
        fsb.SimConfig(weight_scale=0.5).validate()
    with pytest.raises(ValueError, match="step_base must be > 0"):
        fsb.SimConfig(step_base=-1.0).validate()
    with pytest.raises(ValueError, match="pond_size"):
        fsb.SimConfig(pond_size=float("nan")).validate()
    fsb.SimConfig().validate()
    assert fsb.SimConfig(weight_scale=3.0).weight_max() == 6.0


@pytest.mark.parametrize("n,g", [(0, 1), (1, 2), (7, 8), (10**9, 8), (10**7 + 3, 3), (5, 1)])
def test_shard_range_is_a_contiguous_partition(n, g):
    nxt = 0
    for r in range(g):
        first, count = fsb.shard_range(n, g, r)
        assert first == nxt
        assert first == (n * r) // g
        nxt = first + count
    assert nxt == n


def test_shard_range_rejects_bad_rank():
    with pytest.raises(fsb.FsbError):
        fsb.shard_range(10, 2, 2)


def test_checksum_helper_matches_oracle(orc):
    cfg = oracle.baseline_config(1234, 3)
    fish = orc.init(cfg)
    assert fsb.checksum(fsb.School(fish)) == orc.checksum(fish)
    assert fsb.checksum(fsb.School()) == fsb.kChecksumEmpty


def test_objective_helper():
    assert fsb.objective(100.0, 100.0, 200.0) == 0.0
    assert fsb.objective(103.0, 104.0, 200.0) == 5.0


@pytest.mark.skipif(has_gpu(), reason="a GPU is present")
def test_no_gpu_fails_loudly():
    """No CPU fallback: engine creation reports FSB_ERR_CUDA."""
    assert fsb.device_count() == 0
    with pytest.raises(fsb.FsbError) as ei:
        fsb.Engine(fsb.SimConfig(num_fish=10))
    assert ei.value.code == N.FSB_ERR_CUDA
    with pytest.raises(fsb.FsbError):
        fsb.init_school(fsb.SimConfig(num_fish=10))


def test_invalid_config_rejected_before_device():
    c = fsb.SimConfig(step_base=0.0)._c()
    h = ctypes.c_void_p()
    rc = fsb.lib().fsb_engine_create(ctypes.byref(c), None, ctypes.byref(h))
    assert rc == N.FSB_ERR_INVALID_CONFIG


def test_product_does_not_reference_oracle():
    """The product package never imports or links the checker."""
    pkg = os.path.join(ROOT, "paper_2507_20173_b200")
    for dp, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dp, f)).read()
                assert "import oracle" not in src and "liboracle" not in src and "fsb_oracle" not in src, f
    out = subprocess.run(["ldd", fsb.lib_path()], capture_output=True, text=True).stdout
    assert "oracle" not in out and "fsbref" not in out


def test_nccl_shim_exports_the_entry_points_the_engine_loads():
    """tests/cpp/libnccl_shim.so (test infrastructure for tests/test_nccl_shim.py)
    must export exactly what fsb_engine.cu's nccl_load() dlsym()s, and name a
    shared-memory object in its unique id."""
    import ctypes

    path = os.path.join(ROOT, "tests", "cpp", "libnccl_shim.so")
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp"), path], check=True)  # no-op when built
    shim = ctypes.CDLL(path)
    src = open(os.path.join(ROOT, "paper_2507_20173_b200", "csrc", "fsb_engine.cu")).read()
    import re

    wanted = set(re.findall(r'dlsym\(h, "(nccl\w+)"\)', src))
    assert wanted == {"ncclGetUniqueId", "ncclCommInitRank", "ncclCommDestroy", "ncclAllGather", "ncclGetErrorString"}
    for name in wanted:
        assert hasattr(shim, name), name
    uid = ctypes.create_string_buffer(128)
    assert shim.ncclGetUniqueId(uid) == 0
    assert uid.value.startswith(b"/fsb_nccl_shim_")
