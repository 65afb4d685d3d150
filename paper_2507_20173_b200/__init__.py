"""B200-native Fish School Behaviour step engine (arxiv 2507.20173 hot path).

The product is libfsb_b200.so (sm_100a CUDA kernels + C-ABI, include/fsb_b200.h)
with two host-side mirrors of the reference API: include/fsb/gpu.hpp (C++,
header-only) and :mod:`paper_2507_20173_b200.sim` (Python, ctypes).
"""
from .sim import (  # noqa: F401
    FISH_DTYPE,
    EatResult,
    Engine,
    GpuExecutor,
    School,
    SimConfig,
    SimResult,
    baseline_config,
    barycentre,
    checksum,
    device_count,
    eat_phase,
    init_school,
    kChecksumEmpty,
    kInitStep,
    kWeightMin,
    move_phase,
    nccl_unique_id,
    objective,
    shard_range,
    simulate,
)
from ._native import FsbError, lib, lib_path  # noqa: F401
