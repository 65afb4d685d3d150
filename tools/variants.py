#!/usr/bin/env python3
"""A/B tuning: build compile-time variants of libfsb_b200.so and time them.

    python tools/variants.py build            # here (CPU): nvcc all variants
    python tools/variants.py run [--only C1]  # on the GPU box: bench_configs per variant

Variants live in build/variants/ (git-ignored, travels to the GPU box).
Experiments that lost and were removed from the sources after measurement
(per-thread cp.async prefetch ring, L2 bulk prefetch, bulk ring with STG
stores, IMAD.HI shifts, one fish per thread) are in profiles/r0*_variants.jsonl;
L2 evict_last carry-over and the cluster grid's predrawn RNG in
profiles/r04_ab_session.jsonl.

Instrumented experiment builds that are not product code were removed from
csrc/fsb_kernels.cu in round 2 (their measurements stay in profiles/): the
L2-window compute-only builds (FSB_MEM_WINDOW, profiles/r03_variants.jsonl),
the grid kernels' globaltimer phase stamps (FSB_GRID_TIMING,
profiles/r03_grid_phases.jsonl, r03_grid_ctas.jsonl, r03_cgrid_leaders.jsonl),
the persistent kernel without its exchange (FSB_CLUSTER_EXP,
profiles/r04_ab_session.jsonl), the register double-buffered claimed-tile
kernel (FSB_DYN_PIPE, profiles/r05_ab_pipe.jsonl) and the contiguous-chunk
claimed tiles (FSB_DYN_STRIPED=0).  Their sources are in git history at
commit 7dc3518 (`git show 7dc3518:paper_2507_20173_b200/csrc/fsb_kernels.cu`).
Round 2, session 3, removed after measurement (sources at commit 3ae1e18):
the warp-specialised kernel's memory-only / no-load / compute-only probes
(FSB_WS_EXP), its 640-thread two-groups-per-consumer form (FSB_WS_U), and the
persistent warp-specialised grid (FSB_FLAG_WS_GRID, wgrid_kernel) with its
per-step timing build -- profiles/round2_ab_ws_variants.jsonl,
profiles/round2_ab_wsgrid.jsonl, profiles/round2_wgrid_timing.txt; and the
persistent cluster kernel's per-phase SM-cycle stamps (clock64 around the fish
update, the block reduction and the DSMEM exchange of thread 0 of every CTA;
method and numbers in profiles/round2_cluster_phases.txt); the blocked
[x|y|w|p] x 64-fish state layout (garbage-data timing probe at 068ec7c, 3 %
faster; the full engine on real data, not committed, equal:
profiles/round2_ab_blocked_layout_real_data.jsonl); and the step
kernels' per-step CTA done-time spread (FSB_SPREAD_EXP with tools/cta_spread.py,
sources at c84bfe5, profiles/round2_cta_done_spread.jsonl); tiles claimed from one global counter
by every warp of the grid (FSB_GLOBAL_CLAIM with tools/gc_probe.py, sources at
9291174, profiles/round2_ab_global_claim.txt); the persistent cluster kernel
with one exchange level -- every warp pushes its max key to every CTA, no block
barrier (FSB_CLUSTER_WPUSH, sources at 4a0a102,
profiles/round2_ab_cluster_warp_push.jsonl).
Session 6: per-thread prefetch.global.L2 of the tile's next group(s) from the
claimed-tile kernel's full-group loop (2-3 % slower, profiles/round2_ab_dyn_full.jsonl);
the warp-specialised kernel with software-pipelined consumers -- round r+1's
RNG draws made in the same basic block as round r's fp64 arithmetic, at 1024 /
896 / 768 threads per CTA (64 / 72 / 80 registers) -- bit-exact, equal to the
plain kernel within noise (profiles/round2_ab_ws_pipe.jsonl): every structure
lands on the same ~6.0 TB/s of moved bytes.
"""
from __future__ import annotations

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "build", "variants")

VARIANTS = {
    # LDG kernel: p<pairs per thread>b<min blocks>; bulk kernel: b<pairs>s<stages>m<min blocks>
    "default": [],
    # device-side bounds checks (FSB_CHECK) compiled in: run the GPU tests with FSB_LIB pointing here
    "debug": ["-DFSB_DEBUG_CHECKS=1"],
    "p4b2": ["-DFSB_PAIRS=4", "-DFSB_MIN_BLOCKS=2"],
    "p1b4": ["-DFSB_PAIRS=1", "-DFSB_MIN_BLOCKS=4"],
    "p2b3": ["-DFSB_PAIRS=2", "-DFSB_MIN_BLOCKS=3"],
    "p2b2": ["-DFSB_PAIRS=2", "-DFSB_MIN_BLOCKS=2"],
    "p1b5": ["-DFSB_PAIRS=1", "-DFSB_MIN_BLOCKS=5"],
    "p1b6": ["-DFSB_PAIRS=1", "-DFSB_MIN_BLOCKS=6"],
    "b2s3m2": ["-DFSB_BULK_PAIRS=2", "-DFSB_BULK_STAGES=3", "-DFSB_BULK_MIN_BLOCKS=2"],
    "b1s4m3": ["-DFSB_BULK_PAIRS=1", "-DFSB_BULK_STAGES=4", "-DFSB_BULK_MIN_BLOCKS=3"],
    "b2s2m3": ["-DFSB_BULK_PAIRS=2", "-DFSB_BULK_STAGES=2", "-DFSB_BULK_MIN_BLOCKS=3"],
    "b4s2m1": ["-DFSB_BULK_PAIRS=4", "-DFSB_BULK_STAGES=2", "-DFSB_BULK_MIN_BLOCKS=1"],
    # bulk ring with more compute warps per SM (compute threads x stages x CTAs per SM): all slower
    "bk992s3m1": ["-DFSB_BULK_COMPUTE=992", "-DFSB_BULK_STAGES=3", "-DFSB_BULK_MIN_BLOCKS=1"],
    # LDG kernel with bigger CTAs (fewer CTA partials in the per-step grid reduction)
    "t512b2": ["-DFSB_STEP_THREADS=512", "-DFSB_MIN_BLOCKS=2"],
    "t1024b1": ["-DFSB_STEP_THREADS=1024", "-DFSB_MIN_BLOCKS=1"],
    # cluster-reduced grid kernel: CTAs per cluster
    "cg2": ["-DFSB_CGRID_CLUSTER=2"],
    "cg4": ["-DFSB_CGRID_CLUSTER=4"],
    "cg16": ["-DFSB_CGRID_CLUSTER=16"],
    # persistent cluster kernel: fish per CTA before another CTA is added
    "c512": ["-DFSB_CLUSTER_MIN_FISH=512"],
    "c128": ["-DFSB_CLUSTER_MIN_FISH=128"],
    # persistent cluster / cluster-grid kernels: acquire at cluster scope on the DSMEM mbarrier waits
    "clacq": ["-DFSB_CLUSTER_ACQ=1"],
    "c1024": ["-DFSB_CLUSTER_MIN_FISH=1024"],
    # persistent cluster kernel: fish per thread
    "cf2": ["-DFSB_CLUSTER_F=2"],
    "cf2m512": ["-DFSB_CLUSTER_F=2", "-DFSB_CLUSTER_MIN_FISH=512"],
    "cf4": ["-DFSB_CLUSTER_F=4"],
    # claimed-tile kernel: CTA size x CTAs per SM (default 1024 x 1, 64 registers)
    "d576x2": ["-DFSB_DYN_THREADS=576", "-DFSB_DYN_MIN_BLOCKS=2"],
    "d384x3": ["-DFSB_DYN_THREADS=384", "-DFSB_DYN_MIN_BLOCKS=3"],
    "d640x2": ["-DFSB_DYN_THREADS=640", "-DFSB_DYN_MIN_BLOCKS=2"],
    # shared-memory grid kernel: threads per CTA x pairs per thread (x pairs per pass)
    "sg768": ["-DFSB_SGRID_THREADS=768", "-DFSB_SGRID_PAIRS=5"],
    "sg640": ["-DFSB_SGRID_THREADS=640", "-DFSB_SGRID_PAIRS=6"],
    "sg512u2": ["-DFSB_SGRID_THREADS=512", "-DFSB_SGRID_PAIRS=8", "-DFSB_SGRID_U=2"],
    "sg1024": ["-DFSB_SGRID_THREADS=1024", "-DFSB_SGRID_PAIRS=4"],
    "spinacq": ["-DFSB_SPIN_ACQ=1"],
    "sg512u2np": ["-DFSB_SGRID_U=2", "-DFSB_SGRID_PRE=0"],
    "sg512np": ["-DFSB_SGRID_PRE=0"],
    "sgnopredraw": ["-DFSB_SGRID_PREDRAW=0"],
    # shared-memory grid: pairs per thread (default 7) x pairs drawn during the barrier (default 1)
    "sgp8d1": ["-DFSB_SGRID_PAIRS=8"],
    "sgp7d2": ["-DFSB_SGRID_PREDRAW=2"],
    "sgp8d2": ["-DFSB_SGRID_PAIRS=8", "-DFSB_SGRID_PREDRAW=2"],
    "sgp8d3": ["-DFSB_SGRID_PAIRS=8", "-DFSB_SGRID_PREDRAW=3"],
    "sgp8d4": ["-DFSB_SGRID_PAIRS=8", "-DFSB_SGRID_PREDRAW=4"],
    "sg1024np": ["-DFSB_SGRID_THREADS=1024", "-DFSB_SGRID_PAIRS=4", "-DFSB_SGRID_PRE=0"],
    "sg768u2np": ["-DFSB_SGRID_THREADS=768", "-DFSB_SGRID_PAIRS=5", "-DFSB_SGRID_U=2", "-DFSB_SGRID_PRE=0"],
    # claimed-tile kernel: minimum 32-pair groups per tile
    "dg1": ["-DFSB_DYN_MIN_GROUPS=1"],
    "dg2": ["-DFSB_DYN_MIN_GROUPS=2"],
    "dg8": ["-DFSB_DYN_MIN_GROUPS=8"],
    "dynguarded": ["-DFSB_DYN_FAST=0"],
    # claimed-tile kernel: the unguarded loop with 64-bit pair indices and the per-pair range predicate
    "dynfull0": ["-DFSB_DYN_FULL=0"],
    "dg16": ["-DFSB_DYN_MIN_GROUPS=16"],
    # warp-specialised kernel (FSB_FLAG_WS_TILES): round buffers in the ring
    "wsr2": ["-DFSB_WS_ROUNDS=2"],
}


def build(names=None):
    from paper_2507_20173_b200 import _build

    os.makedirs(OUT, exist_ok=True)
    for name, flags in VARIANTS.items():
        if names and name not in names:
            continue
        lib = os.path.join(OUT, f"libfsb_{name}.so")
        cmd = [_build.nvcc(), *_build.NVCC_FLAGS, *flags, "-Xptxas", "-v", "-I", _build.INCLUDE, "-I",
               _build.CSRC, *[os.path.join(_build.CSRC, s) for s in _build.SOURCES], "-o", lib, "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode:
            raise SystemExit(r.stderr)
        regs = [l for l in r.stderr.splitlines() if "registers" in l]
        print(name, "built;", "step regs:", [l.split("Used")[1].split(",")[0] for l in regs][:10])


def run(only: str, reps: int, names=None):
    for name in names or VARIANTS:
        lib = os.path.join(OUT, f"libfsb_{name}.so")
        env = dict(os.environ, FSB_LIB=lib)
        r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "bench_configs.py"), "--only", only,
                            "--reps", str(reps), "--bulk-ab"], capture_output=True, text=True, env=env)
        for line in r.stdout.splitlines():
            d = json.loads(line)
            d["variant"] = name
            print(json.dumps(d), flush=True)
        if r.returncode:
            print(json.dumps({"variant": name, "error": r.stderr[-500:]}), flush=True)


if __name__ == "__main__":
    names = None
    if "--names" in sys.argv:
        names = sys.argv[sys.argv.index("--names") + 1].split(",")
    if sys.argv[1] == "build":
        build(names)
    else:
        only = "C0,C1"
        reps = 5
        if "--only" in sys.argv:
            only = sys.argv[sys.argv.index("--only") + 1]
        run(only, reps, names)
