#!/usr/bin/env python3
"""bench.py -- fish-updates/s of the B200 FSB engine (BASELINE.json metric).

A bench "step" is one simulation step over the whole school: swim + objective
+ global max(prev-cur) + barycentre sums + the (deferred) weight update for
every fish.  Workload at N=1: BASELINE.json configs[1] =
10,000,000 fish (fp64 SoA, 320 MB of state > 126 MB L2), the reference
SimConfig mapping pond_size=200, weight_scale=1, step_base=0.1, seed=7.
Multi-GPU (torchrun, N > 1) or --scaling: BASELINE configs[3]'s weak-scaling
share, 1.25e8 fish per GPU (10^9 fish at N=8), contiguous shards, one NCCL
allgather of 4 fp64 per step inside the CUDA graph.  The same record carries
the N=1 point at that per-GPU size (rank 0's GPU alone, timed before the
collective run) and the per-step cost of the NCCL and peer exchanges measured
on one rank.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--scaling]

`value` = fish-updates/s with the school resident in HBM (device events around
exactly K steps, max over ranks).  `e2e` = the same metric through the C-ABI
with host buffers: upload of the AoS School from pinned memory, K steps with
the max_diff trace returned to the host, download of the School, all timed.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FISH_PER_GPU = 10_000_000   # BASELINE configs[1]: the single-GPU metric
C3_SHARE = 125_000_000      # BASELINE configs[3] weak scaling: 1.25e8 per GPU, 1e9 fish at 8 GPUs
BYTES_PER_UPDATE = 80  # read + write of the 5 x fp64 fish state
MOVED_BYTES_PER_UPDATE = 64  # this design: read + write of x, y, w, prev (cur recomputed)
METRIC = "fish-updates/sec (fish x steps / s)"
UNIT = "fish-updates/s"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, device: int, period: float = 0.002):
        self.device, self.period = device, period
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        return {
            "sm_mhz": statistics.median(self.samples) if self.samples else None,
            "sm_max_mhz": self.max_mhz,
            "samples": len(self.samples),
            "reasons": sorted(self.reasons),
        }


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def allreduce_max(world, v: float, local: int) -> float:
    if world == 1:
        return v
    import torch
    import torch.distributed as dist

    t = torch.tensor([v], dtype=torch.float64, device=f"cuda:{local}")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def cpu_baseline_sample(n: int, steps: int):
    """Rank-0 CPU baseline: the reference's sequential path (oracle/_ref, the
    reference headers compiled unmodified), 1 core, n fish x `steps` steps."""
    import oracle

    cfg = oracle.baseline_config(n, steps + 1)
    try:
        ref = oracle.Reference()
        total, _, _ = ref.time_steps(cfg, warmup=1, steps=steps, threads=1, construct=oracle.SEQUENTIAL)
        kind = "reference"
    except Exception:
        # oracle port (plain C restatement), timed the same way
        orc = oracle.Oracle()
        fish = orc.init(cfg)
        orc.run(cfg, fish, 0, 1)
        t0 = time.perf_counter()
        orc.run(cfg, fish, 1, steps)
        total = time.perf_counter() - t0
        kind = "port"
    return {
        "value": n * steps / total,
        "unit": UNIT,
        "cores": 1,
        "kind": kind,
        "sample": f"{n} fish x {steps} steps (sequential construct, 1 core, after 1 warm-up step; "
                  f"{total:.2f} s on {cpu_model()})",
    }


def fish_per_gpu(args, world: int) -> int:
    """configs[1] (1e7) for the single-GPU metric; the configs[3] weak-scaling
    share (1.25e8 per GPU) under torchrun with N > 1 or with --scaling."""
    if args.fish:
        return args.fish
    return C3_SHARE if (world > 1 or args.scaling) else FISH_PER_GPU


def workload(n_per_gpu: int, world: int) -> str:
    """The config.workload string both arms print (the driver pairs them)."""
    if n_per_gpu == FISH_PER_GPU:
        which = "BASELINE configs[1]"
    elif n_per_gpu == C3_SHARE:
        which = "BASELINE configs[3] weak-scaling share, 1e9 fish at 8 GPUs"
    else:
        which = "custom size"
    return (f"FSB {n_per_gpu} fish per GPU fp64 SoA, pond 200, w0 1.0, step_base 0.1, "
            f"seed 7 ({which}); {n_per_gpu * world} fish total")


def common_config(n_local: int, world: int) -> dict:
    """The config dict both arms print, key for key; arm-specific details go
    to the sibling key "arm"."""
    return {"workload": workload(n_local, world), "fish_per_gpu": n_local, "fish_total": n_local * world,
            "pond_size": 200.0, "weight_scale": 1.0, "step_base": 0.1, "seed": 7}


def run_reference(args, world, rank):
    """--impl reference: the reference's own CPU implementation (oracle/_ref =
    the reference headers compiled with its flags) on all host threads, with its
    default RunConfig schedule (static:50, Reduction; schedule.hpp:71-75)."""
    if rank != 0:
        return
    import oracle

    threads = os.cpu_count() or 1
    n = fish_per_gpu(args, world)
    cfg = oracle.baseline_config(n, args.warmup + args.steps)
    ref = oracle.Reference()
    total, per, _ = ref.time_steps(cfg, warmup=args.warmup, steps=args.steps, threads=threads,
                                   sched=oracle.STATIC, chunk=50, construct=oracle.REDUCTION)
    value = n * args.steps / total
    sample = (f"{n} fish x {args.steps} steps per run on {threads} threads ({cpu_model()}); "
              f"RunConfig{{{threads}, static:50, Reduction}} = the reference default construct "
              f"(its max drops a worker's partial, executor.hpp:243 -- timing only)")
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (reference init_school, seed 7)",
        "config": common_config(n, world),
        "arm": {"parallelism": f"cpu {threads} threads", "construct": "reference default RunConfig",
                "sample": f"{n} fish (the per-GPU school) on the host, the bounded sample of the "
                          f"{n * world}-fish workload"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def load_profile_traffic(n: int, kernel: str):
    """dram bytes per step-kernel launch from the committed ncu --set full summary
    (only when it captured the same kernel at the same school size)."""
    path = os.path.join(ROOT, "profiles", "step_kernel_ncu.json")
    try:
        with open(path) as f:
            p = json.load(f)
        if int(p.get("fish", -1)) == n and p.get("kernel_id", "step_kernel") == kernel:
            return float(p["dram_bytes_per_launch"]), p.get("source")
    except Exception:
        pass
    return None, None


def issue_roofline(n: int, kernel: str, kernel_s: float, clocks: dict):
    """The step kernel's second roofline: SM instruction issue (one warp
    instruction per SMSP per cycle).  Instructions per fish from the committed
    ncu capture (profiles/step_kernel_ncu.json), clock from the timed region."""
    try:
        with open(os.path.join(ROOT, "profiles", "step_kernel_ncu.json")) as f:
            p = json.load(f)
        if p.get("kernel_id", "step_kernel") != kernel:
            return None
        instr_per_fish = float(p["thread_instructions_per_fish"])
    except Exception:
        return None
    import torch

    sms = torch.cuda.get_device_properties(0).multi_processor_count if torch.cuda.is_available() else 148
    mhz = clocks.get("sm_mhz") or clocks.get("sm_max_mhz") or 1965.0
    peak = sms * 4 * mhz * 1e6  # warp instructions / s
    achieved = instr_per_fish / 32.0 * n / kernel_s
    return {"bound": "issue", "unit": "warp-instr/s", "instr_per_fish": instr_per_fish, "achieved": achieved,
            "peak": peak, "frac": achieved / peak,
            "note": "issue-active fraction the step kernel sustains; with HBM frac_moved ~0.8 both limits bind"}


def same_bytes_memory_bound(state_bytes: int, device: int):
    """Memory-only kernels over the step's own traffic (the state read and
    written once): torch's in-place fp64 add (the step's in-place pattern) and
    an out-of-place copy, best of 5 with CUDA events.  At 320 MB they run below
    the 4 GB copy of MEASURED_PEAKS.json (launch ramp and tail), so they are
    the practical bound the step kernel is compared with."""
    import torch

    n = state_bytes // 8
    a = torch.ones(n, dtype=torch.float64, device=f"cuda:{device}")
    b = torch.empty_like(a)
    out = {}
    for name, fn in (("inplace_add", lambda: a.add_(1.0)), ("copy", lambda: b.copy_(a))):
        for _ in range(3):
            fn()
        best = None
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            e1.synchronize()
            t = e0.elapsed_time(e1) * 1e-3
            best = t if best is None else min(best, t)
        out[name] = {"us": best * 1e6, "gbs": 2 * state_bytes / best / 1e9}
    del a, b
    torch.cuda.empty_cache()
    return out


def time_one_rank(n: int, steps: int, warmup: int, device: int, **kw):
    """One world-1 engine at n fish on this GPU: device time of `steps` steps
    after `warmup` (graph of step kernels; the same run() the bench times)."""
    import paper_2507_20173_b200 as fsb

    cfg = fsb.baseline_config(n, warmup + steps)
    with fsb.Engine(cfg, device=device, **kw) as eng:
        eng.init()
        eng.run(0, warmup)
        _, _, t = eng.run(warmup, steps)
        return t.seconds_loop, t.seconds_eat


def scaling_points(n_local: int, args, device: int):
    """Rank 0, before the collective run: the N=1 point at the same per-GPU
    size, and the per-step cost of each exchange measured on one rank (the
    in-graph NCCL allgather, the peer-window stores of the step kernel) as the
    difference to the plain single-rank graph."""
    import paper_2507_20173_b200 as fsb

    plain, plain_eat = time_one_rank(n_local, args.steps, args.warmup, device, strategy="stream")
    nccl, nccl_eat = time_one_rank(n_local, args.steps, args.warmup, device, strategy="stream", force_nccl=True,
                                   nccl_unique_id=fsb.nccl_unique_id())
    peer, peer_eat = time_one_rank(n_local, args.steps, args.warmup, device, strategy="stream", peer=True)
    k = args.steps
    return {
        "n1_value": n_local * k / plain,
        "n1_ms_per_step": 1e3 * plain / k,
        "n1_fish": n_local,
        "exchange_us_per_step_one_rank": {
            "nccl_allgather": 1e6 * (nccl - plain) / k,
            "peer_window": 1e6 * (peer - plain) / k,
        },
        "eat_region_us_per_step_one_rank": {"plain": 1e6 * plain_eat / k, "nccl_allgather": 1e6 * nccl_eat / k,
                                            "peer_window": 1e6 * peer_eat / k},
        "note": "rank 0's GPU alone, before the collective run; exchange cost = the graph with the exchange "
                "minus the plain graph, on one rank (the N>1 run adds the NVLink transfer)",
    }


def run_ours(args, world, rank, local):
    import ctypes

    import numpy as np

    import paper_2507_20173_b200 as fsb
    from paper_2507_20173_b200 import _native as N

    n_local = fish_per_gpu(args, world)
    n_total = n_local * world
    scaling = None
    if (world > 1 or args.scaling) and rank == 0 and not args.no_scaling_points:
        scaling = scaling_points(n_local, args, local)
    barrier(world)
    cfg = fsb.baseline_config(n_total, args.warmup + args.steps)
    uid = None
    if world > 1 and not args.peer:
        import torch.distributed as dist

        obj = [fsb.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    elif args.force_nccl:
        uid = fsb.nccl_unique_id()
    eng = fsb.Engine(cfg, device=local, rank=rank, world_size=world, nccl_unique_id=uid,
                     strategy=args.strategy, alternate=not args.no_alternate, bulk=args.bulk,
                     force_nccl=args.force_nccl, peer=args.peer, ws_tiles=args.ws)
    if args.peer and world > 1:
        import torch.distributed as dist

        handles = [None] * world
        dist.all_gather_object(handles, eng.peer_handle())
        eng.peer_connect(handles)
    eng.init()
    if args.warmup:
        eng.run(0, args.warmup)
    barrier(world)
    eng.synchronize()
    with ClockSampler(local) as clk:
        trace, _, timing = eng.run(args.warmup, args.steps)
    eng.synchronize()
    barrier(world)
    t_dev = allreduce_max(world, timing.seconds_loop, local)
    t_eat = allreduce_max(world, timing.seconds_eat, local)
    launches = eng.last_launches()
    strategy_used, fallback = eng.last_strategy()
    value = n_total * args.steps / t_dev

    # The step kernel's average launch duration.  (a) The timed region itself -- one graph of K
    # PDL-chained step kernels plus the trailing eat between one event pair on the engine stream --
    # divided by K: an upper bound (it carries the eat kernel's share), and the figure the ncu launch
    # list agrees with (110-111 us at 1e7).  (b) An event pair around each of up to 50 eager launches:
    # every pair also times the event records between two kernels (about 4 us more per launch).
    # The roofline uses (a); (b) is reported beside it.
    kms = eng.time_step_kernels(args.warmup + args.steps, max(3, min(args.steps, 50)))
    kernel_pairs_s = float(np.mean(kms[1:])) * 1e-3 if len(kms) > 1 else float(kms[0]) * 1e-3
    kernel_s = t_dev / args.steps if strategy_used == "stream" else kernel_pairs_s
    peak_gbs, peak_src = peaks()
    achieved = BYTES_PER_UPDATE * n_local / kernel_s / 1e9
    _, cta_threads = eng.grid()
    kernel = ("step_kernel_bulk" if args.bulk else "step_kernel_ws" if args.ws
              else ("step_kernel" if cta_threads == 256 else "step_kernel_dyn"))
    traffic, traffic_src = load_profile_traffic(n_local, kernel)
    same_bytes = same_bytes_memory_bound(n_local * MOVED_BYTES_PER_UPDATE // 2, local)

    # e2e through the C-ABI with host buffers (pinned), all copies timed
    e2e = None
    if not args.no_e2e:
        L = N.lib()
        nbytes = n_local * 40
        hp = ctypes.c_void_p()
        N.check(L.fsb_host_alloc(ctypes.byref(hp), nbytes))
        host = np.ctypeslib.as_array((ctypes.c_uint8 * nbytes).from_address(hp.value)).view(fsb.FISH_DTYPE)
        eng.download(host)  # a valid School in pinned host memory
        eng.upload(host)    # untimed warm-up of the path (first-use allocations, first H2D)
        barrier(world)
        t0 = time.perf_counter()
        eng.upload(host)
        t1 = time.perf_counter()
        tr, _, _ = eng.run(args.warmup, args.steps)
        t2 = time.perf_counter()
        eng.download(host)
        t3 = time.perf_counter()
        t_e2e = t3 - t0
        barrier(world)
        t_e2e = allreduce_max(world, t_e2e, local)
        N.check(L.fsb_host_free(hp))
        e2e = {
            "value": n_total * args.steps / t_e2e,
            "unit": UNIT,
            "h2d_bytes_per_step": nbytes / args.steps,
            "d2h_bytes_per_step": (nbytes + 8 * args.steps) / args.steps,
            "upload_ms": 1e3 * (t1 - t0), "run_ms": 1e3 * (t2 - t1), "download_ms": 1e3 * (t3 - t2),
            "note": f"per rank: AoS School upload from pinned host memory + K={args.steps} steps + trace and "
                    "School download, wall clock, max over ranks; the school crosses PCIe once each way per "
                    "call, so e2e grows with K (the per-step bytes shrink as 1/K)",
        }

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_baseline_sample(min(n_local, FISH_PER_GPU), args.cpu_steps)

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": value,
            "unit": UNIT,
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": 1e3 * t_dev / args.steps,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (reference init_school on device, seed 7)",
            "config": common_config(n_local, world),
            "arm": {
                "parallelism": f"fish-sharded x{world}" + (" + NCCL allgather(4 fp64)/step" if world > 1 else ""),
                "strategy": args.strategy,
                "strategy_used": strategy_used,
                "fallback": fallback,
                "l2": f"inputs larger than L2 ({n_local * 32 / 1e6:.0f} MB resident state vs 126 MB L2)",
                "timed": "K fused step kernels + 1 trailing eat kernel, one CUDA graph launch",
            },
            "eat_region": {"seconds": t_eat, "us_per_step": 1e6 * t_eat / args.steps,
                           "note": "SimResult::seconds_eat on the device: from every fish of a step updated to "
                                   "the next kernel holding the global max (max over ranks)"},
            "roofline": {
                "bound": "hbm",
                "kernel": kernel,
                "achieved": achieved,
                "peak": peak_gbs,
                "unit": "GB/s",
                "frac": achieved / peak_gbs,
                "traffic": traffic,
                "algorithmic_bytes_per_fish_update": BYTES_PER_UPDATE,
                "moved_bytes_per_fish_update": MOVED_BYTES_PER_UPDATE,
                "achieved_moved": achieved * MOVED_BYTES_PER_UPDATE / BYTES_PER_UPDATE,
                "frac_moved": achieved * MOVED_BYTES_PER_UPDATE / BYTES_PER_UPDATE / peak_gbs,
                "note": "the compact state (cur recomputed, eat deferred into the next pass) moves 64 B "
                        "per fish-update against the 80 B algorithmic figure, so frac on 80 B can reach "
                        "1.25 at the HBM limit; the kernel is co-limited by instruction issue (DESIGN.md)",
                "kernel_ms": kernel_s * 1e3,
                "kernel_ms_source": ("timed region / K (graph of K step kernels + trailing eat, one event "
                                     "pair, max over ranks): an upper bound on the launch duration"
                                     if strategy_used == "stream" else "event pair per eager launch"),
                "kernel_ms_event_pairs": kernel_pairs_s * 1e3,
                "same_bytes_memory_only": same_bytes,
                "frac_vs_same_bytes_inplace": (same_bytes["inplace_add"]["us"] * 1e-6 / kernel_s
                                               if same_bytes else None),
                "peak_source": peak_src,
                "traffic_source": traffic_src,
            },
            "issue_roofline": issue_roofline(n_local, kernel, kernel_s, clk.summary()),
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "trace_last": float(trace[-1]),
        }
        if scaling:
            line["scaling_points"] = scaling
        print(json.dumps(line), flush=True)
    eng.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--fish", type=int, default=0,
                    help="fish per GPU (default: 1e7 = configs[1]; 1.25e8 = the configs[3] share for N > 1)")
    ap.add_argument("--scaling", action="store_true",
                    help="the weak-scaling workload (1.25e8 fish per GPU) even at N=1, with the N=1 point "
                         "and the one-rank exchange costs in the record")
    ap.add_argument("--no-scaling-points", action="store_true",
                    help="skip the N=1 point and exchange costs measured before an N>1 / --scaling run")
    ap.add_argument("--strategy", default="auto", choices=["auto", "stream", "persistent"])
    ap.add_argument("--no-alternate", action="store_true",
                    help="fixed tile order (default reverses odd steps to reuse L2 across steps)")
    ap.add_argument("--bulk", action="store_true",
                    help="cp.async.bulk shared-memory ring step kernel instead of the LDG one (A/B)")
    ap.add_argument("--ws", action="store_true",
                    help="warp-specialised step kernel (TMA producer warp + 31 consumer warps per SM; A/B)")
    ap.add_argument("--force-nccl", action="store_true",
                    help="exercise the NCCL exchange path even on one rank (testing)")
    ap.add_argument("--peer", action="store_true",
                    help="per-step exchange by NVLink peer stores from the step kernel instead of NCCL")
    ap.add_argument("--cpu-steps", type=int, default=40)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)
    if args.impl == "reference":
        # CPU only: rank 0 times the reference, the other ranks exit without
        # work -- no process group (nothing is exchanged)
        run_reference(args, int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")))
        return
    world, rank, local = dist_setup(args)
    try:
        run_ours(args, world, rank, local)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
