"""Command line: the reference's `fsb simulate` / `fsb exp*` on the B200 engine.

    python -m paper_2507_20173_b200 simulate [--fish N] [--steps T] [--seed S]
                                             [--strategy auto|stream|persistent|grid]
                                             [--device D] [--out PATH]
    python -m paper_2507_20173_b200 gpuexp   [--exp 1|3|all] [--fish N] [--steps T] [--seed S]
                                             [--reps R] [--warmup W] [--out PATH]
    torchrun --nproc-per-node G -m paper_2507_20173_b200 gpuexp --exp 3 ...   (the G axis)

`simulate` mirrors cli.hpp:179-207: one record in the reference CSV schema
(records.py) to stdout or --out, and the human-readable line
"total <s> s, eat <s> s, checksum <hex>" to stderr (stdout when --out is given).

`gpuexp` is the GPU analogue of the paper's sweeps (bench.hpp:79-148;
PAPER.md:118-131), `reps` measured repetitions after `warmup` discarded ones,
one record each:
  * Exp 1 (thread scaling, bench.hpp:79-103): the step kernel's grid from an
    eighth of the SMs to 8 CTAs per SM -- the fish-per-thread axis (`chunk`);
  * Exp 3 (aggregation constructs, bench.hpp:132-148): the GPU's ways of
    computing the step's global max -- a red.max key slot read across the
    kernel boundary (the graph's default), the last-CTA fold across a kernel
    boundary, in-graph NCCL allgather, NVLink peer window, cluster DSMEM +
    leader slots, shared-memory grid counter barrier, flat counter barrier,
    REDUX + DSMEM in one cluster -- each with its eat-region time
    (SimResult::seconds_eat, measured on the device), times the GPU count G
    (one rank per GPU under torchrun; the multi-rank constructs are the NCCL
    and peer exchanges).
SimConfig keeps the reference CLI's defaults (only fish/steps/seed are
settable, cli.hpp:66-79).  Exit codes follow cli.hpp:251-255: 0 ok, 1 runtime
failure, 2 usage error.
"""
from __future__ import annotations

import argparse
import math
import os
import sys

from . import records, sim


def _config(a) -> sim.SimConfig:
    return sim.SimConfig(num_fish=a.fish, num_steps=a.steps, seed=a.seed)


def _sms(device: int) -> int:
    try:
        import torch

        return torch.cuda.get_device_properties(device).multi_processor_count
    except Exception:
        return 148


SCHEDULE = {"stream": "graph", "persistent": "cluster", "grid": "grid"}


def _record(experiment, eng, cfg, t, rep, construct="gpu", gpus=1, gpu_threads=None,
            checksum=None) -> records.BenchRecord:
    """threads = GPUs (the team running the construct), schedule = the step
    loop the engine executed, chunk = fish per GPU thread (records.py)."""
    used, _ = eng.last_strategy()
    if gpu_threads is None:
        ctas, tpc = eng.grid()
        gpu_threads = ctas * tpc
    return records.BenchRecord(experiment=experiment, threads=gpus, schedule=SCHEDULE.get(used, used),
                               chunk=max(1, -(-cfg.num_fish // max(1, gpus * gpu_threads))), construct=construct,
                               rep=rep, fish=cfg.num_fish, steps=cfg.num_steps, seconds_total=t.seconds_total,
                               seconds_eat=t.seconds_eat,
                               checksum=eng.checksum() if checksum is None else checksum)


def _failed(experiment, construct, cfg, gpus, schedule="graph") -> records.BenchRecord:
    # bench.hpp:182-188: a failed cell becomes one NaN row
    return records.BenchRecord(experiment, gpus, schedule, 0, construct, 0, cfg.num_fish, cfg.num_steps,
                               math.nan, math.nan, 0)


def _emit(recs, out_path, err) -> int:
    if out_path:
        try:
            with open(out_path, "w", newline="") as f:
                records.write_csv(f, recs)
        except OSError:
            err.write(f"error: cannot open '{out_path}' for writing\n")
            return 1
    else:
        records.write_csv(sys.stdout, recs)
    return 0


def cmd_simulate(a) -> int:
    cfg = _config(a)
    cfg.validate()
    with sim.Engine(cfg, device=a.device, strategy=a.strategy) as eng:
        _, _, t = eng.simulate(barycentre=False)
        rec = _record("custom", eng, cfg, t, 0)
    rc = _emit([rec], a.out, sys.stderr)
    if rc:
        return rc
    info = sys.stdout if a.out else sys.stderr
    info.write(f"total {records.format_seconds(rec.seconds_total)} s, eat "
               f"{records.format_seconds(rec.seconds_eat)} s, checksum {records.format_checksum(rec.checksum)}\n")
    return 0


# ---- Exp 1 analogue: grid size / fish per thread ------------------------------------
def exp1(a, cfg) -> list:
    sms = _sms(a.device)
    recs = []
    for ctas in sorted({max(1, sms // 8), max(1, sms // 4), max(1, sms // 2), sms, 2 * sms, 4 * sms, 8 * sms}):
        try:
            with sim.Engine(cfg, device=a.device, strategy="stream", static_tiles=True) as eng:
                eng.set_grid(ctas)
                for r in range(a.warmup + a.reps):
                    _, _, t = eng.simulate(barycentre=False)
                    if r >= a.warmup:
                        recs.append(_record("gpu-exp1", eng, cfg, t, r - a.warmup, construct="gpu-lastcta"))
        except Exception as e:
            sys.stderr.write(f"gpu-exp1 ctas={ctas}: {e}\n")
            recs.append(_failed("gpu-exp1", "gpu-lastcta", cfg, 1))
    return recs


# ---- Exp 2 analogue: work distribution x granularity --------------------------------
# bench.hpp:103-127 sweeps the schedule kind (static / dynamic / guided) and its
# chunk.  On the GPU: static chunks (one per CTA, the static-chunk kernel), warps
# claiming tiles of 1..256 groups of 64 fish (the claimed-tile kernel: dynamic),
# and the two shared-memory pipelines (the warp-specialised TMA kernel, the
# bulk ring), each as the graph of step kernels.  chunk = fish per unit of work.
def exp2(a, cfg) -> list:
    plans = [("static", dict(static_tiles=True), None)]
    plans += [("dynamic", dict(dynamic_tiles=True), g) for g in (1, 2, 4, 8, 16, 32, 64, 128, 256)]
    plans += [("tma-ws", dict(ws_tiles=True), None), ("bulk-ring", dict(bulk=True), None)]
    recs = []
    for sched, kw, groups in plans:
        try:
            with sim.Engine(cfg, device=a.device, strategy="stream", **kw) as eng:
                if groups is not None:
                    eng.set_tile_groups(groups)
                ctas, tpc = eng.grid()
                if sched == "static":
                    chunk = -(-cfg.num_fish // ctas)
                elif sched == "dynamic":
                    # tiles never fewer than the kernel's slots allow (fsb_engine_set_tile_groups)
                    per = -(-((cfg.num_fish // 2 + 31) // 32) // (ctas * 1024))
                    chunk = 64 * max(groups, per)
                elif sched == "tma-ws":
                    chunk = 31 * 64  # one round: 31 groups, one per consumer warp
                else:
                    chunk = 2 * 256  # one ring stage: 256 pairs
                for r in range(a.warmup + a.reps):
                    _, _, t = eng.simulate(barycentre=False)
                    if r >= a.warmup:
                        # the claimed-tile kernel's graph reduces by the key slot, the other kernels by the last CTA
                        rec = _record("gpu-exp2", eng, cfg, t, r - a.warmup,
                                      construct="gpu-keyslot" if sched == "dynamic" else "gpu-lastcta")
                        rec.schedule, rec.chunk = sched, chunk
                        recs.append(rec)
        except Exception as e:
            sys.stderr.write(f"gpu-exp2 {sched} {groups}: {e}\n")
            recs.append(_failed("gpu-exp2", "gpu-lastcta", cfg, 1, schedule=sched))
    return recs


# ---- Exp 3 analogue: reduction constructs x G ---------------------------------------
# (construct, engine kwargs, multi-rank capable)
CONSTRUCTS = [
    ("gpu-keyslot", dict(strategy="stream"), False),  # the graph's default: split fold (red.max key per step)
    ("gpu-lastcta", dict(strategy="stream", last_cta_fold=True), False),
    ("gpu-nccl", dict(strategy="stream", force_nccl=True), True),
    ("gpu-peer", dict(strategy="stream", peer=True), True),
    ("gpu-smem-counter", dict(strategy="grid"), False),
    ("gpu-cluster-slots", dict(strategy="grid", l2_grid=True), False),
    ("gpu-flat-counter", dict(strategy="grid", flat_grid=True), False),
    ("gpu-redux-dsmem", dict(strategy="persistent"), False),
]


def _dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world == 1:
        return 1, 0, None
    import torch.distributed as dist

    if not dist.is_initialized():
        dist.init_process_group("gloo")  # host-side plumbing only (uids, handles, times); the data path is NCCL/NVLink
    return world, dist.get_rank(), dist


def _chained_checksum(eng, world, rank, dist) -> int:
    """fsb::checksum (sim.hpp:158-176) over the whole school: FNV-1a continued
    shard by shard in rank order."""
    h = sim.kChecksumEmpty
    for r in range(world):
        if rank == r:
            h = eng.checksum(h)
        if dist is not None:
            obj = [h]
            dist.broadcast_object_list(obj, src=r)
            h = obj[0]
    return h


def exp3(a, cfg) -> list:
    world, rank, dist = _dist()
    device = int(os.environ.get("LOCAL_RANK", a.device))
    recs = []
    for name, kw, multi in CONSTRUCTS:
        if world > 1 and not multi:
            continue
        if name == "gpu-redux-dsmem" and cfg.num_fish > 16384:
            continue
        try:
            kw = dict(kw)
            if kw.get("force_nccl") or (world > 1 and not kw.get("peer")):
                uid = [sim.nccl_unique_id() if rank == 0 else None]
                if dist is not None:
                    dist.broadcast_object_list(uid, src=0)
                kw["nccl_unique_id"] = uid[0]
                kw["force_nccl"] = True
            with sim.Engine(cfg, device=device, rank=rank, world_size=world, **kw) as eng:
                if kw.get("peer") and world > 1:
                    handles = [None] * world
                    dist.all_gather_object(handles, eng.peer_handle())
                    eng.peer_connect(handles)
                for r in range(a.warmup + a.reps):
                    _, _, t = eng.simulate(barycentre=False)
                    if world > 1:  # the job's times: max over ranks
                        tt = [None] * world
                        dist.all_gather_object(tt, (t.seconds_total, t.seconds_eat))
                        t.seconds_total = max(x[0] for x in tt)
                        t.seconds_eat = max(x[1] for x in tt)
                    h = _chained_checksum(eng, world, rank, dist)
                    if r >= a.warmup and rank == 0:
                        recs.append(_record("gpu-exp3", eng, cfg, t, r - a.warmup, construct=name, gpus=world,
                                            checksum=h))
        except Exception as e:
            sys.stderr.write(f"gpu-exp3 {name}: {e}\n")
            if rank == 0:
                recs.append(_failed("gpu-exp3", name, cfg, world))
    return recs


def cmd_gpuexp(a) -> int:
    cfg = _config(a)
    cfg.validate()
    recs = []
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if a.exp in ("1", "all") and world == 1:
        recs += exp1(a, cfg)
    if a.exp in ("2", "all") and world == 1:
        recs += exp2(a, cfg)
    if a.exp in ("3", "all"):
        recs += exp3(a, cfg)
    if int(os.environ.get("RANK", "0")) != 0:
        return 0
    return _emit(recs, a.out, sys.stderr)


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2507_20173_b200",
                                 description="Fish School Behaviour simulation on B200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    for name in ("simulate", "gpuexp"):
        p = sub.add_parser(name)
        p.add_argument("--fish", type=int, default=10000)
        p.add_argument("--steps", type=int, default=1000)
        p.add_argument("--seed", type=int, default=1)
        p.add_argument("--device", type=int, default=0)
        p.add_argument("--out", default="")
        if name == "simulate":
            p.add_argument("--strategy", default="auto", choices=["auto", "stream", "persistent", "grid"])
        else:
            p.add_argument("--exp", default="all", choices=["1", "2", "3", "all"])
            p.add_argument("--reps", type=int, default=5)
            p.add_argument("--warmup", type=int, default=1)
    try:
        a = ap.parse_args(argv)
    except SystemExit as e:
        return 0 if e.code == 0 else 2
    try:
        return cmd_simulate(a) if a.cmd == "simulate" else cmd_gpuexp(a)
    except ValueError as e:
        sys.stderr.write(f"error: {e}\n")
        return 2
    except Exception as e:
        sys.stderr.write(f"error: {e}\n")
        return 1


if __name__ == "__main__":
    sys.exit(main())
