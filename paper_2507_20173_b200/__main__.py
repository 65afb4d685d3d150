"""Command line: the reference's `fsb simulate` / `fsb exp*` on the B200 engine.

    python -m paper_2507_20173_b200 simulate [--fish N] [--steps T] [--seed S]
                                             [--strategy auto|stream|persistent]
                                             [--device D] [--out PATH]
    python -m paper_2507_20173_b200 gpuexp   [--fish N] [--steps T] [--seed S]
                                             [--reps R] [--warmup W] [--out PATH]

`simulate` mirrors cli.hpp:179-207: one record in the reference CSV schema
(records.py) to stdout or --out, and the human-readable line
"total <s> s, eat <s> s, checksum <hex>" to stderr (stdout when --out is given).
`gpuexp` is the GPU analogue of the paper's configuration sweeps (bench.hpp:
79-148): the step-loop strategies and step kernels of this
engine, `reps` measured repetitions after `warmup` discarded ones, one record
each.  SimConfig keeps the reference CLI's defaults (only fish/steps/seed are
settable, cli.hpp:66-79).  Exit codes follow cli.hpp:251-255: 0 ok, 1 runtime
failure, 2 usage error.
"""
from __future__ import annotations

import argparse
import math
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


def _record(experiment, strategy, cfg, eng, t, rep, threads=1) -> records.BenchRecord:
    # threads = GPU threads of the step kernel's grid; chunk = fish per thread
    return records.BenchRecord(experiment=experiment, threads=threads,
                               schedule="cluster" if strategy == "persistent" else "graph",
                               chunk=max(1, cfg.num_fish // threads), construct="gpu", rep=rep, fish=cfg.num_fish,
                               steps=cfg.num_steps, seconds_total=t.seconds_total, seconds_eat=t.seconds_eat,
                               checksum=eng.checksum())


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
    strategy = a.strategy
    with sim.Engine(cfg, device=a.device, strategy=strategy) as eng:
        _, _, t = eng.simulate(barycentre=False)
        used = "persistent" if eng.last_launches() == 1 and cfg.num_steps > 0 else "stream"
        rec = _record("custom", used, cfg, eng, t, 0)
    rc = _emit([rec], a.out, sys.stderr)
    if rc:
        return rc
    info = sys.stdout if a.out else sys.stderr
    info.write(f"total {records.format_seconds(rec.seconds_total)} s, eat "
               f"{records.format_seconds(rec.seconds_eat)} s, checksum {records.format_checksum(rec.checksum)}\n")
    return 0


def cmd_gpuexp(a) -> int:
    cfg = _config(a)
    cfg.validate()
    recs = []
    # (experiment, strategy, step kernel, CTAs per SM or None = automatic grid)
    plans = [("gpu-stream", "stream", False, None), ("gpu-stream-bulk", "stream", True, None)]
    if cfg.num_fish <= 16384:
        plans.append(("gpu-persistent", "persistent", False, None))
    # Exp 1 analogue (thread count): the CTA count of the step kernel, 1..8 per SM
    plans += [("gpu-grid", "stream", False, k) for k in (1, 2, 4, 8)]
    for name, strategy, bulk, per_sm in plans:
        try:
            with sim.Engine(cfg, device=a.device, strategy=strategy, bulk=bulk) as eng:
                if per_sm:
                    eng.set_grid(per_sm * _sms(a.device))
                ctas, tpc = eng.grid()
                threads = 1 if strategy == "persistent" else ctas * tpc
                for r in range(a.warmup + a.reps):
                    _, _, t = eng.simulate(barycentre=False)
                    if r >= a.warmup:
                        recs.append(_record(name, strategy, cfg, eng, t, r - a.warmup, threads))
        except Exception as e:  # bench.hpp:182-188: a failed cell becomes a NaN row
            sys.stderr.write(f"{name}: {e}\n")
            recs.append(records.BenchRecord(name, 1, strategy, cfg.num_fish, "gpu", 0, cfg.num_fish,
                                            cfg.num_steps, math.nan, math.nan, 0))
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
            p.add_argument("--strategy", default="auto", choices=["auto", "stream", "persistent"])
        else:
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
