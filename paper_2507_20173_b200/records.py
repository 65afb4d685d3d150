"""GPU rows in the reference's results schema (SURVEY.md 8(f) "next" #2).

Mirrors fsb::BenchRecord (bench.hpp:49-75) and the CSV format of csv.hpp:
header kCsvHeader (csv.hpp:23-24), seconds with 9 significant digits and NaN
for failed cells (csv.hpp:30-36), checksum as 16 lowercase hex digits
(csv.hpp:38-42).  GPU rows fill the columns as follows:
  * threads      = number of GPUs (the team that runs the construct, where
                   the reference has OpenMP threads);
  * schedule     = the step loop the engine executed: "graph" (CUDA graph of
                   step kernels), "grid" (one cooperative grid for all steps),
                   "cluster" (one thread-block cluster for all steps); in the
                   gpu-exp2 rows the work distribution of the step kernel
                   instead: "static", "dynamic", "tma-ws", "bulk-ring";
  * chunk        = fish per GPU thread of the step kernel's grid
                   (fish / (GPUs x CTAs x threads per CTA), rounded up) -- the gpu-exp1
                   sweep's axis; in the gpu-exp2 rows the fish per unit of work
                   (per CTA chunk, claimed tile, TMA round or ring stage);
  * construct    = "gpu" (simulate), or the reduction construct of the global
                   max in the gpu-exp3 rows (gpu-keyslot, gpu-lastcta, gpu-nccl, gpu-peer,
                   gpu-smem-counter, gpu-cluster-slots, gpu-flat-counter,
                   gpu-redux-dsmem);
  * seconds_eat  = SimResult::seconds_eat: the max region only, measured on
                   the device (include/fsb_b200.h fsb_timing).
The reference's own read_csv / validate_records / report charts accept them
next to its CPU rows (tests/test_records.py checks this with the reference's
csv.hpp).
"""
from __future__ import annotations

import io
import math
from dataclasses import dataclass
from typing import Iterable, List

CSV_HEADER = "experiment,threads,schedule,chunk,construct,rep,fish,steps,seconds_total,seconds_eat,checksum"


@dataclass
class BenchRecord:
    experiment: str = "custom"
    threads: int = 0
    schedule: str = ""
    chunk: int = 0
    construct: str = ""
    rep: int = 0
    fish: int = 0
    steps: int = 0
    seconds_total: float = 0.0
    seconds_eat: float = 0.0
    checksum: int = 0

    def failed(self) -> bool:  # bench.hpp:62
        return math.isnan(self.seconds_total)


def format_seconds(v: float) -> str:
    """csv.hpp:30-36: '%.9g', NaN for failed cells."""
    if math.isnan(v):
        return "NaN"
    return "%.9g" % v


def format_checksum(v: int) -> str:
    return "%016x" % v


def write_csv(out, records: Iterable[BenchRecord]) -> None:
    """csv.hpp:46-54."""
    out.write(CSV_HEADER + "\n")
    for r in records:
        out.write(",".join([r.experiment, str(r.threads), r.schedule, str(r.chunk), r.construct, str(r.rep),
                            str(r.fish), str(r.steps), format_seconds(r.seconds_total),
                            format_seconds(r.seconds_eat), format_checksum(r.checksum)]) + "\n")


def write_csv_string(records: Iterable[BenchRecord]) -> str:
    buf = io.StringIO()
    write_csv(buf, records)
    return buf.getvalue()


def read_csv(text: str) -> List[BenchRecord]:
    """csv.hpp:114-145 (same header check, 11 fields per row, blank lines skipped)."""
    lines = text.splitlines()
    if not lines:
        raise ValueError("line 1: missing header")
    if lines[0].rstrip("\r") != CSV_HEADER:
        raise ValueError(f"line 1: unknown header '{lines[0]}'")
    recs = []
    for n, line in enumerate(lines[1:], start=2):
        line = line.rstrip("\r")
        if not line:
            continue
        f = line.split(",")
        if len(f) != 11:
            raise ValueError(f"line {n}: expected 11 fields, got {len(f)}")
        sec = lambda s: float("nan") if s == "NaN" else float(s)  # noqa: E731
        recs.append(BenchRecord(f[0], int(f[1]), f[2], int(f[3]), f[4], int(f[5]), int(f[6]), int(f[7]),
                                sec(f[8]), sec(f[9]), int(f[10], 16)))
    return recs
