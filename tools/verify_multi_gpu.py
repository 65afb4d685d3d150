#!/usr/bin/env python3
"""Parity of BASELINE's multi-GPU configs on REAL multi-GPU hardware.

    torchrun --nnodes=1 --nproc-per-node G --master-addr 127.0.0.1 tools/verify_multi_gpu.py [--peer] [--config C2|C3|all]

One rank per GPU.  Each config runs as ONE fsb_engine_run -- the graph of step
kernels with the per-step exchange inside it: NCCL allgather by default, the
NVLink peer windows with --peer -- and is checked against the reference's own
digests (tests/golden/baseline_digests.json): every step's max_diff on every
rank, the FNV checksum chained through the ranks' shards in rank order, the
barycentre within 1e-12.  This pool offers one GPU per call, so the same check
runs there with a stand-in for NCCL's transport (tests/test_nccl_shim.py) and
this script has only been run with G = 1; it is the command for a box with
NVLink peers.  Prints one JSON line per config on rank 0; exit code 1 on a mismatch.
"""
import argparse
import json
import os
import struct
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
CONFIGS = {"C2": ("C2_1e8x50", 10**8, 50), "C3": ("C3_1e9x20", 10**9, 20), "C1": ("C1_1e7x100", 10**7, 100)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="all", help="C1, C2, C3 or all (= C2 and C3)")
    ap.add_argument("--peer", action="store_true", help="NVLink peer windows instead of the NCCL allgather")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    import torch
    import torch.distributed as dist

    import paper_2507_20173_b200 as fsb

    torch.cuda.set_device(local)
    dist.init_process_group("nccl" if world > 1 else "gloo", rank=rank, world_size=world,
                            **({"device_id": torch.device("cuda", local)} if world > 1 else {}))
    golden = json.load(open(os.path.join(ROOT, "tests", "golden", "baseline_digests.json")))
    bad = 0
    for key in (["C2", "C3"] if args.config == "all" else [args.config]):
        name, n, steps = CONFIGS[key]
        g = golden[name]
        cfg = fsb.baseline_config(n, steps)
        uid = None
        if world > 1 and not args.peer:
            obj = [fsb.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            uid = obj[0]
        with fsb.Engine(cfg, device=local, rank=rank, world_size=world, nccl_unique_id=uid,
                        peer=args.peer) as e:
            if args.peer and world > 1:
                handles = [None] * world
                dist.all_gather_object(handles, e.peer_handle())
                e.peer_connect(handles)
            e.init()
            trace, bary, tm = e.run(0, steps, barycentre=True)
            trace_ok = [struct.pack("<d", float(v)).hex() for v in trace] == g["trace_hex"]
            # the digest of the gathered school: rank r continues from rank r-1's FNV state
            h = [None]
            for r in range(world):
                if r == rank:
                    h[0] = e.checksum(h[0]) if r else e.checksum()
                dist.broadcast_object_list(h, src=r)
            want = np.array([struct.unpack("<d", bytes.fromhex(v))[0] for v in g["barycentre_fsum"]])
            bary_ok = bool(np.all(np.abs(bary[-1] - want) <= 1e-12 * np.abs(want)))
            ok = [None] * world
            dist.all_gather_object(ok, (trace_ok, bary_ok))
            dist.barrier()  # nobody closes its windows while a peer may still address them
        if rank == 0:
            sum_ok = f"{h[0]:016x}" == g["final_checksum"]
            good = sum_ok and all(t and b for t, b in ok)
            bad += 0 if good else 1
            print(json.dumps({"config": name, "gpus": world, "exchange": "peer" if args.peer else "nccl",
                              "trace_ok_per_rank": [t for t, _ in ok], "barycentre_ok_per_rank": [b for _, b in ok],
                              "checksum": f"{h[0]:016x}", "checksum_ok": sum_ok,
                              "ms_per_step": 1e3 * tm.seconds_loop / steps,
                              "fish_updates_per_s": n * steps / tm.seconds_loop, "ok": good}), flush=True)
    dist.destroy_process_group()
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
