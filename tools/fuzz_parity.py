#!/usr/bin/env python3
"""Randomised parity sweep on the GPU box: random SimConfigs (school size, steps,
seed, pond size, step length, weight scale -- including values far outside the
BASELINE mapping, where walls clamp, weights saturate or the in-range fast
paths do not apply) through a random engine choice (strategy, step kernel,
alternation, checked mode, split runs), each compared with the CPU oracle:
the downloaded school byte for byte, every step's max_diff bit for bit, the
barycentre within 1e-12.  The oracle is the checker (tests/ and tools only).

    python tools/fuzz_parity.py --cases 3000 --seed 1 > gpurun_out/fuzz.jsonl
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import paper_2507_20173_b200 as fsb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cases", type=int, default=1000)
ap.add_argument("--seed", type=int, default=1)
ap.add_argument("--max-fish", type=int, default=300_000)
ap.add_argument("--sharded", action="store_true",
                help="every case as G = 2..8 shards on this GPU through the host exchange (fsb_engine_partial / "
                     "set_partials between move and eat), the gathered school against the unsharded oracle")
args = ap.parse_args()
rng = np.random.default_rng(args.seed)
orc = oracle.Oracle()
KERNELS = [{}, {"static_tiles": True}, {"dynamic_tiles": True}, {"ws_tiles": True}, {"bulk": True}]
bad, t0 = 0, time.time()
counts = {}
for case in range(args.cases):
    n = int(np.exp(rng.uniform(0, np.log(args.max_fish))))
    steps = int(rng.integers(1, 13))
    pond = float(2.0 ** rng.uniform(-3, 12)) if rng.random() < 0.7 else float(rng.uniform(1, 500))
    # step lengths from a tiny fraction of the pond to several ponds (every move hits a wall)
    step_base = pond * float(10.0 ** rng.uniform(-5, 0.7))
    wscale = float(rng.choice([1.0, 1.5, 2.0, 10.0, float(2.0 ** rng.uniform(0, 8))]))
    cfg = fsb.SimConfig(num_fish=n, pond_size=pond, weight_scale=wscale, num_steps=steps,
                        seed=int(rng.integers(0, 2**64, dtype=np.uint64)), step_base=step_base)
    strategy = str(rng.choice(["auto", "stream", "grid", "persistent"] if n <= 16384 else ["auto", "stream", "grid"]))
    kw = dict(rng.choice(KERNELS)) if strategy == "stream" else {}
    if strategy == "grid" and rng.random() < 0.3:
        kw[str(rng.choice(["flat_grid", "l2_grid"]))] = True
    kw["alternate"] = bool(rng.random() < 0.7)
    if rng.random() < 0.15:
        kw["checked"] = True
    split = int(rng.integers(1, steps)) if steps > 1 and rng.random() < 0.3 else 0
    ocfg = oracle.Config.make(num_fish=n, pond_size=pond, weight_scale=wscale, num_steps=steps, seed=cfg.seed,
                              step_base=step_base)
    if args.sharded:
        world = int(rng.integers(2, 9))
        skw = dict(rng.choice(KERNELS[:4]))
        want_fish, want_trace = orc.simulate(ocfg)
        try:
            engs = [fsb.Engine(cfg, device=0, rank=r, world_size=world, host_exchange=True, **skw)
                    for r in range(world)]
            try:
                for e in engs:
                    e.init()
                trace = []
                for t in range(steps):
                    for e in engs:
                        e.move(t)
                    parts = np.stack([e.partial() for e in engs])
                    for e in engs:
                        e.set_partials(parts)
                    trace.append({e.eat().max_diff for e in engs})
                got = b"".join(e.download().tobytes() for e in engs)
            finally:
                for e in engs:
                    e.close()
            ok = (got == want_fish.tobytes() and all(len(m) == 1 for m in trace)
                  and np.array([m.pop() for m in trace]).tobytes() == want_trace.tobytes())
            err = ""
        except Exception as ex:  # noqa: BLE001
            ok, err = False, repr(ex)
        counts[f"G={world}"] = counts.get(f"G={world}", 0) + 1
        if not ok:
            bad += 1
            print(json.dumps({"case": case, "ok": False, "n": n, "steps": steps, "pond": pond,
                              "step_base": step_base, "weight_scale": wscale, "seed": cfg.seed, "world": world,
                              "kw": skw, "error": err}), flush=True)
        continue
    # a third of the cases start from an UPLOADED hand-built school instead of init: fish outside the pond,
    # weights outside [1, w_max], arbitrary prev / current objectives (the explicit-cur kernels), special values
    upload = None
    first = 0
    if rng.random() < 0.33 and n <= 50_000:
        upload = np.zeros(n, dtype=oracle.FISH_DTYPE)
        upload["x"] = rng.uniform(-0.2 * pond, 1.2 * pond, n)
        upload["y"] = rng.uniform(-0.2 * pond, 1.2 * pond, n)
        upload["weight"] = np.where(rng.random(n) < 0.5, 1.0, rng.uniform(0.25, 3.0 * cfg.weight_max(), n))
        upload["prev_objective"] = rng.uniform(0, pond, n)
        upload["current_objective"] = rng.uniform(0, pond, n)
        special = np.array([0.0, -0.0, 5e-324, 1e-310, 1e300, pond / 2, pond, np.nextafter(pond, np.inf)])
        for f in ("x", "y", "weight", "prev_objective", "current_objective"):
            k = int(rng.integers(0, min(n, 8) + 1))
            upload[f][rng.integers(0, n, k)] = rng.choice(special, k)
        if rng.random() < 0.5:  # a consistent current objective: the compact kernels after an upload
            for i in range(n):
                upload["current_objective"][i] = orc.objective(upload["x"][i], upload["y"][i], pond)
        first = int(rng.integers(0, 2**40))
        want_fish = upload.copy()
        want_trace = orc.run(ocfg, want_fish, first, steps)
    else:
        want_fish, want_trace = orc.simulate(ocfg)
    try:
        with fsb.Engine(cfg, device=0, strategy=strategy, **kw) as eng:
            if upload is not None:
                eng.upload(upload)
                trace, bary, _ = eng.run(first, steps, barycentre=True)
            elif split:
                eng.init()
                a, ba, _ = eng.run(0, split, barycentre=True)
                b, bb, _ = eng.run(split, steps - split, barycentre=True)
                trace, bary = np.concatenate([a, b]), np.concatenate([ba, bb])
            else:
                eng.init()
                trace, bary, _ = eng.run(0, steps, barycentre=True)
            got = eng.download()
            used = eng.last_strategy()[0]
        want_b = np.array(orc.barycentre_sums(want_fish))
        # (an uploaded school may hold 1e300 or non-finite sums: compare the barycentre only when it is finite)
        bary_ok = (not np.all(np.isfinite(want_b))) or bool(np.all(np.abs(bary[-1] - want_b) <= 1e-12 * np.abs(want_b)))
        ok = got.tobytes() == want_fish.tobytes() and trace.tobytes() == want_trace.tobytes() and bary_ok
        err = ""
    except Exception as ex:  # noqa: BLE001
        ok, used, err = False, "?", repr(ex)
    counts[used] = counts.get(used, 0) + 1
    if not ok:
        bad += 1
        print(json.dumps({"case": case, "ok": False, "n": n, "steps": steps, "pond": pond, "step_base": step_base,
                          "weight_scale": wscale, "seed": cfg.seed, "strategy": strategy, "kw": kw, "split": split,
                          "uploaded": upload is not None, "first_step": first,
                          "error": err}), flush=True)
print(json.dumps({"cases": args.cases, "rng_seed": args.seed, "mismatches": bad, "strategies_run": counts,
                  "max_fish": args.max_fish, "seconds": round(time.time() - t0, 1)}), flush=True)
sys.exit(1 if bad else 0)
