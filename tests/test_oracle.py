"""Pin the oracle (oracle/fsb_oracle.c) against the reference's own outputs.

tests/golden/ was produced by the UNMODIFIED reference (oracle/_ref, see
tests/golden/make_golden.py).  Everything here runs on CPU.
"""
import os

import numpy as np
import pytest

import oracle
from conftest import bits, unhex


def cfg_of(d):
    return oracle.Config.make(**d)


def test_rng_known_answers(orc, golden_small):
    for args, want in golden_small["rng"]["bits"]:
        seed, fish, step, lane = (int(a) for a in args)
        assert orc.L.oracle_bits(seed, fish, step, lane) == int(want)


def test_objective_known_answers(orc, golden_small):
    for x, y, p, want in golden_small["rng"]["objective"]:
        assert bits(orc.objective(x, y, p)) == want
    # test_sim.cpp:33-38
    assert orc.objective(100.0, 100.0, 200.0) == 0.0
    assert orc.objective(103.0, 104.0, 200.0) == 5.0
    assert abs(orc.objective(0.0, 0.0, 200.0) - 100.0 * np.sqrt(2.0)) <= 1e-9


def test_eat_examples(orc, golden_small):
    cfg = oracle.Config.make()
    for name, case in golden_small["eat_examples"].items():
        rows = [[unhex(v) for v in r] for r in case["input"]]
        fish = np.array([tuple(r) for r in rows], dtype=oracle.FISH_DTYPE) if rows else \
            np.zeros(0, dtype=oracle.FISH_DTYPE)
        m = orc.eat(cfg, fish)
        assert bits(m) == case["max_diff"], name
        assert [bits(w) for w in fish["weight"]] == case["weights"], name
    # the literal assertions of test_sim.cpp:139-191
    ex = golden_small["eat_examples"]
    assert unhex(ex["three_fish"]["max_diff"]) == 6.0
    assert [unhex(w) for w in ex["three_fish"]["weights"]] == [5.0 + 6.0 / 6.0, 5.0, 5.0 + (7.0 - 9.0) / 6.0]
    assert unhex(ex["lone_fish"]["max_diff"]) == 2.5 and unhex(ex["lone_fish"]["weights"][0]) == 6.0
    assert unhex(ex["empty"]["max_diff"]) == -np.inf
    assert unhex(ex["no_improvement"]["max_diff"]) == 0.0


@pytest.mark.parametrize("name", [
    "baseline_1000x20", "defaults_10000x100_seed7", "walls_200x50", "band_500x60",
    "small_500x20_seed42", "one_fish_x30", "ragged_4097x7", "empty_0x5", "c4_4096x2000",
])
def test_small_runs_every_step(orc, golden_small, golden_states, name):
    g = golden_small["runs"][name]
    cfg = cfg_of(g["config"])
    fish = orc.init(cfg)
    assert f"{orc.checksum(fish):016x}" == g["init_checksum"]
    if name + "__init" in golden_states:
        assert fish.tobytes() == golden_states[name + "__init"].tobytes()
    for t in range(cfg.num_steps):
        orc.move(cfg, t, fish)
        m = orc.eat(cfg, fish)
        assert bits(m) == g["trace_hex"][t], f"{name} step {t} max_diff"
        assert f"{orc.checksum(fish):016x}" == g["step_checksums"][t], f"{name} step {t} checksum"
    if name + "__final" in golden_states:
        assert fish.tobytes() == golden_states[name + "__final"].tobytes()
    if cfg.num_fish:
        want = [unhex(v) for v in g["barycentre_fsum"]]
        got = orc.barycentre_sums(fish)
        for a, b in zip(got, want):
            assert abs(a - b) <= 1e-15 * abs(b)


def test_simulate_equals_phase_loop(orc, golden_small):
    g = golden_small["runs"]["defaults_10000x100_seed7"]
    cfg = cfg_of(g["config"])
    fish, trace = orc.simulate(cfg)
    assert f"{orc.checksum(fish):016x}" == g["step_checksums"][-1]
    assert [bits(v) for v in trace] == g["trace_hex"]
    # acceptance.cpp:63-102 digest of the reference defaults, seed 7
    assert f"{orc.checksum(fish):016x}" == "f7e6675cbe28eb38"


@pytest.mark.parametrize("name", ["C0_1e6x100", "C4_4096x100000"])
def test_baseline_configs(orc, golden_baseline, name):
    g = golden_baseline[name]
    cfg = cfg_of(g["config"])
    fish, trace = orc.simulate(cfg)
    assert f"{orc.checksum(fish):016x}" == g["final_checksum"]
    assert bits(trace[-1]) == g["trace_last_hex"]
    if g["trace_hex"]:
        assert [bits(v) for v in trace] == g["trace_hex"]
    if g.get("trace_every_1000_hex"):
        assert [bits(v) for v in trace[999::1000]] == g["trace_every_1000_hex"]
    want = [unhex(v) for v in g["barycentre_fsum"]]
    got = orc.barycentre_sums(fish)
    for a, b in zip(got, want):
        assert abs(a - b) <= 1e-14 * abs(b)


def test_sampled_replay_matches_whole_run(orc):
    """One fish replayed alone with the run's trace equals its state in the run."""
    cfg = oracle.baseline_config(3001, 15)
    fish, trace = orc.simulate(cfg)
    idx = [0, 1, 17, 1500, 2999, 3000]
    assert orc.replay(cfg, idx, trace).tobytes() == fish[idx].tobytes()
    cfg = oracle.Config.make(num_fish=500, num_steps=60, seed=42, step_base=10.0)  # clamp-heavy
    fish, trace = orc.simulate(cfg)
    assert orc.replay(cfg, range(500), trace).tobytes() == fish.tobytes()


def test_sharded_oracle_matches_whole(orc):
    """Global-index RNG keys make a contiguous shard reproduce the same fish."""
    cfg = oracle.baseline_config(1001, 5)
    whole = orc.init(cfg)
    parts = [orc.init(cfg, first=a, n=b - a) for a, b in ((0, 333), (333, 700), (700, 1001))]
    assert np.concatenate(parts).tobytes() == whole.tobytes()
    for t in range(cfg.num_steps):
        orc.move(cfg, t, whole)
        off = 0
        for p in parts:
            orc.move(cfg, t, p, first=off)
            off += len(p)
    assert np.concatenate(parts).tobytes() == whole.tobytes()


@pytest.mark.skipif(not os.path.exists(oracle.REF_SO) and not os.path.isdir(oracle.REF_INCLUDE),
                    reason="reference not available")
@pytest.mark.parametrize("kw", [
    dict(num_fish=777, num_steps=33, seed=5, pond_size=200.0, weight_scale=1.0, step_base=0.1),
    dict(num_fish=2048, num_steps=40, seed=9, pond_size=3.0, weight_scale=4.0, step_base=2.5),
    dict(num_fish=64, num_steps=200, seed=123456789, pond_size=1e3, weight_scale=1.5, step_base=0.01),
])
def test_oracle_equals_reference(orc, kw):
    ref = oracle.Reference()
    cfg = oracle.Config.make(**kw)
    f1, t1 = orc.simulate(cfg)
    f2, t2, _ = ref.simulate(cfg)
    assert f1.tobytes() == f2.tobytes()
    assert t1.tobytes() == t2.tobytes()
