"""Parity of the sm_100a engine with the oracle and the reference's golden
vectors, through the C-ABI.  Requires a B200 (pytest -m gpu).

Bar: bit-exact positions, weights, objectives and max_diff trace (fp64, no
FMA); barycentre sums within 1e-12 relative of the compensated oracle.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
import paper_2507_20173_b200 as fsb
from conftest import ROOT, bits, unhex

pytestmark = pytest.mark.gpu

BARY_RTOL = 1e-12  # north_star: barycentre within 1e-12 relative in fp64


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if fsb.device_count() == 0:
        pytest.fail("no CUDA device: the GPU tests must run on a B200")


def ocfg(cfg: fsb.SimConfig):
    return oracle.Config.make(num_fish=cfg.num_fish, pond_size=cfg.pond_size,
                              weight_scale=cfg.weight_scale, num_steps=cfg.num_steps, seed=cfg.seed,
                              step_base=cfg.step_base)


def rel_ok(got, want, rtol=BARY_RTOL):
    got, want = np.asarray(got), np.asarray(want)
    return np.all(np.abs(got - want) <= rtol * np.abs(want))


STRATS = ["stream", "persistent", "grid"]


def make(cfg, strategy="auto", **kw):
    return fsb.Engine(cfg, device=0, strategy=strategy, **kw)


@pytest.mark.parametrize("strategy", STRATS)
@pytest.mark.parametrize("name", [
    "baseline_1000x20", "defaults_10000x100_seed7", "walls_200x50", "band_500x60",
    "small_500x20_seed42", "one_fish_x30", "ragged_4097x7", "c4_4096x2000",
])
def test_golden_runs_every_step(golden_small, golden_states, name, strategy):
    """Per-step checksum + max_diff of the reference, one run() call per step."""
    g = golden_small["runs"][name]
    cfg = fsb.SimConfig(**g["config"])
    steps = min(cfg.num_steps, 200)
    with make(cfg, strategy) as eng:
        eng.init()
        assert f"{eng.checksum():016x}" == g["init_checksum"]
        for t in range(steps):
            trace, _, _ = eng.run(t, 1)
            assert bits(trace[0]) == g["trace_hex"][t], f"step {t}"
            assert f"{eng.checksum():016x}" == g["step_checksums"][t], f"step {t}"
        if steps < cfg.num_steps:
            trace, _, _ = eng.run(steps, cfg.num_steps - steps)
            assert [bits(v) for v in trace] == g["trace_hex"][steps:]
        assert f"{eng.checksum():016x}" == g["step_checksums"][-1]
        if name + "__final" in golden_states:
            assert eng.download().tobytes() == golden_states[name + "__final"].tobytes()


@pytest.mark.parametrize("strategy", STRATS)
@pytest.mark.parametrize("alternate", [True, False])
@pytest.mark.parametrize("n,t", [(1, 9), (2, 9), (3, 9), (31, 9), (33, 9), (255, 7), (1025, 7),
                                 (2 * 1024 + 1, 6), (12289, 5), (16384, 5), (65536, 3)])
def test_sizes_bit_exact(orc, n, t, strategy, alternate):
    cfg = fsb.baseline_config(n, t)
    want_fish, want_trace = orc.simulate(ocfg(cfg))
    with make(cfg, strategy, alternate=alternate) as eng:
        try:
            trace, bary, _ = eng.simulate(barycentre=True)
        except fsb.FsbError as e:
            # the persistent cluster holds at most 16 CTAs x 2048 fish; above that
            # an explicit persistent request is refused (AUTO falls back to stream)
            assert strategy == "persistent" and n > 16384 and e.code == 6
            return
        got = eng.download()
    assert got.tobytes() == want_fish.tobytes()
    assert trace.tobytes() == want_trace.tobytes()
    assert rel_ok(bary[-1], orc.barycentre_sums(want_fish))


KERNELS = {"static": dict(static_tiles=True), "dynamic": dict(dynamic_tiles=True), "bulk": dict(bulk=True),
           "ws": dict(ws_tiles=True)}


@pytest.mark.parametrize("n,t", [(1, 5), (513, 5), (70_001, 6), (1_000_000, 4), (3_000_001, 3)])
@pytest.mark.parametrize("alternate", [True, False])
@pytest.mark.parametrize("kernel", list(KERNELS))
def test_step_kernel_variants_bit_exact(orc, n, t, alternate, kernel):
    """Every compact-state step kernel at every size: the static-chunk LDG
    kernel, the claimed-tile LDG kernel (FSB_FLAG_DYNAMIC_TILES) and the
    cp.async.bulk ring (FSB_FLAG_FORCE_BULK) and the warp-specialised TMA
    kernel (FSB_FLAG_WS_TILES)."""
    cfg = fsb.baseline_config(n, t)
    want_fish, want_trace = orc.simulate(ocfg(cfg))
    with make(cfg, "stream", alternate=alternate, **KERNELS[kernel]) as eng:
        trace, bary, _ = eng.simulate(barycentre=True)
        got = eng.download()
    assert got.tobytes() == want_fish.tobytes()
    assert trace.tobytes() == want_trace.tobytes()
    assert rel_ok(bary[-1], orc.barycentre_sums(want_fish))


@pytest.mark.parametrize("strategy", STRATS)
def test_per_step_barycentre(orc, strategy):
    cfg = fsb.SimConfig(num_fish=12000, pond_size=50.0, weight_scale=2.0, num_steps=12, seed=99,
                        step_base=0.9)
    fish = orc.init(ocfg(cfg))
    want = []
    for t in range(cfg.num_steps):
        orc.move(ocfg(cfg), t, fish)
        orc.eat(ocfg(cfg), fish)
        want.append(orc.barycentre_sums(fish))
    with make(cfg, strategy) as eng:
        _, bary, _ = eng.simulate(barycentre=True)
        sums, xy = eng.barycentre()
    assert rel_ok(bary, np.array(want))
    assert rel_ok(sums, want[-1])
    assert rel_ok(xy, [want[-1][0] / want[-1][2], want[-1][1] / want[-1][2]], 1e-12)


@pytest.mark.parametrize("strategy", STRATS)
def test_barycentre_after_max_only_run(orc, strategy):
    """A run without the per-step sums (the persistent kernel then reduces the
    max only) followed by the barycentre query of the final state."""
    cfg = fsb.baseline_config(4096, 30)
    want_fish, want_trace = orc.simulate(ocfg(cfg))
    with make(cfg, strategy) as eng:
        eng.init()
        trace, bary, _ = eng.run(0, 30, barycentre=False)
        assert bary is None and trace.tobytes() == want_trace.tobytes()
        sums, _ = eng.barycentre()
        assert rel_ok(sums, orc.barycentre_sums(want_fish))
        assert bits(eng.eat().max_diff) == bits(orc.eat(ocfg(cfg), want_fish))


def test_large_stream_bit_exact(orc):
    cfg = fsb.SimConfig(num_fish=1_000_003, pond_size=200.0, weight_scale=10.0, num_steps=25, seed=7,
                        step_base=1.0)
    want_fish, want_trace = orc.simulate(ocfg(cfg))
    with make(cfg, "stream") as eng:
        trace, bary, _ = eng.simulate(barycentre=True)
        got = eng.download()
    assert got.tobytes() == want_fish.tobytes()
    assert trace.tobytes() == want_trace.tobytes()
    assert rel_ok(bary[-1], orc.barycentre_sums(want_fish))


def test_phase_api_move_then_eat(orc):
    """move_phase / eat_phase as separate calls: the state after each phase."""
    cfg = fsb.SimConfig(num_fish=5001, num_steps=6, seed=3)
    oc = ocfg(cfg)
    fish = orc.init(oc)
    with make(cfg) as eng:
        eng.init()
        for t in range(cfg.num_steps):
            orc.move(oc, t, fish)
            eng.move(t)
            assert eng.download().tobytes() == fish.tobytes(), f"after move {t}"
            m = orc.eat(oc, fish)
            r = eng.eat()
            assert bits(r.max_diff) == bits(m)
            assert eng.download().tobytes() == fish.tobytes(), f"after eat {t}"


def test_host_school_phase_functions(orc):
    """The reference call shapes on a host School (sim.hpp:84,110)."""
    cfg = fsb.SimConfig(num_fish=700, num_steps=5, seed=11)
    oc = ocfg(cfg)
    ex = fsb.GpuExecutor()
    school = fsb.init_school(cfg, ex)
    want = orc.init(oc)
    assert school.fishes.tobytes() == want.tobytes()
    for t in range(cfg.num_steps):
        fsb.move_phase(school, cfg, t, ex)
        r = fsb.eat_phase(school, cfg, ex)
        orc.move(oc, t, want)
        assert bits(r.max_diff) == bits(orc.eat(oc, want))
        assert school.fishes.tobytes() == want.tobytes()
    res = fsb.simulate(cfg, ex)
    assert fsb.checksum(res.school) == fsb.checksum(school)
    ex.close()


def test_eat_examples_from_reference_tests(golden_small):
    """test_sim.cpp:139-191 hand-built schools (current_objective != objective(x,y))."""
    cfg = fsb.SimConfig()
    ex = fsb.GpuExecutor()
    for name, case in golden_small["eat_examples"].items():
        rows = [tuple(unhex(v) for v in r) for r in case["input"]]
        school = fsb.School(np.array(rows, dtype=fsb.FISH_DTYPE) if rows else None)
        r = fsb.eat_phase(school, cfg, ex)
        assert bits(r.max_diff) == case["max_diff"], name
        assert [bits(w) for w in school.fishes["weight"]] == case["weights"], name
        # x, y, prev, cur untouched
        for k, fld in enumerate(("x", "y")):
            assert [bits(v) for v in school.fishes[fld]] == [r_[k] for r_ in case["input"]]
    ex.close()


@pytest.mark.parametrize("strategy", STRATS)
def test_upload_inconsistent_then_run(orc, strategy):
    """An uploaded school whose current_objective is arbitrary (explicit-cur path)."""
    rng = np.random.default_rng(5)
    n = 3001
    fish = np.zeros(n, dtype=oracle.FISH_DTYPE)
    fish["x"] = rng.uniform(0, 200, n)
    fish["y"] = rng.uniform(0, 200, n)
    fish["weight"] = rng.uniform(1, 20, n)
    fish["prev_objective"] = rng.uniform(0, 150, n)
    fish["current_objective"] = rng.uniform(0, 150, n)
    cfg = fsb.SimConfig(num_fish=n, num_steps=4, seed=17)
    oc = ocfg(cfg)
    with make(cfg, strategy) as eng:
        eng.upload(fish)
        assert eng.download().tobytes() == fish.tobytes()
        want = fish.copy()
        m = orc.eat(oc, want)  # eat first (uses the explicit cur)
        assert bits(eng.eat().max_diff) == bits(m)
        assert eng.download().tobytes() == want.tobytes()
        trace, _, _ = eng.run(0, 4)
        want_trace = orc.run(oc, want, 0, 4)
        assert trace.tobytes() == want_trace.tobytes()
        assert eng.download().tobytes() == want.tobytes()
    with make(cfg, strategy) as eng:  # run straight after the upload
        eng.upload(fish)
        want = fish.copy()
        trace, _, _ = eng.run(0, 4)
        assert trace.tobytes() == orc.run(oc, want, 0, 4).tobytes()
        assert eng.download().tobytes() == want.tobytes()


@pytest.mark.parametrize("strategy", ["stream", "grid"])
@pytest.mark.parametrize("kernel", list(KERNELS))
@pytest.mark.parametrize("n,t", [(4097, 9), (300_001, 5)])
def test_in_range_mode_equals_checked(orc, strategy, kernel, n, t):
    """The step kernels with the fp64 operand guards elided (in-range mode, the
    default for an init'd school) and evaluated (FSB_FLAG_CHECKED) agree with
    the oracle bit for bit."""
    cfg = fsb.baseline_config(n, t)
    want_fish, want_trace = orc.simulate(ocfg(cfg))
    for checked in (False, True):
        with make(cfg, strategy, checked=checked, **KERNELS[kernel]) as eng:
            trace, _, _ = eng.simulate(barycentre=False)
            assert trace.tobytes() == want_trace.tobytes(), checked
            assert eng.download().tobytes() == want_fish.tobytes(), checked


def _hostile(kind, n, rng):
    fish = np.zeros(n, dtype=oracle.FISH_DTYPE)
    fish["x"] = rng.uniform(0, 200, n)
    fish["y"] = rng.uniform(0, 200, n)
    fish["weight"] = rng.uniform(1, 20, n)
    o = np.sqrt((fish["x"] - 100) ** 2 + (fish["y"] - 100) ** 2)
    fish["prev_objective"] = o
    fish["current_objective"] = o
    k = slice(0, n, 7)
    if kind == "denormal_prev":
        fish["prev_objective"][k] = 5e-310
    elif kind == "huge_weight":
        fish["weight"][k] = 1e300
    elif kind == "outside_pond":
        fish["x"][k] = -3.0
        fish["y"][1::7] = 1e6
    elif kind == "centre_and_ties":
        fish["x"][k] = 100.0
        fish["y"][k] = 100.0
        fish["prev_objective"][k] = 0.0
        fish["current_objective"][k] = 0.0
        fish["prev_objective"][1::7] = fish["current_objective"][1::7]
    elif kind == "negative_zero":
        fish["prev_objective"][k] = -0.0
    return fish


@pytest.mark.parametrize("strategy", ["stream", "persistent"])
@pytest.mark.parametrize("kind", ["denormal_prev", "huge_weight", "outside_pond", "centre_and_ties",
                                  "negative_zero"])
def test_upload_out_of_range_state(orc, strategy, kind):
    """States outside the in-range mode's bounds (fsb_math.cuh) take the guarded
    kernels and still match the oracle; in-range edge values (fish at the pond
    centre, prev == cur) are exact in either mode."""
    n = 5003
    fish = _hostile(kind, n, np.random.default_rng(23))
    cfg = fsb.SimConfig(num_fish=n, num_steps=5, seed=29)
    oc = ocfg(cfg)
    for checked in (False, True):
        with make(cfg, strategy, checked=checked) as eng:
            eng.upload(fish)
            want = fish.copy()
            trace, _, _ = eng.run(0, 5)
            assert trace.tobytes() == orc.run(oc, want, 0, 5).tobytes(), (kind, checked)
            assert eng.download().tobytes() == want.tobytes(), (kind, checked)


@pytest.mark.parametrize("over", [dict(pond_size=1e-130), dict(pond_size=1e160), dict(step_base=1e-125),
                                  dict(step_base=1e200), dict(weight_scale=1e160)])
def test_config_outside_in_range_bounds(orc, over):
    """Configurations outside the in-range bounds run the guarded kernels."""
    kw = dict(num_fish=20_001, num_steps=6, seed=31)
    kw.update(over)
    cfg = fsb.SimConfig(**kw)
    want_fish, want_trace = orc.simulate(ocfg(cfg))
    with make(cfg, "stream") as eng:
        trace, _, _ = eng.simulate(barycentre=False)
        assert trace.tobytes() == want_trace.tobytes()
        assert eng.download().tobytes() == want_fish.tobytes()


@pytest.mark.parametrize("kernel", list(KERNELS))
def test_grid_override_bit_exact(orc, kernel):
    """fsb_engine_set_grid (the CTA-count sweep): any grid, including more CTAs
    than 64-pair blocks, gives the oracle's state and trace."""
    cfg = fsb.baseline_config(100_003, 6)
    want_fish, want_trace = orc.simulate(ocfg(cfg))
    with make(cfg, "stream", **KERNELS[kernel]) as eng:
        auto = eng.grid()
        for ctas in (1, 7, 148, 1000, 5000, 0):
            eng.set_grid(ctas)
            assert eng.grid()[0] == (ctas or auto[0])
            trace, _, _ = eng.simulate(barycentre=False)
            assert trace.tobytes() == want_trace.tobytes(), ctas
            assert eng.download().tobytes() == want_fish.tobytes(), ctas
        with pytest.raises(fsb.FsbError):
            eng.set_grid(-1)


@pytest.mark.parametrize("groups", [1, 3, 64, 4096, 0])
def test_tile_groups_bit_exact(orc, groups):
    """fsb_engine_set_tile_groups (the gpu-exp2 granularity sweep): any claimed
    tile size gives the oracle's state and trace."""
    cfg = fsb.baseline_config(300_001, 5)
    want_fish, want_trace = orc.simulate(ocfg(cfg))
    with make(cfg, "stream", dynamic_tiles=True) as eng:
        eng.set_tile_groups(groups)
        trace, _, _ = eng.simulate(barycentre=False)
        assert trace.tobytes() == want_trace.tobytes()
        assert eng.download().tobytes() == want_fish.tobytes()
        with pytest.raises(fsb.FsbError):
            eng.set_tile_groups(-1)


def test_dynamic_tiles_explicit_cur_and_repeatable(orc):
    """The claimed-tile kernel on its explicit-cur instantiation (first step
    after an inconsistent upload), and bitwise repeatability of its sums
    (tile partials folded in tile order, whichever warp claimed them)."""
    rng = np.random.default_rng(9)
    n = 200_003
    fish = np.zeros(n, dtype=oracle.FISH_DTYPE)
    fish["x"] = rng.uniform(0, 200, n)
    fish["y"] = rng.uniform(0, 200, n)
    fish["weight"] = rng.uniform(1, 2, n)
    fish["prev_objective"] = rng.uniform(0, 150, n)
    fish["current_objective"] = rng.uniform(0, 150, n)
    cfg = fsb.SimConfig(num_fish=n, num_steps=6, seed=41, weight_scale=1.0, pond_size=200.0, step_base=0.1)
    outs = []
    for _ in range(2):
        with make(cfg, "stream", dynamic_tiles=True) as eng:
            eng.upload(fish)
            want = fish.copy()
            trace, bary, _ = eng.run(0, 6, barycentre=True)
            assert trace.tobytes() == orc.run(ocfg(cfg), want, 0, 6).tobytes()
            assert eng.download().tobytes() == want.tobytes()
            outs.append(bary.tobytes())
    assert outs[0] == outs[1]


@pytest.mark.parametrize("flat", [False, True])
@pytest.mark.parametrize("n,t", [(1, 4), (1025, 7), (100_003, 6), (2_000_001, 3)])
def test_grid_strategy_both_exchanges(orc, flat, n, t):
    """FSB_STRATEGY_GRID with the cluster-reduced exchange (default) and the
    flat counter barrier (FSB_FLAG_FLAT_GRID): trace and state bit-exact, the
    per-step barycentre within tolerance, and repeatable bit for bit."""
    cfg = fsb.baseline_config(n, t)
    want_fish, want_trace = orc.simulate(ocfg(cfg))
    outs = []
    for _ in range(2):
        with make(cfg, "grid", flat_grid=flat) as eng:
            trace, bary, _ = eng.simulate(barycentre=True)
            assert trace.tobytes() == want_trace.tobytes()
            assert eng.download().tobytes() == want_fish.tobytes()
            assert rel_ok(bary[-1], orc.barycentre_sums(want_fish))
            outs.append(bary.tobytes())
    assert outs[0] == outs[1]


def test_long_stream_run_is_chunked(orc):
    """A run longer than one graph (1024 steps) goes through several graphs."""
    cfg = fsb.baseline_config(20_000, 2500)
    want_fish, want_trace = orc.simulate(ocfg(cfg))
    with make(cfg, "stream") as eng:
        trace, _, _ = eng.simulate(barycentre=False)
        assert eng.last_launches() == 2500 + 3  # 3 graphs, each with its trailing eat
        assert trace.tobytes() == want_trace.tobytes()
        assert eng.download().tobytes() == want_fish.tobytes()


@pytest.mark.parametrize("strategy,kw", [("stream", {}), ("stream", {"ws_tiles": True}), ("grid", {}),
                                         ("persistent", {})])
def test_run_split_equals_whole(orc, strategy, kw):
    """A run cut into pieces equals the whole run (each piece ends with its
    trailing eat; the persistent kernels restart their per-step state)."""
    cfg = fsb.baseline_config(4096 if strategy == "persistent" else 40_000, 12)
    with make(cfg, strategy, **kw) as a, make(cfg, strategy, **kw) as b:
        a.init()
        b.init()
        ta, _, _ = a.run(0, 12)
        tb1, _, _ = b.run(0, 5)
        tb2, _, _ = b.run(5, 7)
        tb3, _, _ = b.run(12, 0)
        assert ta.tobytes() == np.concatenate([tb1, tb2, tb3]).tobytes()
        assert a.download().tobytes() == b.download().tobytes()


@pytest.mark.parametrize("strategy", STRATS + ["ws"])
@pytest.mark.parametrize("first", [2**32 + 3, 2**63 + 7, 2**64 - 4])
def test_large_step_index(orc, strategy, first):
    """The step index is a full u64 RNG word (rng.hpp:34-36): runs starting
    anywhere up to just below kInitStep = 2^64-1 match the oracle."""
    n = 4096 if strategy == "persistent" else 50_001
    cfg = fsb.baseline_config(n, 3)
    fish = orc.init(ocfg(cfg))
    want_trace = orc.run(ocfg(cfg), fish, first, 3)
    kw = {"ws_tiles": True} if strategy == "ws" else {}
    with make(cfg, "stream" if strategy == "ws" else strategy, **kw) as eng:
        eng.init()
        trace, _, _ = eng.run(first, 3)
        assert trace.tobytes() == want_trace.tobytes()
        assert eng.download().tobytes() == fish.tobytes()


@pytest.mark.parametrize("strategy", STRATS)
@pytest.mark.parametrize("seed", [0, 1, 2**63, 2**64 - 1])
def test_extreme_seeds(orc, strategy, seed):
    """Seed words at the ends of the u64 range (the first fold_in operand)."""
    n = 3000 if strategy == "persistent" else 30_001
    cfg = fsb.SimConfig(num_fish=n, num_steps=6, seed=seed, pond_size=200.0, weight_scale=1.0, step_base=0.1)
    want_fish, want_trace = orc.simulate(ocfg(cfg))
    with make(cfg, strategy) as eng:
        trace, _, _ = eng.simulate(barycentre=False)
        assert trace.tobytes() == want_trace.tobytes()
        assert eng.download().tobytes() == want_fish.tobytes()


def test_empty_school():
    cfg = fsb.SimConfig(num_fish=0, num_steps=4)
    with make(cfg) as eng:
        eng.init()
        trace, bary, _ = eng.run(0, 4, barycentre=True)
        assert np.all(trace == -np.inf)
        assert eng.eat().max_diff == -np.inf
        assert eng.checksum() == fsb.kChecksumEmpty
        assert eng.download().shape == (0,)


def test_repeatable_bitwise():
    cfg = fsb.baseline_config(300_001, 10)
    outs = []
    for _ in range(2):
        with make(cfg, "stream") as eng:
            trace, bary, _ = eng.simulate(barycentre=True)
            outs.append((trace.tobytes(), bary.tobytes(), eng.checksum()))
    assert outs[0] == outs[1]


def test_time_step_kernels_keeps_state_valid(orc):
    cfg = fsb.baseline_config(200_000, 6)
    fish = orc.init(ocfg(cfg))
    orc.run(ocfg(cfg), fish, 0, 6)
    with make(cfg, "stream") as eng:
        eng.init()
        ms = eng.time_step_kernels(0, 6)
        assert ms.shape == (6,) and np.all(ms > 0)
        assert eng.download().tobytes() == fish.tobytes()


@pytest.mark.parametrize("kernel", ["static", "dynamic", "ws"])
def test_force_nccl_world1(orc, kernel):
    """The NCCL exchange path (allgather in the graph) on one rank, with both
    step kernels (the claimed-tile one is the multi-GPU bench's: 1e7 per GPU)."""
    cfg = fsb.baseline_config(100_000, 8)
    uid = fsb.nccl_unique_id()
    want_fish, want_trace = orc.simulate(ocfg(cfg))
    with make(cfg, "stream", nccl_unique_id=uid, force_nccl=True,
              **KERNELS[kernel]) as eng:
        trace, _, _ = eng.simulate(barycentre=False)
        assert trace.tobytes() == want_trace.tobytes()
        assert eng.download().tobytes() == want_fish.tobytes()
        eng.move(8)
        orc.move(ocfg(cfg), 8, want_fish)
        assert bits(eng.eat().max_diff) == bits(orc.eat(ocfg(cfg), want_fish))


def test_nccl_before_torch_import():
    """An NCCL engine created before torch is imported must not shadow the NCCL
    torch links (libnccl.so.2 is shared by soname): a fresh process creates a
    FORCE_NCCL engine, then imports torch and runs a CUDA op."""
    code = ("import paper_2507_20173_b200 as fsb\n"
            "cfg = fsb.baseline_config(1000, 2)\n"
            "e = fsb.Engine(cfg, nccl_unique_id=fsb.nccl_unique_id(), force_nccl=True)\n"
            "e.simulate()\n"
            "import torch\n"
            "assert torch.ones(4, device='cuda').sum().item() == 4.0\n"
            "e.close()\n")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]


@pytest.mark.parametrize("n,t,kw", [(100_001, 9, {}), (100_001, 9, {"dynamic_tiles": True}),
                                    (100_001, 9, {"ws_tiles": True}), (4096, 30, {}),
                                    (1, 5, {}), (0, 3, {})])
def test_peer_exchange_world1(orc, n, t, kw):
    """FSB_FLAG_PEER_EXCHANGE on one rank: the step kernel pushes its partial
    into the (self-mapped) peer window and the next kernel acquires the epoch
    flag -- the same code path the NVLink exchange takes across GPUs."""
    cfg = fsb.baseline_config(n, t)
    want_fish, want_trace = orc.simulate(ocfg(cfg))
    with make(cfg, "auto", peer=True, **kw) as eng:
        trace, bary, _ = eng.simulate(barycentre=True)
        assert trace.tobytes() == want_trace.tobytes()
        assert eng.download().tobytes() == want_fish.tobytes()
        if n:
            assert rel_ok(bary[-1], orc.barycentre_sums(want_fish))
            sums, _ = eng.barycentre()
            assert rel_ok(sums, orc.barycentre_sums(want_fish))
        # phases and the eager per-kernel timing path advance the same epochs
        eng.move(t)
        orc.move(ocfg(cfg), t, want_fish)
        assert bits(eng.eat().max_diff) == bits(orc.eat(ocfg(cfg), want_fish))
        eng.time_step_kernels(t + 1, 3)
        orc.run(ocfg(cfg), want_fish, t + 1, 3)
        tr, _, _ = eng.run(t + 4, 2)
        assert tr.tobytes() == orc.run(ocfg(cfg), want_fish, t + 4, 2).tobytes()
        assert eng.download().tobytes() == want_fish.tobytes()


@pytest.mark.parametrize("name", ["C0_1e6x100", "C1_1e7x100", "C4_4096x100000", "C2_1e8x50"])
def test_baseline_configs_match_reference_digests(golden_baseline, orc, name):
    if name not in golden_baseline:
        pytest.skip("digest not generated")
    g = golden_baseline[name]
    cfg = fsb.SimConfig(**g["config"])
    with make(cfg) as eng:
        trace, bary, _ = eng.simulate(barycentre=True)
        assert f"{eng.checksum():016x}" == g["final_checksum"]
    assert bits(trace[-1]) == g["trace_last_hex"]
    if g.get("trace_hex"):
        assert [bits(v) for v in trace] == g["trace_hex"]
    if g.get("trace_every_1000_hex"):
        assert [bits(v) for v in trace[999::1000]] == g["trace_every_1000_hex"]
    assert rel_ok(bary[-1], [unhex(v) for v in g["barycentre_fsum"]])


@pytest.mark.parametrize("name", ["C0_1e6x100", "C1_1e7x100", "C4_4096x100000"])
def test_baseline_configs_every_step(golden_baseline, name):
    """SURVEY 8(d) correctness gates: the reference checksum after every step
    (C0, C1) or every 1000th step (C4), the engine run chunk by chunk."""
    g = golden_baseline[name]
    every = g["step_checksums_every"]
    cfg = fsb.SimConfig(**g["config"])
    with make(cfg) as eng:
        eng.init()
        assert f"{eng.checksum():016x}" == g["init_checksum"]
        for k, want in enumerate(g["step_checksums"]):
            eng.run(k * every, every)
            assert f"{eng.checksum():016x}" == want, f"after step {(k + 1) * every - 1}"


@pytest.mark.parametrize("mode", ["nccl", "peer"])
def test_cpp_multi_gpu_example(golden_baseline, mode):
    """examples/simulate_multi_gpu (one host thread per GPU, C++ drop-in) on the
    GPUs present, exchanging by NCCL or by peer windows connected within the
    process: the chained shard checksum equals the reference C0 digest."""
    exe = os.path.join(ROOT, "examples", "simulate_multi_gpu")
    if not os.path.exists(exe):
        subprocess.run(["make", "-s", "-C", os.path.dirname(exe)], check=True)
    g = golden_baseline["C0_1e6x100"]
    r = subprocess.run([exe, str(fsb.device_count()), "1000000", "100", "7", mode], capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr
    digest, last, _ = r.stdout.split()
    assert digest == g["final_checksum"]
    assert bits(float(last)) == g["trace_last_hex"]


def test_cpp_dropin_suite():
    """tests/cpp/test_gpu_sim: the reference's test_sim.cpp cases via fsb::gpu."""
    exe = os.path.join(ROOT, "tests", "cpp", "test_gpu_sim")
    if not os.path.exists(exe):
        subprocess.run(["make", "-s", "-C", os.path.dirname(exe)], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout


def test_cpp_dropin_reference_types():
    """tests/cpp/test_dropin_reftypes: INTEGRATION.md section 1 as a reference user
    writes it -- the reference's own fsb/sim.hpp types (FSB_GPU_USE_REFERENCE_TYPES)
    through fsb::gpu, checked against the reference's parfor path: init_school,
    move/eat step by step, test_sim.cpp:217-225 and acceptance.cpp:63-102
    criterion 1 for every GPU strategy.  Built where /root/reference exists
    (build()); the binary travels to the GPU box."""
    exe = os.path.join(ROOT, "tests", "cpp", "test_dropin_reftypes")
    if not os.path.exists(exe):
        pytest.skip("built only where the reference headers exist (run build() in the dev container)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "4 cases, 0 failed" in r.stdout, r.stdout


def test_fast_math_selftest():
    """The guarded fast fp64 paths of the step kernel equal __ddiv_rn / __dsqrt_rn
    bit-for-bit on 2^27 operands (raw bit patterns incl. NaN/inf/subnormals, and
    the simulation's ranges), and their guards never fail on in-range values."""
    from paper_2507_20173_b200 import _native as N

    out = np.zeros(4, dtype=np.uint64)
    for seed in (1, 2):
        N.check(N.lib().fsb_selftest_fast_math(0, 1 << 26, seed, out.ctypes.data))
        assert out.tolist() == [0, 0, 0, 0], out


def test_cli_simulate_record(tmp_path, capsys):
    """`simulate` with the reference CLI's flags (cli.hpp:179-207): the record's
    checksum is the reference digest of SimConfig{fish 1e4, steps 100, seed 7}
    (acceptance.cpp:63-102 / SURVEY App. C) and the row is in the reference schema."""
    from paper_2507_20173_b200 import records
    from paper_2507_20173_b200.__main__ import main as cli_main

    out = tmp_path / "r.csv"
    assert cli_main(["simulate", "--fish", "10000", "--steps", "100", "--seed", "7", "--out", str(out)]) == 0
    recs = records.read_csv(out.read_text())
    assert len(recs) == 1 and recs[0].checksum == 0xF7E6675CBE28EB38
    assert recs[0].construct == "gpu" and recs[0].seconds_eat <= recs[0].seconds_total
    # Exp 1 at 2e6 fish: 1/8 of the SMs .. 8 CTAs per SM spans 6..434 fish per thread
    assert cli_main(["gpuexp", "--exp", "1", "--fish", "2000000", "--steps", "10", "--reps", "2", "--warmup", "1",
                     "--out", str(out)]) == 0
    exp1 = records.read_csv(out.read_text())
    assert len({r.checksum for r in exp1}) == 1 and not any(r.failed() for r in exp1)
    assert len(exp1) == 14 and len({r.chunk for r in exp1}) >= 5  # the fish-per-thread axis
    assert all(r.experiment == "gpu-exp1" and r.schedule == "graph" for r in exp1)
    # Exp 2 (bench.hpp:103-127 analogue): static / dynamic tiles of 1..256 groups / TMA / bulk ring
    assert cli_main(["gpuexp", "--exp", "2", "--fish", "1000001", "--steps", "6", "--reps", "1", "--warmup", "1",
                     "--out", str(out)]) == 0
    exp2 = records.read_csv(out.read_text())
    assert len(exp2) == 12 and len({r.checksum for r in exp2}) == 1 and not any(r.failed() for r in exp2)
    assert {r.schedule for r in exp2} == {"static", "dynamic", "tma-ws", "bulk-ring"}
    assert len({r.chunk for r in exp2 if r.schedule == "dynamic"}) >= 6  # the granularity axis
    assert cli_main(["gpuexp", "--exp", "3", "--fish", "4096", "--steps", "50", "--reps", "2", "--warmup", "1",
                     "--out", str(out)]) == 0
    text = out.read_text()
    recs = records.read_csv(text)
    assert len({r.checksum for r in recs}) == 1 and not any(r.failed() for r in recs)
    exp3 = [r for r in recs if r.experiment == "gpu-exp3"]
    assert {r.construct for r in exp3} == {"gpu-keyslot", "gpu-lastcta", "gpu-nccl", "gpu-peer", "gpu-smem-counter",
                                          "gpu-cluster-slots", "gpu-flat-counter", "gpu-redux-dsmem"}
    assert len(exp3) == 16 and all(r.threads == 1 for r in exp3)
    assert {r.schedule for r in exp3} == {"graph", "grid", "cluster"}
    # Exp 3 rows carry a measured eat region (bench.hpp:132-148), valid for the reference's validate_records
    assert all(0.0 < r.seconds_eat < r.seconds_total for r in recs)
    ref = os.path.join(ROOT, "oracle", "_ref", "libfsbref.so")
    if os.path.exists(ref):
        import ctypes

        L = oracle.Reference().L
        L.ref_read_csv.restype = ctypes.c_int
        L.ref_read_csv.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_int), ctypes.c_char_p, ctypes.c_int]
        issues = ctypes.c_int(-1)
        err = ctypes.create_string_buffer(256)
        assert L.ref_read_csv(text.encode(), ctypes.byref(issues), err, 256) == len(recs), err.value
        assert issues.value == 0


def test_gather_matches_download(orc):
    cfg = fsb.baseline_config(100_001, 3)
    with make(cfg) as eng:
        eng.simulate(barycentre=False)
        full = eng.download()
        idx = np.array([0, 5, 100_000, 77, 5], dtype=np.uint64)
        assert eng.gather(idx).tobytes() == full[idx.astype(np.int64)].tobytes()


def test_c3_billion_fish(golden_baseline, orc):
    """C3 (1e9 fish x 20 steps, 32 GB of state): the max_diff trace against the
    reference's, 1,000,000 sampled fish replayed on the CPU from their initial state
    with the GPU trace, the final checksum streamed over all 40 GB
    of Fish bytes, and the barycentre."""
    cfg = fsb.baseline_config(10**9, 20)
    g = golden_baseline.get("C3_1e9x20")
    with make(cfg) as eng:
        trace, bary, _ = eng.simulate(barycentre=True)
        if g:
            assert [bits(v) for v in trace] == g["trace_hex"]
        rng = np.random.default_rng(3)
        idx = np.unique(np.concatenate([rng.integers(0, 10**9, 1_000_000), [0, 1, 10**9 - 2, 10**9 - 1]]))
        got = eng.gather(idx.astype(np.uint64))
        want = orc.replay(ocfg(cfg), idx, trace)
        assert got.tobytes() == want.tobytes()
        if g:
            assert f"{eng.checksum():016x}" == g["final_checksum"]
            assert rel_ok(bary[-1], [unhex(v) for v in g["barycentre_fsum"]])


# ---- AUTO fallback when the device refuses the co-resident launch -----------------
@pytest.mark.parametrize("n,what", [(100_003, "grid"), (4096, "persistent")])
def test_auto_falls_back_when_launch_refused(orc, monkeypatch, n, what):
    """A profiler replay, MPS or a shared device can refuse the cooperative /
    cluster launch; AUTO then runs the graph of step kernels (bit-exact), an
    explicit request fails loudly (FSB_FAULT_INJECT refuses the launch)."""
    cfg = fsb.baseline_config(n, 6)
    want_fish, want_trace = orc.simulate(ocfg(cfg))
    with make(cfg) as eng:
        eng.simulate(barycentre=False)
        assert eng.last_strategy() == (what, "")
    monkeypatch.setenv("FSB_FAULT_INJECT", what)
    with make(cfg) as eng:
        trace, _, t = eng.simulate(barycentre=False)
        strat, why = eng.last_strategy()
        got = eng.download()
    assert strat == "stream" and "refused" in why, (strat, why)
    assert trace.tobytes() == want_trace.tobytes()
    assert got.tobytes() == want_fish.tobytes()
    with make(cfg, what) as eng:
        with pytest.raises(fsb.FsbError, match="refused"):
            eng.simulate(barycentre=False)


# ---- eat-region time (SimResult::seconds_eat, sim.hpp:103,112,130) -------------------
@pytest.mark.parametrize("strategy,n", [("stream", 200_003), ("stream", 3_000_001), ("grid", 200_003),
                                        ("persistent", 4096)])
def test_seconds_eat_is_measured(strategy, n):
    """The max region is measured on the device: positive, below the loop time,
    and the two add up to the loop (the reference's validate_records rules,
    csv.hpp:161-179)."""
    cfg = fsb.baseline_config(n, 20)
    with make(cfg, strategy) as eng:
        eng.init()
        eng.run(0, 5)
        _, _, t = eng.run(5, 20)
        assert eng.last_strategy()[0] == strategy
    assert 0.0 < t.seconds_eat < t.seconds_loop
    assert t.seconds_move == pytest.approx(t.seconds_loop - t.seconds_eat, rel=1e-12)
    # a step's max costs at least a CTA reduction and at most the step
    per = t.seconds_eat / 20
    assert 2e-7 < per < t.seconds_loop / 20, per


def test_flat_grid_seconds_eat():
    cfg = fsb.baseline_config(100_003, 10)
    with make(cfg, "grid", flat_grid=True) as eng:
        _, _, t = eng.simulate(barycentre=False)
    assert 0.0 < t.seconds_eat < t.seconds_loop


def test_phase_eat_seconds_is_the_max_only(orc):
    cfg = fsb.baseline_config(500_001, 3)
    with make(cfg) as eng:
        eng.init()
        eng.move(0)
        r = eng.eat()
        assert 0.0 < r.seconds < 1e-3
        # after an upload the max needs its own pass over the school: still only the max
        eng.upload(eng.download())
        r2 = eng.eat()
        assert 0.0 < r2.seconds < 1e-3


# ---- the shared-memory-resident grid (school on chip for all steps) ---------------
@pytest.mark.parametrize("n,t", [(16_385, 7), (300_001, 5), (1_000_000, 4), (1_050_001, 3), (1_060_864, 2),
                                 (1_060_866, 2), (1_100_001, 3)])
def test_smem_grid_and_l2_grid_bit_exact(orc, n, t):
    """Up to ~1.06e6 fish the grid strategy keeps every CTA's pairs in shared
    memory; past that (and with l2_grid) the L2-resident cluster grid runs.
    Both are bit-exact with the oracle; the sums within 1e-12."""
    cfg = fsb.baseline_config(n, t)
    want_fish, want_trace = orc.simulate(ocfg(cfg))
    ref = orc.barycentre_sums(want_fish)
    for l2 in (False, True):
        with make(cfg, "grid", l2_grid=l2) as eng:
            trace, bary, tm = eng.simulate(barycentre=True)
            got = eng.download()
            assert eng.last_strategy()[0] == "grid"
        assert trace.tobytes() == want_trace.tobytes(), (n, l2)
        assert got.tobytes() == want_fish.tobytes(), (n, l2)
        assert rel_ok(bary[-1], ref), (n, l2)
        assert 0.0 < tm.seconds_eat < tm.seconds_loop


# ---- AUTO at its thresholds ----------------------------------------------------------
@pytest.mark.parametrize("n,want", [(16_384, "persistent"), (16_385, "grid"), (1_060_864, "grid"),
                                    (1_060_866, "stream"), (2_500_000, "stream"), (3_000_000, "stream")])
def test_auto_thresholds_bit_exact(orc, n, want):
    """AUTO's choice at each boundary (persistent cluster <= 16,384 fish < the
    shared-memory grid <= its capacity, 148 SMs x 3,584 pairs = 1,060,864 fish
    < graph of claimed-tile step kernels):
    the strategy it runs and the oracle's state and trace on both sides."""
    cfg = fsb.baseline_config(n, 3)
    want_fish, want_trace = orc.simulate(ocfg(cfg))
    with make(cfg, "auto") as eng:
        trace, bary, _ = eng.simulate(barycentre=True)
        assert eng.last_strategy()[0] == want
        got = eng.download()
        ctas, tpc = eng.grid()
        assert tpc == 1024  # the stream strategy's kernel is the claimed-tile one at every size
    assert got.tobytes() == want_fish.tobytes()
    assert trace.tobytes() == want_trace.tobytes()
    assert rel_ok(bary[-1], orc.barycentre_sums(want_fish))


# ---- the two per-step reductions of a one-rank graph ---------------------------------
@pytest.mark.parametrize("n,t", [(1, 3), (63, 4), (100_003, 7), (3_000_001, 4)])
def test_split_fold_equals_last_cta_fold(orc, n, t):
    """The graph's default reduction (every CTA red.max's its max key into the
    step's slot, the next kernel folds the sums beside its run: FastFold) and
    FSB_FLAG_LAST_CTA_FOLD (arrival counter + last-CTA fold inside the kernel):
    the oracle's school and trace from both, split runs included, the barycentre
    within tolerance, the cached sums of the final state valid after the run."""
    cfg = fsb.baseline_config(n, t)
    want_fish, want_trace = orc.simulate(ocfg(cfg))
    want_b = orc.barycentre_sums(want_fish)
    for last_cta in (False, True):
        with make(cfg, "stream", last_cta_fold=last_cta) as eng:
            eng.init()
            a, ba, tm = eng.run(0, 1, barycentre=True)
            b, bb, _ = eng.run(1, t - 1, barycentre=True) if t > 1 else (a[:0], ba[:0], None)
            trace, bary = np.concatenate([a, b]), np.concatenate([ba, bb])
            assert trace.tobytes() == want_trace.tobytes(), last_cta
            assert eng.download().tobytes() == want_fish.tobytes(), last_cta
            assert rel_ok(bary[-1], want_b), last_cta
            sums, _ = eng.barycentre()  # the rank partial the consumer folded
            assert rel_ok(sums, want_b), last_cta
            assert 0.0 < tm.seconds_eat < tm.seconds_loop
