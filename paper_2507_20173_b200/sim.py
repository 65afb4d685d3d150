"""Python mirror of the reference simulation API (proj/include/fsb/sim.hpp).

Same names, argument meaning and error behaviour as the reference, with the
``parfor::Executor&`` argument replaced by a :class:`GpuExecutor` (or an
:class:`Engine` for device-resident work).  All compute goes through the
C-ABI (include/fsb_b200.h) into the sm_100a kernels; there is no CPU path.

    reference (sim.hpp)                       here
    ----------------------------------------  -------------------------------------
    struct Fish                  :26-32       FISH_DTYPE (numpy structured, 40 B)
    struct SimConfig             :34-50       SimConfig
    struct School                :52-56       School
    objective(x, y, pond)        :59-63       objective
    init_school(cfg)             :65-79       init_school(cfg, exec)
    move_phase(school,cfg,step,exec) :84-99   move_phase(school, cfg, step, exec)
    EatResult / eat_phase        :101-123     EatResult / eat_phase(school, cfg, exec)
    SimResult / simulate         :125-152     SimResult / simulate(cfg, exec)
    checksum(school)             :154-176     checksum(school)
    (none)                       barycentre(school) / Engine.barycentre()
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _native as N

kWeightMin = 1.0  # sim.hpp:24
kChecksumEmpty = 0xCBF29CE484222325  # sim.hpp:156
kInitStep = (1 << 64) - 1  # rng.hpp:27

FISH_DTYPE = np.dtype(
    [
        ("x", "<f8"),
        ("y", "<f8"),
        ("weight", "<f8"),
        ("prev_objective", "<f8"),
        ("current_objective", "<f8"),
    ]
)

STRATEGIES = {"auto": N.STRATEGY_AUTO, "stream": N.STRATEGY_STREAM, "persistent": N.STRATEGY_PERSISTENT,
              "grid": N.STRATEGY_GRID}


@dataclass
class SimConfig:
    """sim.hpp:34-50 (defaults included)."""

    num_fish: int = 10000
    pond_size: float = 200.0
    weight_scale: float = 10.0
    num_steps: int = 1000
    seed: int = 1
    step_base: float = 1.0

    def weight_max(self) -> float:
        return 2.0 * self.weight_scale

    def validate(self) -> None:
        """Raises ValueError (the reference throws std::invalid_argument)."""
        c = self._c()
        N.check(N.lib().fsb_config_validate(ctypes.byref(c)))

    def _c(self) -> N.fsb_sim_config:
        return N.fsb_sim_config(int(self.num_fish), float(self.pond_size), float(self.weight_scale),
                                int(self.num_steps), int(self.seed) & ((1 << 64) - 1),
                                float(self.step_base))


def baseline_config(num_fish: int, num_steps: int, seed: int = 7) -> SimConfig:
    """BASELINE.json configs on the reference SimConfig."""
    return SimConfig(num_fish=num_fish, pond_size=200.0, weight_scale=1.0, num_steps=num_steps,
                     seed=seed, step_base=0.1)


class School:
    """sim.hpp:52-56: owns the fish (AoS, Fish byte layout)."""

    def __init__(self, fishes: Optional[np.ndarray] = None):
        if fishes is None:
            fishes = np.zeros(0, dtype=FISH_DTYPE)
        self.fishes = np.ascontiguousarray(fishes, dtype=FISH_DTYPE)

    def size(self) -> int:
        return int(self.fishes.shape[0])

    def copy(self) -> "School":
        return School(self.fishes.copy())


@dataclass
class EatResult:
    """sim.hpp:101-104."""

    max_diff: float = -math.inf
    seconds: float = 0.0


@dataclass
class SimResult:
    """sim.hpp:125-131, plus the per-step barycentre sums (north_star)."""

    school: School = field(default_factory=School)
    max_diff_trace: np.ndarray = field(default_factory=lambda: np.zeros(0))
    seconds_total: float = 0.0
    seconds_move: float = 0.0
    seconds_eat: float = 0.0
    barycentre_trace: Optional[np.ndarray] = None  # [num_steps, 3]: sum x*f, sum y*f, sum f


def objective(x: float, y: float, pond_size: float) -> float:
    """sim.hpp:59-63 (host scalar helper; CPython floats are IEEE binary64, no FMA)."""
    dx = x - pond_size / 2.0
    dy = y - pond_size / 2.0
    return math.sqrt(dx * dx + dy * dy)


def _ptr(a: Optional[np.ndarray]) -> ctypes.c_void_p:
    return ctypes.c_void_p(a.ctypes.data if a is not None and a.size else 0)


class Engine:
    """One shard of a device-resident school (fsb_engine_*).

    Single GPU: ``Engine(cfg)``.  Multi-GPU: one Engine per process/GPU with
    ``rank``, ``world_size`` and a shared 128-byte ``nccl_unique_id``
    (:func:`nccl_unique_id` on rank 0, broadcast by the caller).
    """

    def __init__(self, cfg: SimConfig, device: int = 0, rank: int = 0, world_size: int = 1,
                 nccl_unique_id: Optional[bytes] = None, strategy: str = "auto",
                 alternate: bool = True, force_nccl: bool = False, bulk=False, pdl: bool = True,
                 peer: bool = False, checked: bool = False, static_tiles: bool = False,
                 dynamic_tiles: bool = False, flat_grid: bool = False, host_exchange: bool = False,
                 l2_grid: bool = False, ws_tiles: bool = False, last_cta_fold: bool = False):
        self.cfg = cfg
        L = N.lib()
        self._uid = ctypes.create_string_buffer(nccl_unique_id, 128) if nccl_unique_id else None
        flags = ((0 if alternate else N.FLAG_NO_ALTERNATE) | (N.FLAG_FORCE_NCCL if force_nccl else 0)
                 | (N.FLAG_FORCE_BULK if bulk else 0)
                 | (0 if pdl else N.FLAG_NO_PDL) | (N.FLAG_PEER_EXCHANGE if peer else 0)
                 | (N.FLAG_CHECKED if checked else 0) | (N.FLAG_STATIC_TILES if static_tiles else 0)
                 | (N.FLAG_DYNAMIC_TILES if dynamic_tiles else 0) | (N.FLAG_FLAT_GRID if flat_grid else 0)
                 | (N.FLAG_HOST_EXCHANGE if host_exchange else 0) | (N.FLAG_L2_GRID if l2_grid else 0)
                 | (N.FLAG_LAST_CTA_FOLD if last_cta_fold else 0)
                 | (N.FLAG_WS_TILES if ws_tiles else 0))
        opts = N.fsb_engine_options(device, rank, world_size,
                                    ctypes.cast(self._uid, ctypes.c_void_p) if self._uid else None,
                                    STRATEGIES[strategy], flags)
        h = ctypes.c_void_p()
        c = cfg._c()
        N.check(L.fsb_engine_create(ctypes.byref(c), ctypes.byref(opts), ctypes.byref(h)))
        self._h = h
        first, count = ctypes.c_uint64(), ctypes.c_uint64()
        N.check(L.fsb_engine_shard(h, ctypes.byref(first), ctypes.byref(count)))
        self.first, self.count = first.value, count.value
        self.device, self.rank, self.world_size = device, rank, world_size

    # lifecycle ------------------------------------------------------------------
    def close(self) -> None:
        if getattr(self, "_h", None):
            N.lib().fsb_engine_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # state ------------------------------------------------------------------------
    def init(self) -> None:
        N.check(N.lib().fsb_engine_init(self._h))

    def upload(self, fishes: np.ndarray) -> None:
        f = np.ascontiguousarray(fishes, dtype=FISH_DTYPE)
        N.check(N.lib().fsb_engine_upload(self._h, _ptr(f), f.shape[0]))

    def download(self, out: Optional[np.ndarray] = None) -> np.ndarray:
        if out is None:
            out = np.empty(self.count, dtype=FISH_DTYPE)
        N.check(N.lib().fsb_engine_download(self._h, _ptr(out), out.shape[0]))
        return out

    # phases -------------------------------------------------------------------------
    def move(self, step: int) -> float:
        s = ctypes.c_double()
        N.check(N.lib().fsb_engine_move(self._h, step, ctypes.byref(s)))
        return s.value

    def eat(self) -> EatResult:
        m, s = ctypes.c_double(), ctypes.c_double()
        N.check(N.lib().fsb_engine_eat(self._h, ctypes.byref(m), ctypes.byref(s)))
        return EatResult(m.value, s.value)

    def run(self, first_step: int, num_steps: int, barycentre: bool = False):
        """Steps [first_step, first_step+num_steps): returns (trace, bary|None, fsb_timing)."""
        trace = np.empty(num_steps, dtype=np.float64)
        bary = np.empty((num_steps, 3), dtype=np.float64) if barycentre else None
        t = N.fsb_timing()
        N.check(N.lib().fsb_engine_run(self._h, first_step, num_steps, _ptr(trace), _ptr(bary),
                                       ctypes.byref(t)))
        return trace, bary, t

    def simulate(self, barycentre: bool = True):
        n = self.cfg.num_steps
        trace = np.empty(n, dtype=np.float64)
        bary = np.empty((n, 3), dtype=np.float64) if barycentre else None
        t = N.fsb_timing()
        N.check(N.lib().fsb_engine_simulate(self._h, _ptr(trace), _ptr(bary), ctypes.byref(t)))
        return trace, bary, t

    def barycentre(self):
        """Global sums (sum x*f, sum y*f, sum f) and B = (sum x*f/sum f, sum y*f/sum f)."""
        sums = np.empty(3, dtype=np.float64)
        xy = np.empty(2, dtype=np.float64)
        N.check(N.lib().fsb_engine_barycentre(self._h, _ptr(sums), _ptr(xy)))
        return sums, xy

    def partial(self) -> np.ndarray:
        """This rank's partial of the current state: [max(prev-cur), sum x*f, sum y*f, sum f, epoch]
        (epoch = the exchange sequence number, equal on every rank at the same step)."""
        out = np.empty(5, dtype=np.float64)
        N.check(N.lib().fsb_engine_partial(self._h, _ptr(out)))
        return out

    def set_partials(self, parts) -> None:
        """Host exchange engines: every rank's partial() in rank order (world_size x 5)."""
        a = np.ascontiguousarray(parts, dtype=np.float64).reshape(-1)
        N.check(N.lib().fsb_engine_set_partials(self._h, _ptr(a), a.shape[0]))

    def peer_handle(self) -> bytes:
        """This rank's 64-byte IPC handle (peer exchange engines)."""
        buf = ctypes.create_string_buffer(64)
        N.check(N.lib().fsb_engine_peer_handle(self._h, buf, 64))
        return buf.raw

    def peer_connect(self, handles) -> None:
        """Map every rank's window; `handles` = all ranks' peer_handle() in rank order."""
        blob = b"".join(handles)
        N.check(N.lib().fsb_engine_peer_connect(self._h, blob, len(blob)))

    def peer_connect_local(self, engines) -> None:
        """Connect ranks that live in this process: `engines` = every rank's
        Engine in rank order (fsb_engine_peer_connect_local)."""
        arr = (ctypes.c_void_p * len(engines))(*[e._h.value for e in engines])
        N.check(N.lib().fsb_engine_peer_connect_local(self._h, arr, len(engines)))

    def gather(self, local_idx) -> np.ndarray:
        """Fish at the given shard-local indices (Fish layout)."""
        idx = np.ascontiguousarray(local_idx, dtype=np.uint64)
        out = np.empty(idx.shape[0], dtype=FISH_DTYPE)
        N.check(N.lib().fsb_engine_gather(self._h, _ptr(idx), idx.shape[0], _ptr(out)))
        return out

    def checksum(self, h: int = kChecksumEmpty) -> int:
        out = ctypes.c_uint64()
        N.check(N.lib().fsb_engine_checksum(self._h, h, ctypes.byref(out)))
        return out.value

    def synchronize(self) -> None:
        N.check(N.lib().fsb_engine_synchronize(self._h))

    def stream(self) -> int:
        s = ctypes.c_void_p()
        N.check(N.lib().fsb_engine_stream(self._h, ctypes.byref(s)))
        return s.value or 0

    def time_step_kernels(self, first_step: int, num_steps: int) -> np.ndarray:
        ms = np.empty(num_steps, dtype=np.float64)
        N.check(N.lib().fsb_engine_time_step_kernels(self._h, first_step, num_steps, _ptr(ms)))
        return ms

    def set_grid(self, ctas: int = 0) -> None:
        """CTA count of the compact step / eat kernels (0 = automatic)."""
        N.check(N.lib().fsb_engine_set_grid(self._h, ctas))

    def set_tile_groups(self, groups: int) -> None:
        """Minimum 32-pair groups per claimed tile of the claimed-tile kernel (0 = default)."""
        N.check(N.lib().fsb_engine_set_tile_groups(self._h, groups))

    def grid(self):
        """(CTAs, threads per CTA) of the compact step kernel in use."""
        c, t = ctypes.c_int(), ctypes.c_int()
        N.check(N.lib().fsb_engine_grid(self._h, ctypes.byref(c), ctypes.byref(t)))
        return c.value, t.value

    def last_launches(self) -> int:
        v = ctypes.c_uint64()
        N.check(N.lib().fsb_engine_last_launches(self._h, ctypes.byref(v)))
        return v.value

    def last_strategy(self):
        """(strategy the last run executed: "stream" | "persistent" | "grid", fallback reason or "")."""
        v, why = ctypes.c_int(), ctypes.c_char_p()
        N.check(N.lib().fsb_engine_last_strategy(self._h, ctypes.byref(v), ctypes.byref(why)))
        name = {v_: k for k, v_ in STRATEGIES.items()}.get(v.value, str(v.value))
        return name, (why.value or b"").decode(errors="replace")


class GpuExecutor:
    """Drop-in for the ``parfor::Executor&`` argument of the phase functions.

    Like the reference Executor it is school-size agnostic: it keeps one
    Engine for the most recent (config, school size) and re-creates it when
    either changes.  Phase calls on a host School upload it, run the phase on
    the device and download it (the reference's in-place semantics); use
    :class:`Engine` directly to keep the school resident across steps.
    """

    def __init__(self, device: int = 0, strategy: str = "auto"):
        self.device = device
        self.strategy = strategy
        self._key = None
        self._engine: Optional[Engine] = None

    def engine_for(self, cfg: SimConfig, n: int) -> Engine:
        key = (n, float(cfg.pond_size), float(cfg.weight_scale), int(cfg.seed), float(cfg.step_base),
               int(cfg.num_steps))
        if self._key != key:
            if self._engine is not None:
                self._engine.close()
            c = SimConfig(n, cfg.pond_size, cfg.weight_scale, cfg.num_steps, cfg.seed, cfg.step_base)
            self._engine = Engine(c, device=self.device, strategy=self.strategy)
            self._key = key
        return self._engine

    def close(self) -> None:
        if self._engine is not None:
            self._engine.close()
            self._engine = None
            self._key = None


_default_exec: Optional[GpuExecutor] = None


def _exec(exec_: Optional[GpuExecutor]) -> GpuExecutor:
    global _default_exec
    if exec_ is not None:
        return exec_
    if _default_exec is None:
        _default_exec = GpuExecutor()
    return _default_exec


def init_school(cfg: SimConfig, exec_: Optional[GpuExecutor] = None) -> School:
    """sim.hpp:65-79 (validates first, like the reference)."""
    cfg.validate()
    eng = _exec(exec_).engine_for(cfg, cfg.num_fish)
    eng.init()
    return School(eng.download())


def move_phase(school: School, cfg: SimConfig, step_index: int, exec_: Optional[GpuExecutor] = None) -> float:
    """sim.hpp:84-99: moves every fish in place; returns the device time of the move."""
    eng = _exec(exec_).engine_for(cfg, school.size())
    eng.upload(school.fishes)
    secs = eng.move(step_index)
    eng.download(school.fishes)
    return secs


def eat_phase(school: School, cfg: SimConfig, exec_: Optional[GpuExecutor] = None) -> EatResult:
    """sim.hpp:110-123: global max of prev-cur and the weight update."""
    eng = _exec(exec_).engine_for(cfg, school.size())
    eng.upload(school.fishes)
    r = eng.eat()
    eng.download(school.fishes)
    return r


def simulate(cfg: SimConfig, exec_: Optional[GpuExecutor] = None) -> SimResult:
    """sim.hpp:133-152: init + num_steps x (move, eat), device resident."""
    cfg.validate()
    eng = _exec(exec_).engine_for(cfg, cfg.num_fish)
    trace, bary, t = eng.simulate(barycentre=True)
    return SimResult(School(eng.download()), trace, t.seconds_total, t.seconds_move, t.seconds_eat, bary)


def checksum(school: School) -> int:
    """sim.hpp:158-176: FNV-1a 64 over the exact bytes of every fish."""
    f = school.fishes
    return int(N.lib().fsb_checksum_update(kChecksumEmpty, _ptr(f), f.shape[0]))


def barycentre(school: School, exec_: Optional[GpuExecutor] = None, cfg: Optional[SimConfig] = None):
    """f-weighted barycentre of a host school, computed on the device."""
    cfg = cfg or SimConfig()
    eng = _exec(exec_).engine_for(cfg, school.size())
    eng.upload(school.fishes)
    return eng.barycentre()


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    N.check(N.lib().fsb_nccl_unique_id(buf, 128))
    return buf.raw


def shard_range(num_fish: int, world_size: int, rank: int):
    first, count = ctypes.c_uint64(), ctypes.c_uint64()
    N.check(N.lib().fsb_shard_range(num_fish, world_size, rank, ctypes.byref(first), ctypes.byref(count)))
    return first.value, count.value


def device_count() -> int:
    n = ctypes.c_int()
    N.check(N.lib().fsb_device_count(ctypes.byref(n)))
    return n.value
