"""TEST INFRASTRUCTURE ONLY -- ctypes handles on the parity checkers.

* ``Oracle``   : liboracle.so, the plain-C restatement of the reference FSB
                 algorithm (fsb_oracle.c; each function cites sim.hpp/rng.hpp).
* ``Reference``: _ref/libfsbref.so, the reference headers compiled unmodified
                 (ref_driver.cpp + Makefile).  Only buildable where
                 /root/reference exists; the built .so travels to the GPU box.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs may import this package.  The product package
(paper_2507_20173_b200) never does.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libfsbref.so")
REF_INCLUDE = os.environ.get("FSB_REF_INCLUDE", "/root/reference/proj/include")

FISH_DTYPE = np.dtype(
    [
        ("x", "<f8"),
        ("y", "<f8"),
        ("weight", "<f8"),
        ("prev_objective", "<f8"),
        ("current_objective", "<f8"),
    ]
)
CHECKSUM_EMPTY = 0xCBF29CE484222325

# parfor enums (schedule.hpp:21,26)
STATIC, DYNAMIC, GUIDED, RUNTIME = 0, 1, 2, 3
SEQUENTIAL, REDUCTION, CRITICAL_PARTIAL, CRITICAL_FULL = 0, 1, 2, 3


class Config(ctypes.Structure):
    """fsb::SimConfig fields (sim.hpp:34-50); same layout as fsb_sim_config."""

    _fields_ = [
        ("num_fish", ctypes.c_uint64),
        ("pond_size", ctypes.c_double),
        ("weight_scale", ctypes.c_double),
        ("num_steps", ctypes.c_uint64),
        ("seed", ctypes.c_uint64),
        ("step_base", ctypes.c_double),
    ]

    @classmethod
    def make(cls, num_fish=10000, pond_size=200.0, weight_scale=10.0, num_steps=1000, seed=1,
             step_base=1.0):
        # defaults = the reference SimConfig defaults (sim.hpp:35-40)
        return cls(num_fish, pond_size, weight_scale, num_steps, seed, step_base)


def baseline_config(num_fish, num_steps, seed=7):
    """BASELINE.json configs mapped onto SimConfig."""
    return Config.make(num_fish=num_fish, pond_size=200.0, weight_scale=1.0, num_steps=num_steps,
                       seed=seed, step_base=0.1)


def _ptr(a):
    return ctypes.c_void_p(a.ctypes.data) if a is not None else ctypes.c_void_p(0)


def build(quiet=True):
    """Build liboracle.so (and _ref/libfsbref.so when the reference is present)."""
    cmd = ["make", "-s", "-C", HERE, f"REF_INCLUDE={REF_INCLUDE}"]
    subprocess.run(cmd, check=True, capture_output=quiet)


class Oracle:
    def __init__(self, path=ORACLE_SO):
        if not os.path.exists(path):
            build()
        L = ctypes.CDLL(path)
        u64, dbl, vp = ctypes.c_uint64, ctypes.c_double, ctypes.c_void_p
        cp = ctypes.POINTER(Config)
        sig = {
            "oracle_mix64": (u64, [u64]),
            "oracle_fold_in": (u64, [u64, u64]),
            "oracle_bits": (u64, [u64, u64, u64, u64]),
            "oracle_unit": (dbl, [u64, u64, u64, u64]),
            "oracle_objective": (dbl, [dbl, dbl, dbl]),
            "oracle_validate": (ctypes.c_int, [cp]),
            "oracle_init": (None, [cp, u64, u64, vp]),
            "oracle_move": (None, [cp, u64, u64, u64, vp]),
            "oracle_eat_max": (dbl, [vp, u64]),
            "oracle_eat_apply": (None, [cp, dbl, vp, u64]),
            "oracle_eat": (dbl, [cp, vp, u64]),
            "oracle_simulate": (None, [cp, vp, vp]),
            "oracle_run": (None, [cp, vp, u64, u64, u64, vp]),
            "oracle_checksum": (u64, [vp, u64]),
            "oracle_checksum_update": (u64, [u64, vp, u64]),
            "oracle_barycentre_sums": (None, [vp, u64, vp]),
            "oracle_replay_fish": (None, [cp, u64, vp, u64, vp]),
            "oracle_replay_many": (None, [cp, vp, u64, vp, u64, vp]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        self.L = L

    # thin numpy-friendly wrappers -------------------------------------------------
    def init(self, cfg, first=0, n=None):
        n = cfg.num_fish if n is None else n
        out = np.zeros(n, dtype=FISH_DTYPE)
        self.L.oracle_init(ctypes.byref(cfg), first, n, _ptr(out))
        return out

    def move(self, cfg, step, fish, first=0):
        self.L.oracle_move(ctypes.byref(cfg), step, first, len(fish), _ptr(fish))

    def eat(self, cfg, fish):
        return self.L.oracle_eat(ctypes.byref(cfg), _ptr(fish), len(fish))

    def eat_max(self, fish):
        return self.L.oracle_eat_max(_ptr(fish), len(fish))

    def eat_apply(self, cfg, m, fish):
        self.L.oracle_eat_apply(ctypes.byref(cfg), m, _ptr(fish), len(fish))

    def simulate(self, cfg):
        fish = np.zeros(cfg.num_fish, dtype=FISH_DTYPE)
        trace = np.zeros(cfg.num_steps, dtype=np.float64)
        self.L.oracle_simulate(ctypes.byref(cfg), _ptr(fish), _ptr(trace))
        return fish, trace

    def run(self, cfg, fish, first_step, num_steps):
        trace = np.zeros(num_steps, dtype=np.float64)
        self.L.oracle_run(ctypes.byref(cfg), _ptr(fish), len(fish), first_step, num_steps, _ptr(trace))
        return trace

    def checksum(self, fish):
        return self.L.oracle_checksum(_ptr(fish), len(fish))

    def barycentre_sums(self, fish):
        out = np.zeros(3, dtype=np.float64)
        self.L.oracle_barycentre_sums(_ptr(fish), len(fish), _ptr(out))
        return out

    def objective(self, x, y, pond):
        return self.L.oracle_objective(x, y, pond)

    def replay(self, cfg, indices, trace):
        """Replay the given global fish indices alone with a run's max_diff trace."""
        trace = np.ascontiguousarray(trace, dtype=np.float64)
        idx = np.ascontiguousarray(indices, dtype=np.uint64)
        out = np.zeros(len(idx), dtype=FISH_DTYPE)
        self.L.oracle_replay_many(ctypes.byref(cfg), _ptr(idx), len(idx), _ptr(trace), len(trace), _ptr(out))
        return out


class Reference:
    """The unmodified reference (oracle/_ref/libfsbref.so)."""

    def __init__(self, path=REF_SO):
        if not os.path.exists(path):
            if os.path.exists(os.path.join(REF_INCLUDE, "fsb", "sim.hpp")):
                build()
            if not os.path.exists(path):
                raise FileNotFoundError(f"{path} not built (reference headers absent)")
        L = ctypes.CDLL(path)
        u64, dbl, vp, i = ctypes.c_uint64, ctypes.c_double, ctypes.c_void_p, ctypes.c_int
        cp = ctypes.POINTER(Config)
        sig = {
            "ref_validate": (i, [cp]),
            "ref_objective": (dbl, [dbl, dbl, dbl]),
            "ref_bits": (u64, [u64, u64, u64, u64]),
            "ref_init": (i, [cp, vp]),
            "ref_move": (dbl, [cp, u64, vp, u64, i, i, u64, i]),
            "ref_eat": (dbl, [cp, vp, u64, i, i, u64, i]),
            "ref_simulate": (i, [cp, i, i, u64, i, vp, vp, vp]),
            "ref_checksum": (u64, [vp, u64]),
            "ref_time_steps": (dbl, [cp, i, i, u64, i, u64, u64, vp, vp]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        self.L = L

    def init(self, cfg):
        out = np.zeros(cfg.num_fish, dtype=FISH_DTYPE)
        rc = self.L.ref_init(ctypes.byref(cfg), _ptr(out))
        if rc:
            raise ValueError("invalid SimConfig")
        return out

    def simulate(self, cfg, threads=1, sched=STATIC, chunk=0, construct=SEQUENTIAL):
        fish = np.zeros(cfg.num_fish, dtype=FISH_DTYPE)
        trace = np.zeros(cfg.num_steps, dtype=np.float64)
        secs = np.zeros(3, dtype=np.float64)
        rc = self.L.ref_simulate(ctypes.byref(cfg), threads, sched, chunk, construct, _ptr(fish),
                                 _ptr(trace), _ptr(secs))
        if rc:
            raise ValueError("invalid SimConfig")
        return fish, trace, secs

    def move(self, cfg, step, fish, threads=1, sched=STATIC, chunk=0, construct=SEQUENTIAL):
        return self.L.ref_move(ctypes.byref(cfg), step, _ptr(fish), len(fish), threads, sched, chunk,
                               construct)

    def eat(self, cfg, fish, threads=1, sched=STATIC, chunk=0, construct=SEQUENTIAL):
        return self.L.ref_eat(ctypes.byref(cfg), _ptr(fish), len(fish), threads, sched, chunk,
                              construct)

    def checksum(self, fish):
        return self.L.ref_checksum(_ptr(fish), len(fish))

    def time_steps(self, cfg, warmup, steps, threads=1, sched=STATIC, chunk=0,
                   construct=SEQUENTIAL, want_trace=False):
        per = np.zeros(steps, dtype=np.float64)
        trace = np.zeros(steps, dtype=np.float64) if want_trace else None
        total = self.L.ref_time_steps(ctypes.byref(cfg), threads, sched, chunk, construct, warmup,
                                      steps, _ptr(per), _ptr(trace))
        return total, per, trace
