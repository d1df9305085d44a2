"""Python face of the CPU oracle (TEST INFRASTRUCTURE ONLY).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs import this module, and only as
the checker; the product package never does.  The heavy lifting lives in
``msb_oracle.c`` (see its header for the reference file:line map); this file
adds the float64 pieces the reference computes in Python:

* ``exp_table``   restates ``build_exp_table`` (engine.py:78-94), using the same
  CPython ``math.exp`` so every double is bitwise identical;
* ``OracleEngine`` mirrors ``Engine`` (engine.py:216-440) on a plain +/-1
  lattice: same seeding, stream ids, consumption order, counters and the
  float64 observable expressions of engine.py:372-386.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "libmsb_oracle.so"
_lib = None


def build() -> Path:
    """Compile the oracle with its Makefile (gcc, pthreads)."""
    subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            build()
        L = ctypes.CDLL(str(_LIB_PATH))
        u64, i32, vp = ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p
        L.orc_stream_state.argtypes = [u64, u64, vp]
        L.orc_raw64.argtypes = [u64, u64, u64, u64, vp]
        L.orc_init_random.argtypes = [i32, i32, i32, u64, u64, vp]
        L.orc_flip_phase.argtypes = [i32, i32, i32, i32, vp, vp, vp, vp]
        L.orc_flip_states.argtypes = [i32, i32, u64, u64, u64, vp]
        L.orc_sweeps.argtypes = [i32, i32, i32, i32, vp, vp, vp, vp]
        L.orc_observe.argtypes = [i32, i32, i32, vp, vp, vp]
        L.orc_draw_map_sweep.argtypes = [i32, i32, vp, vp]
        L.orc_set_threads.argtypes = [i32]
        L.orc_flip_phase_philox.argtypes = [i32, i32, i32, i32, u64, u64, u64, vp, vp, vp]
        L.orc_philox_draw.argtypes = [u64, u64, u64]
        L.orc_philox_draw.restype = ctypes.c_uint32
        L.orc_flip_phase_philox_bits.argtypes = [i32, i32, i32, i32, u64, u64, u64, vp, vp, vp]
        L.orc_pbits_draw.argtypes = [u64, u64, u64]
        L.orc_pbits_draw.restype = ctypes.c_uint32
        L.orc_num_threads.restype = i32
        _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.c_void_p)


def _u64(x: int) -> int:
    return int(x) & ((1 << 64) - 1)


def set_threads(n: int) -> None:
    lib().orc_set_threads(int(n))


def num_threads() -> int:
    return int(lib().orc_num_threads())


# --- RNG (rng.py:53-147) -----------------------------------------------------


def stream_state(master: int, stream: int) -> list[int]:
    out = np.zeros(4, np.uint64)
    lib().orc_stream_state(_u64(master), _u64(stream), _p(out))
    return [int(v) for v in out]


def raw64(master: int, stream: int, count: int, skip: int = 0) -> np.ndarray:
    out = np.zeros(count, np.uint64)
    lib().orc_raw64(_u64(master), _u64(stream), int(skip), int(count), _p(out))
    return out


# --- tables (engine.py:78-94) ---------------------------------------------------


def exp_table(T: float, J: float = 1.0) -> np.ndarray:
    if T <= 0:
        raise ValueError("temperature must be positive")
    table = np.zeros(16, dtype=np.float64)
    for own in (0, 1):
        sigma = 2 * own - 1
        for up in range(5):
            de = 2.0 * J * sigma * (2 * up - 4)
            table[8 * own + up] = 1.0 if de <= 0 else math.exp(-de / T)
    return table


# --- engine (engine.py:216-440) on a plain lattice ------------------------------


class OracleEngine:
    """Plain-lattice restatement of the reference ``Engine``."""

    def __init__(self, m, n, temperatures, seed, init="random", coupling=1.0, sim_offset=0,
                 lattices=None, stream="xoshiro"):
        if m < 4 or m % 4 or n < 32 or n % 32:
            raise ValueError("bad dims")
        self.m, self.n = int(m), int(n)
        self.temperatures = tuple(float(t) for t in temperatures)
        self.n_sim = len(self.temperatures)
        self.seed = int(seed)
        self.coupling = float(coupling)
        self.sim_offset = int(sim_offset)
        self.tables = np.stack([exp_table(t, self.coupling) for t in self.temperatures])
        self.states = np.zeros((self.n_sim * (m // 4), 4), np.uint64)
        lib().orc_flip_states(self.n_sim, m, _u64(self.seed), self.sim_offset, 0, _p(self.states))
        self.spins = np.ones((self.n_sim, m, n), np.int8)
        if lattices is not None:
            for s, lat in enumerate(lattices):
                self.spins[s] = lat
        elif init == "random":
            lib().orc_init_random(self.n_sim, m, n, _u64(self.seed), self.sim_offset, _p(self.spins))
        elif init != "all-up":
            raise ValueError(f"unknown init mode {init!r}")
        self.stream = stream
        self.sweeps_done = 0
        self.attempts = 0
        self._flips = np.zeros(1, np.uint64)

    @property
    def sites(self) -> int:
        return self.m * self.n

    @property
    def flips(self) -> int:
        return int(self._flips[0])

    def sweep(self, n_sweeps: int = 1) -> None:
        tab = np.ascontiguousarray(self.tables, dtype=np.float64)
        if self.stream in ("philox", "philox-bits"):
            fn = lib().orc_flip_phase_philox if self.stream == "philox" else lib().orc_flip_phase_philox_bits
            for k in range(n_sweeps):
                for ph in (0, 1):
                    fn(self.n_sim, self.m, self.n, ph, _u64(self.seed), self.sim_offset,
                       2 * (self.sweeps_done + k) + ph, _p(tab), _p(self.spins), _p(self._flips))
        else:
            lib().orc_sweeps(self.n_sim, self.m, self.n, int(n_sweeps), _p(self.states), _p(tab),
                             _p(self.spins), _p(self._flips))
        self.sweeps_done += n_sweeps
        self.attempts += self.sites * self.n_sim * n_sweeps

    def observe(self):
        ups = np.zeros(self.n_sim, np.int64)
        bonds = np.zeros(self.n_sim, np.int64)
        lib().orc_observe(self.n_sim, self.m, self.n, _p(self.spins), _p(ups), _p(bonds))
        return ups, bonds

    def abs_magnetization(self) -> np.ndarray:
        ups, _ = self.observe()
        return np.abs(2.0 * ups / self.sites - 1.0)  # engine.py:375

    def energy_per_spin(self) -> np.ndarray:
        _, bonds = self.observe()
        return np.array([-self.coupling * b / self.sites for b in bonds])  # engine.py:385

    def run(self, n_sweeps: int, measure_interval: int = 100):
        """engine.py:401-440 cadence; returns (sweeps, abs_m, energy)."""
        sw, am, en = [], [], []
        for k in range(1, n_sweeps + 1):
            self.sweep()
            if k % measure_interval == 0 or k == n_sweeps:
                sw.append(self.sweeps_done)
                am.append(self.abs_magnetization())
                en.append(self.energy_per_spin())
        return (np.array(sw, np.int64), np.array(am).reshape(len(sw), self.n_sim),
                np.array(en).reshape(len(sw), self.n_sim))

    def draw_map(self) -> np.ndarray:
        """Draw map of the next sweep without advancing (single sim)."""
        if self.n_sim != 1:
            raise ValueError("draw maps require a single simulation")
        st = self.states.copy()
        out = np.full((self.m, self.n), np.nan)
        lib().orc_draw_map_sweep(self.m, self.n, _p(st), _p(out))
        return out
