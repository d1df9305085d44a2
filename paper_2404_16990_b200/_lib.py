"""ctypes binding of libmsb200.so (include/msb200.h).

The library is built in-tree (``make -C paper_2404_16990_b200`` or
``__graft_entry__.build()``).  There is no fallback: if the shared object is
missing or a call fails, this module raises.  ctypes releases the GIL for
every call, so independent engines can drive their devices from threads
(the reference's ``run_simulations`` fan-out, engine.py:469-479).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

_HERE = Path(__file__).resolve().parent
# MSB200_LIB overrides the in-tree library (tuning builds); default is the in-tree .so
LIB_PATH = Path(os.environ.get("MSB200_LIB", str(_HERE / "libmsb200.so")))

MSB_MODE_FERRO = 0
MSB_MODE_ANTI = 1
MSB_MODE_GENERIC = 2
MSB_MAX_PLANES = 10
MSB_FLIP_SLOTS = 256
MSB_SWEEP_AHEAD_IN = 1
MSB_SWEEP_AHEAD_OUT = 2
MSB_SWEEP_SERIAL = 4
MSB_RNG_XOSHIRO = 0
MSB_RNG_PHILOX = 1
MSB_RNG_PHILOX_BITS = 2
RNG_MODES = {"xoshiro": MSB_RNG_XOSHIRO, "philox": MSB_RNG_PHILOX, "philox-bits": MSB_RNG_PHILOX_BITS}


class MsbError(RuntimeError):
    """A libmsb200 call returned a non-zero status."""


class Geom(ctypes.Structure):
    _fields_ = [
        ("n_sim", ctypes.c_int32),
        ("m", ctypes.c_int32),
        ("n", ctypes.c_int32),
        ("row0", ctypes.c_int32),
        ("rows", ctypes.c_int32),
        ("ghost", ctypes.c_int32),
        ("sim_offset", ctypes.c_int64),
    ]


class SweepParams(ctypes.Structure):
    _fields_ = [
        ("mode", ctypes.c_int32),
        ("n_planes", ctypes.c_int32),
        ("thr9", ctypes.c_void_p),
        ("code_plane", ctypes.c_int8 * 16),
        ("kg", ctypes.c_int32),
        ("jump", ctypes.c_void_p),
        ("fault", ctypes.c_int32),
        ("block_rows", ctypes.c_int32),
        ("work", ctypes.c_void_p),
        ("rng", ctypes.c_int32),
        ("seed", ctypes.c_uint64),
        ("block", ctypes.c_uint64),
        ("flags", ctypes.c_void_p),
    ]


class Halo(ctypes.Structure):
    """msb_halo: in-kernel halo exchange of a slab (include/msb200.h): the
    neighbours' spin buffers and row counts, and their flag buffers."""
    _fields_ = [
        ("up_spins", ctypes.c_void_p), ("down_spins", ctypes.c_void_p),
        ("up_R", ctypes.c_int32), ("down_R", ctypes.c_int32),
        ("up_flags", ctypes.c_void_p), ("down_flags", ctypes.c_void_p),
    ]


class RingSlab(ctypes.Structure):
    """msb_ring_slab: one slab of a ring launch (msb_window_sweep_ring /
    msb_direct_sweep_ring)."""
    _fields_ = [
        ("g", ctypes.POINTER(Geom)), ("p", ctypes.POINTER(SweepParams)),
        ("spins", ctypes.c_void_p), ("states", ctypes.c_void_p), ("cur", ctypes.c_void_p),
        ("next", ctypes.c_void_p), ("flips", ctypes.c_void_p), ("halo", ctypes.POINTER(Halo)),
    ]


class WindowIO(ctypes.Structure):
    """msb_window_io: host I/O fused into a window flip launch (include/msb200.h)."""
    _fields_ = [
        ("lin_in", ctypes.c_void_p), ("lin_out", ctypes.c_void_p),
        ("ups", ctypes.c_void_p), ("unsat", ctypes.c_void_p),
    ]


EXPORTS = (
    "msb_status_string", "msb_last_error", "msb_abi_version", "msb_check_geom", "msb_spin_words",
    "msb_row_pitch", "msb_pieces_per_phase", "msb_default_kg", "msb_plan_thresholds",
    "msb_rng_power_tables", "msb_rng_jump_table", "msb_rng_init", "msb_init_random",
    "msb_init_const", "msb_from_linear", "msb_to_linear", "msb_to_ref16", "msb_from_ref16",
    "msb_plane_words", "msb_rng_planes", "msb_flip", "msb_phase", "msb_sweep",
    "msb_default_window", "msb_window_parts", "msb_window_pieces", "msb_window_words", "msb_window_init", "msb_window_sweep",
    "msb_direct_ok", "msb_direct_sweep", "msb_flag_words",
    "msb_ring_ctx_bytes", "msb_window_sweep_ring", "msb_direct_sweep_ring",
    "msb_observe", "msb_export", "msb_draws", "msb_pack_edges", "msb_unpack_ghosts", "msb_bench_int_peak",
)

_lib = None


def build(force: bool = False) -> Path:
    """Compile libmsb200.so for sm_100a with nvcc (in-tree)."""
    if force and LIB_PATH.exists():
        LIB_PATH.unlink()
    subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return LIB_PATH


def lib() -> ctypes.CDLL:
    """The loaded library; raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise MsbError(f"{LIB_PATH} is missing: build it with `make -C {_HERE}` "
                       "(or __graft_entry__.build()); there is no CPU fallback")
    L = ctypes.CDLL(str(LIB_PATH))
    vp, i32, i64, u64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64
    G = ctypes.POINTER(Geom)
    P = ctypes.POINTER(SweepParams)
    sig = {
        "msb_status_string": ([ctypes.c_int], ctypes.c_char_p),
        "msb_last_error": ([], ctypes.c_char_p),
        "msb_abi_version": ([], ctypes.c_int),
        "msb_check_geom": ([G], ctypes.c_int),
        "msb_spin_words": ([G], i64),
        "msb_row_pitch": ([G], i32),
        "msb_pieces_per_phase": ([G, i32], i64),
        "msb_default_kg": ([G], i32),
        "msb_plan_thresholds": ([vp, i32, vp, vp, vp, vp], ctypes.c_int),
        "msb_rng_power_tables": ([vp], ctypes.c_int),
        "msb_rng_jump_table": ([u64, vp], ctypes.c_int),
        "msb_rng_init": ([G, u64, i32, u64, i32, vp, vp, vp], ctypes.c_int),
        "msb_init_random": ([G, u64, vp, vp, vp, vp], ctypes.c_int),
        "msb_init_const": ([G, i32, vp, vp], ctypes.c_int),
        "msb_from_linear": ([G, vp, vp, vp], ctypes.c_int),
        "msb_to_linear": ([G, vp, vp, vp], ctypes.c_int),
        "msb_to_ref16": ([G, vp, vp, vp], ctypes.c_int),
        "msb_from_ref16": ([G, vp, vp, vp], ctypes.c_int),
        "msb_plane_words": ([G, i32], i64),
        "msb_rng_planes": ([G, P, i32, vp, vp, vp, vp], ctypes.c_int),
        "msb_flip": ([G, P, i32, vp, vp, vp, vp], ctypes.c_int),
        "msb_phase": ([G, P, i32, vp, vp, vp, vp, vp, vp], ctypes.c_int),
        "msb_sweep": ([G, P, vp, vp, vp, i32, i32, vp, vp, vp], ctypes.c_int),
        "msb_default_window": ([G, vp, vp], ctypes.c_int),
        "msb_window_parts": ([G, i32], i32),
        "msb_window_pieces": ([G, i32, i32], i64),
        "msb_window_words": ([G, i32], i64),
        "msb_window_init": ([G, u64, i32, i32, u64, vp, vp, vp], ctypes.c_int),
        "msb_window_sweep": ([G, P, i32, i32, vp, vp, vp, i32, i32, vp, vp, ctypes.POINTER(Halo),
                              ctypes.POINTER(WindowIO), vp], ctypes.c_int),
        "msb_direct_ok": ([G, P], i32),
        "msb_flag_words": ([G], i64),
        "msb_direct_sweep": ([G, P, vp, i32, vp, ctypes.POINTER(Halo), ctypes.POINTER(WindowIO), vp], ctypes.c_int),
        "msb_ring_ctx_bytes": ([i32], i64),
        "msb_window_sweep_ring": ([i32, ctypes.POINTER(RingSlab), i32, i32, i32, i32, vp, vp], ctypes.c_int),
        "msb_direct_sweep_ring": ([i32, ctypes.POINTER(RingSlab), i32, vp, vp], ctypes.c_int),
        "msb_observe": ([G, vp, vp, vp, vp], ctypes.c_int),
        "msb_export": ([G, vp, vp, vp, vp, vp], ctypes.c_int),
        "msb_draws": ([G, P, i32, vp, vp, vp], ctypes.c_int),
        "msb_pack_edges": ([G, i32, vp, vp, vp], ctypes.c_int),
        "msb_unpack_ghosts": ([G, i32, vp, vp, vp], ctypes.c_int),
        "msb_bench_int_peak": ([i32, i32, vp, vp, vp], ctypes.c_int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _lib = L
    return L


def check(status: int, what: str = "") -> None:
    if status != 0:
        L = lib()
        raise MsbError(f"{what}: {L.msb_status_string(status).decode()}: "
                       f"{L.msb_last_error().decode()}")


def call(name: str, *args) -> int:
    """Invoke an ABI function and raise on a non-zero status."""
    fn = getattr(lib(), name)
    st = fn(*args)
    if fn.restype is ctypes.c_int:
        check(st, name)
    return st


def geom(n_sim: int, m: int, n: int, row0: int = 0, rows: int | None = None, ghost: int = 0,
         sim_offset: int = 0) -> Geom:
    return Geom(int(n_sim), int(m), int(n), int(row0), int(m if rows is None else rows),
                int(ghost), int(sim_offset))
