"""The C-ABI library on the host (no GPU): it loads, exports every symbol
include/msb200.h declares, validates geometry like LatticeDims, and its host
pieces -- the threshold planner and the GF(2) jump-ahead tables -- are exact
against the float64 compare and the oracle's stream."""
import ctypes
import math
import re
from pathlib import Path

import numpy as np
import pytest

from oracle import oracle as orc
from paper_2404_16990_b200 import _lib
from paper_2404_16990_b200._lib import call, geom
from paper_2404_16990_b200.engine import build_exp_table

ROOT = Path(__file__).resolve().parents[1]


def test_exports_every_declared_symbol():
    header = (ROOT / "include" / "msb200.h").read_text()
    declared = set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(msb_\w+)\s*\(", header, re.M))
    assert len(declared) >= 25
    L = _lib.lib()
    missing = [name for name in sorted(declared) if not hasattr(L, name)]
    assert not missing, missing
    assert set(_lib.EXPORTS) <= declared
    assert L.msb_abi_version() == 2


def test_geometry_validation_messages():
    L = _lib.lib()
    assert L.msb_check_geom(ctypes.byref(geom(1, 12, 96))) == 0
    for g, text in [(geom(1, 6, 96), "multiple of 4"), (geom(1, 12, 48), "multiple of 32"),
                    (geom(0, 12, 96), "replica"), (geom(1, 12, 96, row0=2, rows=4), "whole lattice")]:
        assert L.msb_check_geom(ctypes.byref(g)) == -1
        assert text in L.msb_last_error().decode()
    with pytest.raises(_lib.MsbError, match="multiple of 4"):
        call("msb_check_geom", ctypes.byref(geom(1, 10, 96)))


def test_sizes():
    L = _lib.lib()
    g = geom(64, 1024, 1024)
    assert L.msb_row_pitch(ctypes.byref(g)) == 16             # 32 words of 16 bits -> 16 uint32
    assert L.msb_spin_words(ctypes.byref(g)) == 64 * 2 * 1024 * 16
    assert L.msb_pieces_per_phase(ctypes.byref(g), 2) == 64 * 1024 * 2
    assert L.msb_default_kg(ctypes.byref(g)) == 1
    assert L.msb_default_kg(ctypes.byref(geom(1, 14336, 14336))) == 8


def plan(tables):
    tables = np.ascontiguousarray(tables, np.float64)
    n_sim = tables.shape[0]
    mode, npl = ctypes.c_int32(), ctypes.c_int32()
    codes = (ctypes.c_int8 * 16)()
    thr = np.zeros(10 * n_sim, np.uint32)
    call("msb_plan_thresholds", tables.ctypes.data_as(ctypes.c_void_p), n_sim, ctypes.byref(mode),
         ctypes.byref(npl), codes, thr.ctypes.data_as(ctypes.c_void_p))
    return mode.value, npl.value, list(codes), thr.reshape(10, n_sim)


def accepts(key, u):
    """Device rule: reject iff (u << 9) >= key (uint32)."""
    return ((u.astype(np.uint64) << 9) & 0xFFFFFFFF) < key if key != 0xFFFFFFFF else np.ones_like(u, bool)


@pytest.mark.parametrize("T,J", [(2.269, 1.0), (0.5, 1.0), (1.0, 1.0), (5.0, 1.0), (1e-6, 1.0), (3.0, 2.0),
                                 (1.5, -1.0), (2.0, 0.0), (1e300, 1.0)])
def test_integer_keys_equal_float64_compare(T, J):
    """For every 23-bit draw, (u<<9) < key  <=>  u * 2**-23 < table[code]
    (engine.py:325-330), exhaustively."""
    table = build_exp_table(T, J)
    mode, npl, codes, thr = plan(table[None, :])
    assert mode == (1 if J < 0 else 0)
    u = np.arange(1 << 23, dtype=np.uint32)
    r = u.astype(np.float64) * 2.0 ** -23
    for code in range(16):
        if code & 7 > 4:
            continue
        pl = codes[code]
        want = r < table[code]
        if pl == -2:
            got = np.ones_like(want)
        elif pl == -1:
            got = np.zeros_like(want)
        else:
            got = accepts(int(thr[pl, 0]), u)
        assert (got == want).all(), (T, J, code)


def test_generic_planes_for_forced_tables():
    n = 3
    for value, planes in [(0.5, 1), (0.0, 0), (1.0, 0)]:
        mode, npl, codes, thr = plan(np.full((n, 16), value))
        if value == 1.0:
            assert mode == 0  # all-accept fits the ferro structure
        else:
            assert mode == 2 and npl == planes
    rng = np.random.default_rng(1)
    t = rng.random((4, 16))
    mode, npl, codes, thr = plan(t)
    assert mode == 2 and npl == 10  # every valid code distinct
    u = np.arange(0, 1 << 23, 977, dtype=np.uint32)
    r = u.astype(np.float64) * 2.0 ** -23
    for s in range(4):
        for code in range(16):
            if code & 7 <= 4:
                assert (accepts(int(thr[codes[code], s]), u) == (r < t[s, code])).all()


# ---- GF(2) jump-ahead vs the oracle's sequential stream -------------------

M64 = (1 << 64) - 1


def apply_table(table, s):
    """Host application of a nibble table to a state [s0..s3] (uint64)."""
    words = []
    for v in s:
        words += [v & 0xFFFFFFFF, v >> 32]
    r = np.zeros(8, np.uint64)
    t = table.reshape(64, 16, 8).astype(np.uint64)
    for p in range(64):
        nib = (words[p // 8] >> (4 * (p % 8))) & 15
        r ^= t[p, nib]
    return [int(r[2 * k]) | (int(r[2 * k + 1]) << 32) for k in range(4)]


def xnext(s):
    x = (s[0] + s[3]) & M64
    out = ((((x << 23) | (x >> 41)) & M64) + s[0]) & M64
    t = (s[1] << 17) & M64
    s[2] ^= s[0]; s[3] ^= s[1]; s[1] ^= s[2]; s[0] ^= s[3]; s[2] ^= t
    s[3] = ((s[3] << 45) | (s[3] >> 19)) & M64
    return out


@pytest.mark.parametrize("J", [1, 7, 64, 4 * 1024, 4 * 14336, 123456789, (1 << 40) + 5])
def test_jump_table_equals_sequential_stream(J):
    table = np.empty(8192, np.uint32)
    call("msb_rng_jump_table", ctypes.c_uint64(J), table.ctypes.data_as(ctypes.c_void_p))
    s = apply_table(table, orc.stream_state(2024, 5))
    got = [xnext(s) for _ in range(4)]
    if J < 10 ** 6:
        want = [int(v) for v in orc.raw64(2024, 5, 4, skip=J)]
        assert got == want
    else:  # compose two smaller jumps instead of stepping 2^40 times
        half = np.empty(8192, np.uint32)
        call("msb_rng_jump_table", ctypes.c_uint64(J // 2), half.ctypes.data_as(ctypes.c_void_p))
        s2 = apply_table(half, apply_table(half, orc.stream_state(2024, 5)))
        if J % 2:
            xnext(s2)
        assert got == [xnext(s2) for _ in range(4)]


def test_power_tables_are_powers_of_two_jumps():
    pw = np.empty(64 * 8192, np.uint32)
    call("msb_rng_power_tables", pw.ctypes.data_as(ctypes.c_void_p))
    for b in (0, 1, 5, 17, 33, 63):
        one = np.empty(8192, np.uint32)
        call("msb_rng_jump_table", ctypes.c_uint64(1 << b), one.ctypes.data_as(ctypes.c_void_p))
        assert (pw[b * 8192:(b + 1) * 8192] == one).all()


def test_window_io_argument_errors():
    """msb_window_sweep rejects a malformed msb_window_io before any device
    work (host-side checks only; no GPU needed)."""
    from paper_2404_16990_b200._lib import Halo, SweepParams, WindowIO, MSB_MODE_FERRO, MSB_RNG_XOSHIRO
    L = _lib.lib()
    dummy = np.zeros(64, np.uint32)
    ptr = dummy.ctypes.data
    p = SweepParams(mode=MSB_MODE_FERRO, n_planes=2, thr9=ptr, kg=1, jump=ptr, work=ptr, rng=MSB_RNG_XOSHIRO)
    g = geom(2, 64, 1024)

    def sweep(g, first, count, io, halo=None, spins=ptr):
        P = 8 if g.ghost else 1  # slab windows need a row per piece
        return L.msb_window_sweep(ctypes.byref(g), ctypes.byref(p), 8, P, spins, ptr, ptr, first, count, ptr, ptr,
                                  ctypes.byref(halo) if halo is not None else None,
                                  ctypes.byref(io) if io is not None else None, None)

    cases = [
        (g, 0, 0, WindowIO(ptr, None, None, None), None, "needs a flip launch"),
        (g, 0, 8, WindowIO(None, ptr, ptr, None), None, "ups and unsat go together"),
        (geom(1, 64, 1024, row0=0, rows=16, ghost=1), 0, 8, WindowIO(ptr, None, None, None), None,
         "flip with an msb_halo"),
        (g, 0, 9, WindowIO(ptr, None, None, None), None, "outside the window"),
        (g, 0, 8, None, Halo(), "msb_halo needs a slab geometry"),
        (geom(1, 64, 1024, row0=0, rows=16, ghost=1), 0, 8, WindowIO(ptr, None, None, None),
         Halo(up_spins=ptr, down_spins=ptr, up_R=18, down_R=18, up_flags=ptr, down_flags=ptr),
         "slab launches need msb_sweep_params.flags"),
    ]
    for gg, first, count, io, halo, text in cases:
        assert sweep(gg, first, count, io, halo) == -1, text
        assert text in L.msb_last_error().decode()


def test_direct_sweep_host_checks():
    """msb_direct_ok / msb_flag_words / msb_direct_sweep argument
    handling (host logic only; no GPU needed): which shapes and tables take
    the direct path, and the errors raised before any device work."""
    from paper_2404_16990_b200._lib import (Halo, SweepParams, MSB_MODE_FERRO, MSB_MODE_GENERIC,
                                             MSB_RNG_PHILOX, MSB_RNG_PHILOX_BITS)
    L = _lib.lib()
    dummy = np.zeros(64, np.uint32)
    ptr = dummy.ctypes.data
    p = SweepParams(mode=MSB_MODE_FERRO, n_planes=2, thr9=ptr, kg=1, jump=ptr, work=ptr, rng=MSB_RNG_PHILOX_BITS)
    ok = lambda g, pp=p: L.msb_direct_ok(ctypes.byref(g), ctypes.byref(pp))
    # 32-draw rows (n/32 % 32 == 0) and n = 512 take it; other widths do not
    assert ok(geom(64, 1024, 1024)) == 1 and ok(geom(3, 512, 512)) == 1 and ok(geom(1, 64, 14336)) == 1
    assert ok(geom(2, 64, 96)) == 0 and ok(geom(2, 64, 160)) == 0
    # rows must split into bands of 2 rows x (32 / quads per row) lanes
    assert ok(geom(1, 12, 1024)) == 0
    # other streams and generic tables do not
    assert ok(geom(2, 64, 1024), SweepParams(mode=MSB_MODE_FERRO, n_planes=2, rng=MSB_RNG_PHILOX, work=ptr)) == 0
    assert ok(geom(2, 64, 1024), SweepParams(mode=MSB_MODE_GENERIC, n_planes=3, rng=MSB_RNG_PHILOX_BITS,
                                             work=ptr)) == 0
    # flag buffer: header + 2 halo slots per (replica, row segment) + one flag per
    # band group of the direct walk (2-row bands x 32/quads-per-row lanes)
    g = geom(64, 1024, 1024)
    assert L.msb_flag_words(ctypes.byref(g)) == 1 + 2 * 64 + 64 * 1024 // 16
    # n = 14336: 56 quads per row -> 7 segments of 8 quads, bands of 2 rows x 4 lanes
    assert L.msb_flag_words(ctypes.byref(geom(1, 64, 14336))) == 1 + 2 * 7 + 64 // 8 * 7
    # slab geometry: the held rows only
    assert L.msb_flag_words(ctypes.byref(geom(2, 64, 1024, row0=16, rows=32, ghost=1))) == 1 + 2 * 2 + 2 * 32 // 16
    # no band walk (12 rows do not split into 16-row groups): header + slots only
    assert L.msb_flag_words(ctypes.byref(geom(2, 12, 1024))) == 1 + 2 * 2
    assert L.msb_flag_words(ctypes.byref(geom(2, 10, 96))) == -1

    def sweep(gg, pp, n, spins=ptr, halo=None):
        return L.msb_direct_sweep(ctypes.byref(gg), ctypes.byref(pp), spins, n, ptr,
                                  ctypes.byref(halo) if halo is not None else None, None, None)

    assert sweep(g, p, 0) == 0                      # nothing to do
    px = SweepParams(mode=MSB_MODE_FERRO, n_planes=2, thr9=ptr, kg=1, work=ptr, rng=MSB_RNG_PHILOX)
    for gg, pp, n, spins, halo, text in [
        (g, px, 2, ptr, None, "bit-plane Philox stream"),
        (g, p, -1, ptr, None, "sweep count"),
        (g, p, 2, None, None, "null buffer"),
        (g, p, 2, ptr, Halo(), "msb_halo needs a slab geometry"),
        (geom(1, 64, 1024, row0=0, rows=32, ghost=1), p, 2, ptr,
         Halo(up_spins=ptr, down_spins=ptr, up_R=34, down_R=34, up_flags=ptr, down_flags=ptr),
         "need msb_sweep_params.flags"),
        (geom(2, 64, 96), p, 2, ptr, None, "direct sweeps need"),
    ]:
        assert sweep(gg, pp, n, spins, halo) < 0, text
        assert text in L.msb_last_error().decode(), (text, L.msb_last_error())


def test_ring_host_checks():
    """msb_window_sweep_ring / msb_direct_sweep_ring / msb_ring_ctx_bytes
    argument handling on the host (no GPU)."""
    from paper_2404_16990_b200._lib import (Halo, RingSlab, SweepParams, MSB_MODE_FERRO, MSB_RNG_PHILOX_BITS,
                                             MSB_RNG_XOSHIRO)
    L = _lib.lib()
    assert L.msb_ring_ctx_bytes(0) == -1 and L.msb_ring_ctx_bytes(17) == -1
    one = L.msb_ring_ctx_bytes(1)
    assert one > 0 and L.msb_ring_ctx_bytes(8) == 8 * one
    dummy = np.zeros(64, np.uint32)
    ptr = dummy.ctypes.data
    arr = (RingSlab * 2)()
    assert L.msb_window_sweep_ring(0, arr, 8, 8, 0, 8, ptr, None) == -1
    assert "ring of 1..MSB_RING_MAX" in L.msb_last_error().decode()
    px = SweepParams(mode=MSB_MODE_FERRO, n_planes=2, thr9=ptr, kg=1, jump=ptr, work=ptr, rng=MSB_RNG_XOSHIRO,
                     flags=ptr)
    pb = SweepParams(mode=MSB_MODE_FERRO, n_planes=2, thr9=ptr, kg=1, jump=ptr, work=ptr, rng=MSB_RNG_PHILOX_BITS,
                     flags=ptr)
    g0, g1 = geom(1, 64, 1024, row0=0, rows=32, ghost=1), geom(1, 64, 1024, row0=32, rows=32, ghost=1)
    h = Halo(up_spins=ptr, down_spins=ptr, up_R=34, down_R=34, up_flags=ptr, down_flags=ptr)
    for v, (g, p) in enumerate(((g0, px), (g1, pb))):
        arr[v].g, arr[v].p, arr[v].spins, arr[v].flips = ctypes.pointer(g), ctypes.pointer(p), ptr, ptr
        arr[v].halo = ctypes.pointer(h)
    assert L.msb_window_sweep_ring(2, arr, 8, 8, 0, 8, ptr, None) == -1
    assert "share the stream kind" in L.msb_last_error().decode()
    arr[1].p = ctypes.pointer(px)
    assert L.msb_window_sweep_ring(2, arr, 8, 8, 0, 8, None, None) == -1
    assert "null ring context" in L.msb_last_error().decode()
    assert L.msb_direct_sweep_ring(2, arr, 2, None, None) == -1
