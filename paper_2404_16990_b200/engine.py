"""Drop-in B200 ``Engine`` / ``run_simulations`` for the reference `multispin`.

Same constructor, methods, attributes, counters and error behaviour as the
reference engine (pkg/src/multispin/engine.py:216-492), but the spins live
on the GPU in a colour-split bit layout and the sweeps run as sm_100a
kernels (libmsb200, include/msb200.h).  Steady state (``run`` / ``_sweeps``
with FERRO/ANTI tables): lookahead windows, ONE cooperative launch per
window of S sweeps (64 by default for whole lattices; ``run`` fits it to its
measurement interval) in which producer warps turn the next window's reference xoshiro256++
draws into accept bit planes while the other warps flip this window's
sweeps with bit-sliced neighbour logic (msb_window_sweep); the bit-plane
counter stream flips without planes (msb_direct_sweep).  ``flip_red`` /
``flip_blue`` alone, forced generic tables, host-supplied ``streams`` and the
recorder take the per-phase kernels (msb_phase).  Results are bit-identical
to the reference on identical seeds, dimensions, temperatures and couplings.

Reference surfaces kept (file:line in pkg/src/multispin/engine.py):
  ``Engine(dims, temperatures, seed, init, coupling, sim_offset)`` 238-272
  ``from_lattices``                                               284-300
  ``update_red_bc`` / ``update_blue_bc`` (called from ``sweep``)    304-310
  ``flip_red`` / ``flip_blue`` / ``sweep``                          345-360
  ``packed`` / ``lattice`` / ``abs_magnetization`` /
  ``energy_per_spin`` / ``halo_mismatches``                         364-397
  ``run`` -> ``Trajectory``                                        401-440
  ``run_simulations``                                              443-492
  attributes ``dims temperatures n_sim seed coupling sim_offset init state
  _tables streams sweeps_done attempts flips recorder``.
``state`` is a host mirror of the device spins in the reference's uint16
layout: reading it materialises the eight arrays with halos; in-place edits
are detected and written back before the next device operation.
"""

from __future__ import annotations

import ctypes
import math
import threading
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import _lib
from ._lib import (call, geom, MsbError, SweepParams, WindowIO, MSB_FLIP_SLOTS, MSB_MAX_PLANES, MSB_MODE_GENERIC,
                   MSB_RNG_PHILOX, MSB_RNG_XOSHIRO, RNG_MODES, MSB_SWEEP_AHEAD_IN, MSB_SWEEP_AHEAD_OUT, MSB_SWEEP_SERIAL)
from .layout import (
    ALL_CODES, ArrayCode, LatticeDims, PackedArrays, check_spins, halo_audit_index, unpack,
)
from .observables import Trajectory
from .rng import DeviceStreams, PhiloxBitStreams, PhiloxStreams

__all__ = ["FLIP_RED", "FLIP_BLUE", "build_exp_table", "Engine", "run_simulations"]

_C = ArrayCode
# (target, lateral source, vertical source, up, right) -- engine.py:57-68.
# The order is the RNG consumption order of a colour phase.
FLIP_RED = (
    (_C.RFE, _C.BFE, _C.BFO, False, False),
    (_C.RBO, _C.BBO, _C.BBE, True, False),
    (_C.RBE, _C.BBE, _C.BBO, False, True),
    (_C.RFO, _C.BFO, _C.BFE, True, True),
)
FLIP_BLUE = (
    (_C.BFE, _C.RFE, _C.RFO, False, True),
    (_C.BBO, _C.RBO, _C.RBE, True, True),
    (_C.BBE, _C.RBE, _C.RBO, False, False),
    (_C.BFO, _C.RFO, _C.RFE, True, False),
)

_M64 = (1 << 64) - 1
_UNIT = 2.0 ** -23


def build_exp_table(T: float, J: float = 1.0) -> np.ndarray:
    """Acceptance table indexed by 8*own + n_up (engine.py:78-94): flipping a
    spin of sign s with u of 4 neighbours up costs 2 J s (2u - 4); the entry
    is min(1, exp(-cost/T)) with CPython's math.exp (bit-identical doubles);
    impossible up-counts 5..7 stay 0."""
    if T <= 0:
        raise ValueError("temperature must be positive")
    table = np.zeros(16, dtype=np.float64)
    for own in (0, 1):
        s = 2 * own - 1
        for u in range(5):
            cost = 2.0 * J * s * (2 * u - 4)
            table[8 * own + u] = 1.0 if cost <= 0 else math.exp(-cost / T)
    return table


# ---------------------------------------------------------------------------
# per-device read-only tables (built once per process and device)
# ---------------------------------------------------------------------------

_TABLE_LOCK = threading.Lock()
_POW_HOST: np.ndarray | None = None
_DEV_TABLES: dict = {}


def _torch():
    import torch
    return torch


def _resolve_device(device):
    torch = _torch()
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2404_16990_b200.Engine needs a CUDA device (B200); "
                           "there is no CPU fallback")
    _lib.lib()  # fail loudly now if the native library is missing
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    dev = torch.device(device)
    if dev.type != "cuda":
        raise ValueError(f"device must be a CUDA device, got {dev}")
    return torch.device("cuda", dev.index if dev.index is not None else torch.cuda.current_device())


def _upload_shared(host_tensor, device):
    """Device copy of a table every engine of the process shares.  The copy
    runs on whatever stream is current; engines read the table on their own
    (non-blocking) streams, so it is completed here, once, before any of them
    can see it."""
    torch = _torch()
    dev = host_tensor.to(device)
    torch.cuda.current_stream(device).synchronize()
    return dev


def _pow_tables(device):
    """Device copy of the 64 nibble tables of A^(2^b) (2 MiB)."""
    global _POW_HOST
    torch = _torch()
    with _TABLE_LOCK:
        key = ("pow", device.index)
        if key not in _DEV_TABLES:
            if _POW_HOST is None:
                host = np.empty(64 * 8192, np.uint32)
                call("msb_rng_power_tables", host.ctypes.data_as(ctypes.c_void_p))
                _POW_HOST = host
            _DEV_TABLES[key] = _upload_shared(torch.from_numpy(_POW_HOST.view(np.int32)), device)
        return _DEV_TABLES[key]


def _jump_table(device, distance: int):
    """Device nibble table of A^distance (32 KiB), cached per device."""
    torch = _torch()
    with _TABLE_LOCK:
        key = ("jump", device.index, distance)
        if key not in _DEV_TABLES:
            host = np.empty(8192, np.uint32)
            call("msb_rng_jump_table", ctypes.c_uint64(distance), host.ctypes.data_as(ctypes.c_void_p))
            _DEV_TABLES[key] = _upload_shared(torch.from_numpy(host.view(np.int32)), device)
        return _DEV_TABLES[key]


def _sweep_jump_table(device, n: int):
    """Device nibble table of A^(4n): advances a stream piece by one sweep."""
    return _jump_table(device, 4 * n)


def _p(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr())


class Engine:
    """Packed checkerboard Metropolis over ``n_sim`` replicas on one GPU.

    Extra keyword-only arguments beyond the reference signature:
    ``device`` (CUDA device; default current), ``kg`` (stream pieces per
    target row, 1/2/4/8/16, for the per-phase path; default chosen by the
    library), ``window`` (sweeps of accept planes generated per launch on the
    steady-state path, ``msb_window_sweep``; default chosen by the library)
    and ``stream``:
    "xoshiro" (default) draws the reference's own xoshiro256++ streams;
    "philox" draws the counter-based ``rng.PhiloxStreams``, which
    the reference Engine reproduces bit-exactly when handed the same object
    as its ``streams``; "philox-bits" draws ``rng.PhiloxBitStreams``, the
    bit-plane form whose comparisons the GPU resolves from the most
    significant plane down, generating only the planes they need.
    """

    def __init__(self, dims: LatticeDims, temperatures, seed: int, init: str = "random",
                 coupling: float = 1.0, sim_offset: int = 0, *, device=None, kg: int | None = None,
                 window: int | None = None, stream: str = "xoshiro"):
        self.dims = dims
        self.temperatures = tuple(float(t) for t in temperatures)
        if not self.temperatures:
            raise ValueError("need at least one simulation temperature")
        self.n_sim = len(self.temperatures)
        self.seed = int(seed)
        self.coupling = float(coupling)
        self.sim_offset = int(sim_offset)
        self.init = init
        self._tables = np.stack([build_exp_table(t, coupling) for t in self.temperatures])
        if init not in ("random", "all-up"):
            raise ValueError(f"unknown init mode {init!r} (expected 'random' or 'all-up')")
        if stream not in RNG_MODES:
            raise ValueError(f"unknown stream {stream!r} (expected 'xoshiro', 'philox' or 'philox-bits')")
        self.stream = stream

        torch = _torch()
        self.device = _resolve_device(device)
        self._stream = torch.cuda.Stream(device=self.device)
        self._cs = ctypes.c_void_p(self._stream.cuda_stream)
        self._g = geom(self.n_sim, dims.m, dims.n, sim_offset=self.sim_offset)
        call("msb_check_geom", ctypes.byref(self._g))
        self.kg = int(kg) if kg is not None else int(_lib.lib().msb_default_kg(ctypes.byref(self._g)))
        self._words_per_sim = int(_lib.lib().msb_spin_words(ctypes.byref(self._g))) // self.n_sim
        n_pieces = int(_lib.lib().msb_pieces_per_phase(ctypes.byref(self._g), self.kg))
        with torch.cuda.device(self.device), torch.cuda.stream(self._stream):
            self._spins = torch.empty(self._words_per_sim * self.n_sim, dtype=torch.int32, device=self.device)
            self._states = torch.empty(2 * 8 * n_pieces, dtype=torch.int32, device=self.device)
            self._thr = torch.zeros(MSB_MAX_PLANES * self.n_sim, dtype=torch.int32, device=self.device)
            self._flips_dev = torch.zeros(MSB_FLIP_SLOTS, dtype=torch.int64, device=self.device)
            # per-phase / per-sweep path planes (2 buffers of up to 10 planes):
            # allocated on first use, the window path has its own
            self._plane_words = int(_lib.lib().msb_plane_words(ctypes.byref(self._g), MSB_MAX_PLANES))
            self._planes_t = None
            self._work = torch.zeros(4, dtype=torch.int32, device=self.device)
            self._obs = torch.zeros(2 * self.n_sim, dtype=torch.int64, device=self.device)
            # band-group phase flags of the window / direct launches (header word
            # advanced by the launches themselves, include/msb200.h)
            self._flags = torch.zeros(int(_lib.lib().msb_flag_words(ctypes.byref(self._g))), dtype=torch.int32,
                                      device=self.device)
        self._fphases = 0  # phases launched on _flags (re-zeroed long before the uint32 counters wrap)
        self._pow = _pow_tables(self.device)
        self._jump = _sweep_jump_table(self.device, dims.n)
        self._params = SweepParams()
        self._params.kg = self.kg
        self._params.jump = self._jump.data_ptr()
        self._params.thr9 = self._thr.data_ptr()
        self._params.work = self._work.data_ptr()
        self._params.rng = RNG_MODES[stream]
        self._params.seed = self.seed & _M64
        self._params.flags = self._flags.data_ptr()
        self._tab_key = None
        self.fault = 0  # test-only adder corruption (selftest seam, cli.py:467-480)
        self.overlap = True  # run the next sweep's RNG concurrently with this sweep's flips
        S, P = ctypes.c_int32(), ctypes.c_int32()
        call("msb_default_window", ctypes.byref(self._g), ctypes.byref(S), ctypes.byref(P))
        self.window, self._wP = int(S.value), int(P.value)
        self._window_user = window is not None
        self._window_default = self.window
        if window is not None:
            self.window = int(window)
            if not 1 <= self.window <= 64:
                raise ValueError("window must be in [1, 64] sweeps")
            self._wP = int(_lib.lib().msb_window_parts(ctypes.byref(self._g), self.window))
        self._wbuf = None       # (states, planes[2], jump table) of the window path, allocated on first use
        self._wvalid = False    # window buffer _wcur holds slots [_wc, S) of the window at block _wbase
        self._wcur = 0
        self._wc = 0
        self._wbase = 0
        self._wkey = None

        if init == "random":
            with torch.cuda.stream(self._stream):
                scratch = torch.empty(self.n_sim * dims.sites // 64, dtype=torch.int64, device=self.device)
            call("msb_init_random", ctypes.byref(self._g), ctypes.c_uint64(self.seed & _M64), _p(self._pow),
                 _p(scratch), _p(self._spins), self._cs)
            scratch.record_stream(self._stream)
            del scratch
        else:
            call("msb_init_const", ctypes.byref(self._g), 1, _p(self._spins), self._cs)
        if stream == "xoshiro":
            call("msb_rng_init", ctypes.byref(self._g), ctypes.c_uint64(self.seed & _M64), self.kg,
                 ctypes.c_uint64(0), -1, _p(self._pow), _p(self._states), self._cs)
            self.streams = DeviceStreams(self.seed, self.n_sim * dims.cells, self.sim_offset * dims.cells)
        else:
            cls = PhiloxStreams if stream == "philox" else PhiloxBitStreams
            self.streams = cls(self.seed, self.n_sim * dims.cells, self.sim_offset * dims.cells)
        self._own_streams = self._streams
        self._blocks = 0        # stream blocks consumed (one per colour phase)
        self._pos = [0, 1]      # block each colour's pieces are positioned at
        self._ahead = False     # next sweep's accept planes already generated (states one sweep on)
        self._ahead_key = None
        self._cur = 0           # plane buffer holding the lookahead
        self._ver = 0           # device-state version
        self._mirror = None     # host uint16 state mirror
        self._mirror_snap = None
        self._mirror_ver = -1
        self._obs_ver = -1
        self._obs_host = None

        self.sweeps_done = 0
        self.attempts = 0
        self._flips_base = 0
        self.recorder = None
        self.update_red_bc()
        self.update_blue_bc()

    @property
    def streams(self):
        """The flip streams (reference seam, engine.py:259-261, 336).  The
        engine's own counter-based stream object is returned positioned at
        the draws the device has consumed (64 * words per stream and colour
        phase), so it can continue this run on the reference Engine."""
        s = self._streams
        if s is getattr(self, "_own_streams", None) and hasattr(s, "position"):
            s.position = self._blocks * 64 * self.dims.words
        return s

    @streams.setter
    def streams(self, value) -> None:
        self._streams = value

    @property
    def _planes(self):
        if self._planes_t is None:
            torch = _torch()
            with torch.cuda.device(self.device), torch.cuda.stream(self._stream):
                self._planes_t = torch.empty(2 * self._plane_words, dtype=torch.int32, device=self.device)
        return self._planes_t

    # -- construction from explicit lattices (engine.py:284-300) -------------

    @classmethod
    def from_lattices(cls, lattices, temperatures, seed: int, coupling: float = 1.0,
                      sim_offset: int = 0, **kw) -> "Engine":
        lattices = [np.asarray(l) for l in lattices]
        dims = check_spins(lattices[0])
        eng = cls(dims, temperatures, seed, init="all-up", coupling=coupling, sim_offset=sim_offset, **kw)
        if len(lattices) != eng.n_sim:
            raise ValueError("one lattice per temperature required")
        for spins in lattices:
            if check_spins(spins) != dims:
                raise ValueError("all lattices must share the same dims")
        eng._upload_lattices(lattices)
        eng.update_red_bc()
        eng.update_blue_bc()
        return eng

    def _upload_lattices(self, lattices) -> None:
        torch = _torch()
        lin = np.stack([np.packbits(np.asarray(l).reshape(-1) > 0, bitorder="little") for l in lattices])
        with torch.cuda.stream(self._stream):
            dev = torch.from_numpy(lin.view(np.int64).copy()).to(self.device, non_blocking=False)
        call("msb_from_linear", ctypes.byref(self._g), _p(dev), _p(self._spins), self._cs)
        self._stream.synchronize()
        self._touch()

    # -- boundary updates (engine.py:304-310) ----------------------------------

    def update_red_bc(self) -> None:
        """Halo/moat refresh of the red arrays.  On the GPU periodicity is
        index arithmetic inside the kernels, so there is nothing to copy; the
        call is kept so wrappers around it (test_acceptance.py:59-69) see the
        same two updates per sweep as the reference."""

    def update_blue_bc(self) -> None:
        """See ``update_red_bc``."""

    # -- thresholds (engine.py:257, 321-331) ---------------------------------

    def _sync_tables(self) -> None:
        tab = np.ascontiguousarray(self._tables, dtype=np.float64)
        if tab.shape != (self.n_sim, 16):
            raise ValueError(f"_tables must have shape {(self.n_sim, 16)}")
        key = tab.tobytes()
        if key == self._tab_key:
            return
        mode, npl = ctypes.c_int32(), ctypes.c_int32()
        codes = (ctypes.c_int8 * 16)()
        thr = np.zeros(MSB_MAX_PLANES * self.n_sim, np.uint32)
        call("msb_plan_thresholds", tab.ctypes.data_as(ctypes.c_void_p), self.n_sim, ctypes.byref(mode),
             ctypes.byref(npl), codes, thr.ctypes.data_as(ctypes.c_void_p))
        torch = _torch()
        with torch.cuda.stream(self._stream):
            self._thr.copy_(torch.from_numpy(thr.view(np.int32)))
        self._stream.synchronize()
        self._params.mode = mode.value
        self._params.n_planes = npl.value
        self._params.code_plane[:] = list(codes)
        self._tab_key = key

    @property
    def flip_mode(self) -> int:
        self._sync_tables()
        return int(self._params.mode)

    # -- host mirror of the reference state layout ---------------------------

    def _touch(self) -> None:
        self._ver += 1

    def _push_host_edits(self) -> None:
        m = self._mirror
        if m is not None and self._mirror_ver == self._ver and not np.array_equal(m, self._mirror_snap):
            self._upload_state(m)

    def _upload_state(self, arr: np.ndarray) -> None:
        torch = _torch()
        with torch.cuda.stream(self._stream):
            dev = torch.from_numpy(np.ascontiguousarray(arr).view(np.int16)).to(self.device)
        call("msb_from_ref16", ctypes.byref(self._g), _p(dev), _p(self._spins), self._cs)
        self._stream.synchronize()
        self._touch()

    @property
    def state(self) -> np.ndarray:
        """uint16 (n_sim, 8, cells+2, words+2) view in the reference layout."""
        if self._mirror is not None and self._mirror_ver == self._ver:
            return self._mirror
        torch = _torch()
        d = self.dims
        shape = (self.n_sim, len(ALL_CODES), d.cols, d.vec_len)
        with torch.cuda.stream(self._stream):
            dev = torch.empty(int(np.prod(shape)), dtype=torch.int16, device=self.device)
        call("msb_to_ref16", ctypes.byref(self._g), _p(self._spins), _p(dev), self._cs)
        self._stream.synchronize()
        host = dev.cpu().numpy().view(np.uint16).reshape(shape)
        if self._mirror is not None and self._mirror.shape == shape:
            self._mirror[...] = host
        else:
            self._mirror = host.copy()
        self._mirror_snap = host
        self._mirror_ver = self._ver
        return self._mirror

    @state.setter
    def state(self, value) -> None:
        d = self.dims
        arr = np.asarray(value)
        shape = (self.n_sim, len(ALL_CODES), d.cols, d.vec_len)
        if arr.shape != shape or arr.dtype != np.uint16:
            raise ValueError(f"expected uint16 state of shape {shape}, got {arr.dtype} {arr.shape}")
        self._upload_state(arr)

    # -- flips (engine.py:314-360) -------------------------------------------

    def _host_draws(self, phase: int):
        """Draws from a user-supplied ``streams`` object (duck-typed seam,
        engine.py:336): u23 integers in the reference block order."""
        torch = _torch()
        d = self.dims
        block = np.asarray(self._streams.unit_block(4 * 16 * d.words), dtype=np.float64)
        expect = (4 * 16 * d.words, self.n_sim * d.cells)
        if block.shape != expect:
            raise ValueError(f"streams.unit_block returned {block.shape}, expected {expect}")
        u = block * (1 << 23)
        k = np.floor(u)
        if not ((k == u) & (block >= 0.0) & (block < 1.0)).all():
            raise ValueError("host draws must be multiples of 2**-23 in [0, 1) (rng.py:113-115 shaping)")
        draws = np.ascontiguousarray(k.T.astype(np.uint32))  # (n_sim*cells, 64*words) = block order
        with torch.cuda.stream(self._stream):
            return torch.from_numpy(draws.view(np.int32).reshape(-1)).to(self.device)

    def _record(self, phase: int) -> None:
        """Feed the recorder hook exactly as engine.py:327-328 does."""
        torch = _torch()
        d = self.dims
        with torch.cuda.stream(self._stream):
            out = torch.empty(self.n_sim * d.cells * 64 * d.words, dtype=torch.int32, device=self.device)
        call("msb_draws", ctypes.byref(self._g), ctypes.byref(self._params), phase, _p(self._states), _p(out),
             self._cs)
        self._stream.synchronize()
        draws = out.cpu().numpy().view(np.uint32).reshape(self.n_sim, d.cells, 4, 16, d.words)
        quarters = FLIP_RED if phase == 0 else FLIP_BLUE
        for q, (target, *_rest) in enumerate(quarters):
            for i in range(4):
                for ii in range(4):
                    r = draws[:, :, q, 4 * i + ii, :].astype(np.float64) * _UNIT
                    self.recorder.record(self.sweeps_done, target, 4 * ii + i, r)

    def _drop_ahead(self) -> None:
        """Discard pre-generated planes: put the stream pieces back at the
        logical position (the next unconsumed block)."""
        self._wvalid = False
        if self._ahead:
            if self.stream == "xoshiro":
                call("msb_rng_init", ctypes.byref(self._g), ctypes.c_uint64(self.seed & _M64), self.kg,
                     ctypes.c_uint64(self._blocks), -1, _p(self._pow), _p(self._states), self._cs)
            self._pos = [self._blocks, self._blocks + 1]
            self._ahead = False

    def _phase(self, phase: int) -> None:
        self._drop_ahead()
        self._push_host_edits()
        self._sync_tables()
        self._params.fault = int(bool(self.fault))
        h = self._blocks
        ext = None
        self._params.block = h
        if self._streams is not self._own_streams:
            ext = self._host_draws(phase)
            self._pos[phase] = None
        else:
            if self.stream == "xoshiro" and self._pos[phase] != h:
                call("msb_rng_init", ctypes.byref(self._g), ctypes.c_uint64(self.seed & _M64), self.kg,
                     ctypes.c_uint64(h), phase, _p(self._pow), _p(self._states), self._cs)
            if self.recorder is not None:
                self._record(phase)
        call("msb_phase", ctypes.byref(self._g), ctypes.byref(self._params), phase, _p(self._spins),
             _p(self._states), _p(ext) if ext is not None else None, _p(self._planes), _p(self._flips_dev),
             self._cs)
        if ext is not None:
            ext.record_stream(self._stream)
        else:
            self._pos[phase] = h + 2
        self._blocks += 1
        self._touch()

    def flip_red(self) -> None:
        """Attempt every red spin once."""
        self._phase(0)

    def flip_blue(self) -> None:
        """Attempt every blue spin once."""
        self._phase(1)

    def sweep(self) -> None:
        """One full sweep: red flips, red copies, blue flips, blue copies."""
        self.flip_red()
        self.update_red_bc()
        self.flip_blue()
        self.update_blue_bc()
        self.sweeps_done += 1
        self.attempts += self.dims.sites * self.n_sim

    def _fast_path_ok(self) -> bool:
        cls = type(self)
        for name in ("sweep", "flip_red", "flip_blue", "update_red_bc", "update_blue_bc"):
            if name in self.__dict__ or getattr(cls, name) is not getattr(Engine, name):
                return False
        return self.recorder is None and self._streams is self._own_streams

    def _sweeps(self, k: int, io=None) -> None:
        """k sweeps through the library, no host sync: lookahead windows
        (FERRO/ANTI tables) or the per-sweep fused path (generic tables,
        ``overlap = False``).  ``io``: a WindowIO for the window path
        (step_packed; the caller checked ``_window_route``)."""
        if k <= 0:
            return
        if io is not None and not self._window_route():
            raise RuntimeError("msb_window_io outside the window path")
        if not self._fast_path_ok():
            for _ in range(k):
                self.sweep()
            return
        self._push_host_edits()
        self._sync_tables()
        self._params.fault = int(bool(self.fault))
        if self.overlap and self._params.mode != MSB_MODE_GENERIC:
            if self._direct_ok():
                self._direct_sweeps(k, io)
            else:
                self._win_sweeps(k, io)
        elif self._pos == [self._blocks, self._blocks + 1] or self._ahead:
            self._sweep_call(k)
        else:  # per-phase positioning pending (a lone flip_red/flip_blue)
            for _ in range(k):
                self.sweep()
            return
        self.sweeps_done += k
        self.attempts += self.dims.sites * self.n_sim * k
        self._touch()

    # -- direct sweeps (msb_direct_sweep, bit-plane Philox stream) --------------

    def _direct_ok(self) -> bool:
        """The bit-plane stream with FERRO/ANTI tables flips without accept
        planes: every warp flips and draws only the bit planes its Metropolis
        tests need (msb_direct_sweep)."""
        return self.stream == "philox-bits" and bool(
            _lib.lib().msb_direct_ok(ctypes.byref(self._g), ctypes.byref(self._params)))

    def _direct_sweeps(self, k: int, io=None) -> None:
        """k sweeps in launches of up to ``window`` sweeps; with ``io`` the
        load goes with the first launch, the export with the last.  Phases
        are ordered by band-group flags (``_flags``)."""
        self._wvalid = False       # windows and per-sweep lookahead planes are stale now
        self._ahead = False
        first = True
        while k > 0:
            r = min(k, self.window)
            lio = None
            if io is not None:
                lio = WindowIO(io.lin_in if first else None, None, None, None)
                if r == k:
                    lio.lin_out, lio.ups, lio.unsat = io.lin_out, io.ups, io.unsat
            first = False
            self._params.block = self._blocks
            self._flag_phases(2 * r)
            call("msb_direct_sweep", ctypes.byref(self._g), ctypes.byref(self._params), _p(self._spins), r,
                 _p(self._flips_dev), None, ctypes.byref(lio) if lio is not None else None, self._cs)
            self._blocks += 2 * r
            k -= r
        self._pos = [self._blocks, self._blocks + 1]  # counter-based: the per-phase path needs no positioning

    def _flag_phases(self, phases: int) -> None:
        """Account for a flag launch of `phases` colour phases; the uint32
        counters are re-zeroed (stream-ordered) long before they could wrap."""
        if self._fphases + phases >= 1 << 31:
            with _torch().cuda.stream(self._stream):
                self._flags.zero_()
            self._fphases = 0
        self._fphases += phases

    # -- lookahead windows (msb_window_sweep) ------------------------------------

    def _win_alloc(self):
        if self._wbuf is None:
            torch = _torch()
            S, P = self.window, self._wP
            npieces = int(_lib.lib().msb_window_pieces(ctypes.byref(self._g), S, P))
            words = int(_lib.lib().msb_window_words(ctypes.byref(self._g), S))
            if npieces < 0 or words < 0:
                raise MsbError(f"window S={S}, P={P} unsupported: {_lib.lib().msb_last_error().decode()}")
            with torch.cuda.device(self.device), torch.cuda.stream(self._stream):
                states = torch.empty(8 * npieces, dtype=torch.int32, device=self.device)
                planes = torch.empty(2 * words, dtype=torch.int32, device=self.device)
            jump = _jump_table(self.device, S * 4 * self.dims.n)
            self._wbuf = (states, planes, words, jump)
        return self._wbuf

    @property
    def _io_groups_ok(self) -> bool:
        """msb_window_io works in groups of 4 chunks of 1024 sites, with
        fewer than 2^31 / 32 chunks (make_win_io, msb_window.cuh)."""
        chunks = self.n_sim * self.dims.m * -(-self.dims.n // 1024)
        return (self.dims.m * -(-self.dims.n // 1024)) % 4 == 0 and 32 * chunks < (1 << 31)

    def _fit_window(self, interval: int, n_sweeps: int) -> None:
        """Window length for measurements every `interval` sweeps (unless the
        caller chose the window).  A measurement that falls inside a window
        splits it, and the launch flipping the remainder runs without
        production, outside the producers' shadow.  So take the longest power
        of two in [8, default] whose remainder is at most 1/16 of the
        interval (cfg2: interval 8 at S = 64 0.75 T, at S = 8 0.92; 100 at S
        = 64 0.87-0.91, at S = 32 0.92), and start the run on a window
        boundary when measurements would otherwise fall inside windows all
        along it.  Powers of two keep the producer units in whole rounds on
        148 SMs; the sweeps do not depend on the window."""
        if self._window_user or not self._window_route() or self._direct_ok():
            return
        S = self._window_default
        if S >= 8:
            while S > 8 and interval % S > interval / 16:
                S //= 2
        if S != self.window:
            P = int(_lib.lib().msb_window_parts(ctypes.byref(self._g), S))
            if P <= 0:
                return
            self.window, self._wP = S, P
            self._wbuf = None
            self._wvalid = False
            self.__dict__.pop("_io_fused", None)  # its producer-round rule depends on the window
        elif self._wvalid and self._wc and interval % S == 0 and n_sweeps >= 2 * S:
            self._wvalid = False  # realign: the window restarts at the next sweep

    def _win_launch(self, first: int, count: int, produce: bool, io=None) -> None:
        states, planes, words, jump = self._wbuf
        cur = planes[self._wcur * words:(self._wcur + 1) * words]
        nxt = planes[(1 - self._wcur) * words:(2 - self._wcur) * words]
        if count == 0:      # produce into the current buffer
            nxt, cur = cur, None
        self._params.jump = jump.data_ptr()
        # Philox: block of the produced window's slot 0
        self._params.block = self._wbase if count == 0 else self._wbase + 2 * self.window
        self._flag_phases(2 * count)
        call("msb_window_sweep", ctypes.byref(self._g), ctypes.byref(self._params), self.window, self._wP,
             _p(self._spins), _p(states), _p(cur) if cur is not None else None, first, count,
             _p(nxt) if produce else None, _p(self._flips_dev), None,
             ctypes.byref(io) if io is not None else None, self._cs)
        self._params.jump = self._jump.data_ptr()

    def _win_sweeps(self, k: int, io=None) -> None:
        self._win_alloc()
        S = self.window
        if self._wvalid and (self._wkey != self._tab_key or self._wbase + 2 * self._wc != self._blocks):
            self._wvalid = False
        if not self._wvalid:
            # position the window's pieces at the next unconsumed block and
            # generate its planes (the per-phase states are left behind)
            self._wbase, self._wc, self._wcur = self._blocks, 0, 0
            if self.stream == "xoshiro":
                call("msb_window_init", ctypes.byref(self._g), ctypes.c_uint64(self.seed & _M64), S, self._wP,
                     ctypes.c_uint64(self._wbase), _p(self._pow), _p(self._wbuf[0]), self._cs)
            self._win_launch(0, 0, True)
            self._wvalid, self._wkey = True, self._tab_key
        self._ahead = False
        self._pos = [None, None]   # per-phase pieces must be re-positioned before a lone phase
        first_launch = True
        while k > 0:
            r = min(k, S - self._wc)
            finish = self._wc + r == S
            lio = None
            if io is not None:  # the load goes with the first flip launch, the export with the last
                lio = WindowIO(io.lin_in if first_launch else None, None, None, None)
                if r == k:
                    lio.lin_out, lio.ups, lio.unsat = io.lin_out, io.ups, io.unsat
            first_launch = False
            self._win_launch(self._wc, r, finish, lio)
            self._blocks += 2 * r
            k -= r
            if finish:
                self._wcur, self._wc, self._wbase = 1 - self._wcur, 0, self._wbase + 2 * S
            else:
                self._wc += r

    def _sweep_call(self, k: int) -> None:
        if self._ahead and self._ahead_key != self._tab_key:
            self._drop_ahead()
        flags = MSB_SWEEP_AHEAD_OUT | (MSB_SWEEP_AHEAD_IN if self._ahead else 0)
        if not self.overlap:
            flags |= MSB_SWEEP_SERIAL
        cur = ctypes.c_int32(self._cur)
        self._params.block = self._blocks + (2 if self._ahead else 0)
        call("msb_sweep", ctypes.byref(self._g), ctypes.byref(self._params), _p(self._spins),
             _p(self._states), _p(self._planes), k, flags, ctypes.byref(cur), _p(self._flips_dev), self._cs)
        self._cur = cur.value
        self._ahead = True
        self._ahead_key = self._tab_key
        self._blocks += 2 * k
        self._pos = [self._blocks, self._blocks + 1]

    def _timed_sweeps(self, k: int, ev0, ev1) -> None:
        """k sweeps of the fast path bracketed by CUDA events on the engine's
        stream (bench.py).  With k = window and an aligned window this is one
        launch: the flips of k sweeps plus the planes of the next k."""
        if not self._fast_path_ok():
            raise RuntimeError("timed sweeps need the engine's own sweep path")
        self._push_host_edits()
        self._sync_tables()
        self._params.fault = int(bool(self.fault))
        ev0.record(self._stream)
        if self.overlap and self._params.mode != MSB_MODE_GENERIC:
            if self._direct_ok():
                self._direct_sweeps(k)
            else:
                self._win_sweeps(k)
        else:
            self._sweep_call(k)
        ev1.record(self._stream)
        self.sweeps_done += k
        self.attempts += self.dims.sites * self.n_sim * k
        self._touch()

    def synchronize(self) -> None:
        self._stream.synchronize()
        if hasattr(self, "_io"):
            self._in_stream.synchronize()
            self._out_stream.synchronize()
            self._host_out.clear()

    @property
    def flips(self) -> int:
        """Accepted flips so far (engine.py:331-332); synchronises the stream."""
        self._stream.synchronize()
        return self._flips_base + int(self._flips_dev.sum().item())

    @flips.setter
    def flips(self, value: int) -> None:
        self._stream.synchronize()
        self._flips_base = int(value) - int(self._flips_dev.sum().item())

    # -- observables (engine.py:364-397) ---------------------------------------

    def packed(self, sim: int) -> PackedArrays:
        return PackedArrays(self.dims, self.state[sim])

    def lattices(self) -> np.ndarray:
        """All replicas' +/-1 lattices, int8 (n_sim, m, n)."""
        return self._lattice_range(0, self.n_sim)

    def lattice(self, sim: int) -> np.ndarray:
        """Unpacked +/-1 lattice of one replica (engine.py:368-370)."""
        if not -self.n_sim <= sim < self.n_sim:
            raise IndexError(f"simulation {sim} out of range")
        sim %= self.n_sim
        return self._lattice_range(sim, sim + 1)[0]

    def _lattice_range(self, lo: int, hi: int) -> np.ndarray:
        self._push_host_edits()
        torch = _torch()
        d = self.dims
        g = geom(hi - lo, d.m, d.n, sim_offset=self.sim_offset + lo)
        with torch.cuda.stream(self._stream):
            lin = torch.empty((hi - lo) * d.sites // 64, dtype=torch.int64, device=self.device)
        base = ctypes.c_void_p(self._spins.data_ptr() + 4 * lo * self._words_per_sim)
        call("msb_to_linear", ctypes.byref(g), base, _p(lin), self._cs)
        self._stream.synchronize()
        bits = np.unpackbits(lin.cpu().numpy().view(np.uint8), bitorder="little")
        return np.where(bits == 1, 1, -1).astype(np.int8).reshape(hi - lo, d.m, d.n)

    # -- host-buffer interop (bit-packed lattices) -----------------------------

    def packed_nbytes(self) -> int:
        """Bytes of all replicas' lattices as bit-packed linear sites."""
        return self.n_sim * self.dims.sites // 8

    def _io_slot(self):
        """Current of two (input, output) device staging buffers for packed
        host I/O.  Copies in and out run on two copy streams (so a load never
        queues behind an earlier store's wait for the sweeps), ordered against
        the engine's stream by events."""
        torch = _torch()
        if not hasattr(self, "_io"):
            words = self.packed_nbytes() // 8
            with torch.cuda.device(self.device):
                self._in_stream = torch.cuda.Stream(device=self.device)
                self._out_stream = torch.cuda.Stream(device=self.device)
                bufs = [(torch.empty(words, dtype=torch.int64, device=self.device),
                         torch.empty(words, dtype=torch.int64, device=self.device)) for _ in range(2)]
            self._io = [{"in": i, "out": o, "in_free": None, "out_full": None} for i, o in bufs]
            self._io_next = 0
            self._host_out = {}  # host buffer address -> event of the pending copy into it
        return self._io[self._io_next]

    def load_packed(self, src) -> None:
        """Replace every replica's lattice from bit-packed host (or device)
        memory: bit i%8 of byte i//8 of replica s is site i = c*n + r
        (np.packbits(lattice > 0, bitorder="little")).  A pinned host tensor
        is copied on the engine's input copy stream into a double-buffered
        staging area, so the copy overlaps device work already queued (the
        previous sweeps); the engine's stream waits only for this copy (and
        the copy waits for any pending ``store_packed`` into ``src``)."""
        self._push_host_edits()
        src = self._packed_src(src)
        if src.device.type == "cuda":
            call("msb_from_linear", ctypes.byref(self._g), _p(src), _p(self._spins), self._cs)
            self._touch()
            return
        slot = self._stage_in(src)
        call("msb_from_linear", ctypes.byref(self._g), _p(slot["in"]), _p(self._spins), self._cs)
        self._in_done(slot)
        self._touch()

    def _packed_src(self, src):
        torch = _torch()
        if isinstance(src, np.ndarray):
            src = torch.from_numpy(np.ascontiguousarray(src).view(np.uint8).reshape(-1))
        if src.numel() * src.element_size() != self.packed_nbytes():
            raise ValueError(f"expected {self.packed_nbytes()} bytes of packed lattices")
        return src

    def _stage_in(self, src):
        """Copy host ``src`` into the current staging slot on the input copy
        stream; the engine's stream waits for it.  Returns the slot."""
        torch = _torch()
        slot = self._io_slot()
        with torch.cuda.stream(self._in_stream):
            if slot["in_free"] is not None:          # its last reader is done
                self._in_stream.wait_event(slot["in_free"])
            pending = self._host_out.pop(src.data_ptr(), None)
            if pending is not None:                  # src is still being written by a store
                self._in_stream.wait_event(pending)
            slot["in"].view(torch.uint8).copy_(src.view(torch.uint8).reshape(-1), non_blocking=True)
            ready = torch.cuda.Event()
            ready.record(self._in_stream)
        self._stream.wait_event(ready)
        return slot

    def _in_done(self, slot) -> None:
        """The engine's stream has enqueued the last reader of slot["in"]."""
        free = _torch().cuda.Event()
        free.record(self._stream)
        slot["in_free"] = free

    def store_packed(self, dst) -> None:
        """Write every replica's lattice, bit-packed as in ``load_packed``,
        into ``dst``.  A pinned host destination is filled on the engine's
        output copy stream (asynchronous: ``synchronize()`` before reading
        it); the engine's stream continues with the next sweeps meanwhile."""
        self._export(dst, None, None)

    def observe_async(self, ups_out, unsat_out) -> None:
        """Enqueue the integer observables (ups, unsatisfied bonds per replica)
        into pinned host int64 tensors without synchronising.  The copies run
        on the output copy stream, so the engine's stream never waits behind
        a large lattice copy in the copy engine."""
        self._export(None, ups_out, unsat_out)

    def step_packed(self, src, n_sweeps: int, dst=None, ups_out=None, unsat_out=None) -> None:
        """One host-I/O step: ``load_packed(src)``, ``n_sweeps`` sweeps,
        ``store_packed(dst)`` and ``observe_async(ups_out, unsat_out)`` (dst
        and the observables optional; pinned host tensors, asynchronous:
        ``synchronize()`` before reading them).  The copies run on the
        engine's copy streams and overlap the sweeps of earlier steps.  On
        the window path the layout conversions and the observables run inside
        the window launches (``msb_window_io``): every warp converts the
        loaded lattice before the first flip, and the flip warps export the
        lattice and the observables after the last one, in their slack
        behind the producers.  Otherwise ``msb_from_linear`` and one
        ``msb_export`` kernel run beside the sweeps."""
        if (ups_out is None) != (unsat_out is None):
            raise ValueError("ups_out and unsat_out go together")
        n_sweeps = int(n_sweeps)
        if n_sweeps > 0:
            self._fit_window(n_sweeps, 0)  # windows that end where the steps end
        self._push_host_edits()
        src = self._packed_src(src)
        if dst is not None and dst.numel() * dst.element_size() != self.packed_nbytes():
            raise ValueError(f"expected {self.packed_nbytes()} bytes of packed lattices")
        if not (n_sweeps > 0 and src.device.type != "cuda" and self._window_route() and self._io_fused_ok):
            self.load_packed(src)
            self._sweeps(n_sweeps)
            self._export(dst, ups_out, unsat_out)
            return
        slot = self._stage_in(src)
        out = self._out_begin(dst, ups_out is not None)
        io = WindowIO(_p(slot["in"]).value, out[1].value, out[2].value, out[3].value)
        self._touch()
        self._sweeps(n_sweeps, io)
        self._in_done(slot)
        self._out_end(out[0], dst, ups_out, unsat_out)

    def _window_route(self) -> bool:
        """Whether ``_sweeps`` runs on lookahead windows."""
        self._sync_tables()
        return self._fast_path_ok() and self.overlap and self._params.mode != MSB_MODE_GENERIC

    @property
    def _io_fused_ok(self) -> bool:
        """Whether step_packed moves its I/O into the window launch
        (msb_window_io): chunk groups fit, and the window's producer units
        fit one round (the library's warp split then leaves the flip warps
        slack behind the producers for the export).  Multi-round shapes have
        no such slack: cfg3's fused launch measured 2092 vs 1988 us for the
        separate kernels; cfg2's 611 vs 615 us."""
        if self._direct_ok():  # every warp flips; the conversions go with them
            return self._io_groups_ok
        if not hasattr(self, "_io_fused"):
            torch = _torch()
            units = -(-int(_lib.lib().msb_window_pieces(ctypes.byref(self._g), self.window, self._wP)) // 32)
            sms = torch.cuda.get_device_properties(self.device).multi_processor_count
            self._io_fused = self._io_groups_ok and -(-units // sms) <= 30
        return self._io_fused

    def _out_begin(self, dst, want_obs):
        """Waits and pointers for an export into the current output staging
        slot (dst) and/or ``_obs``: (slot, lin, ups, unsat) pointers."""
        slot = None
        lin = ups = uns = ctypes.c_void_p(None)
        if dst is not None:
            slot = self._io_slot()
            self._io_next ^= 1
            if slot["out_full"] is not None:         # its previous copy-out is done
                self._stream.wait_event(slot["out_full"])
            lin = _p(slot["out"])
        if want_obs:
            if getattr(self, "_obs_copied", None) is not None:  # previous copy-out of _obs done
                self._stream.wait_event(self._obs_copied)
            ups, uns = _p(self._obs[: self.n_sim]), _p(self._obs[self.n_sim:])
        return slot, lin, ups, uns

    def _out_end(self, slot, dst, ups_out, unsat_out) -> None:
        """Copy the exported lattice / observables out on the output copy
        stream once the engine's stream has produced them.  The copy stream
        runs copies only: a kernel queued there waits behind the next
        cooperative window launch, and every later host-buffer wait would
        move past that window."""
        torch = _torch()
        written = torch.cuda.Event()
        written.record(self._stream)
        with torch.cuda.stream(self._out_stream):
            self._out_stream.wait_event(written)
            if ups_out is not None:  # first: the next step's kernel waits for it, not for the lattice copy
                ups_out.copy_(self._obs[: self.n_sim], non_blocking=True)
                unsat_out.copy_(self._obs[self.n_sim:], non_blocking=True)
                self._obs_copied = torch.cuda.Event()
                self._obs_copied.record(self._out_stream)
            if dst is not None:
                dst.view(torch.uint8).reshape(-1).copy_(slot["out"].view(torch.uint8), non_blocking=True)
                done = torch.cuda.Event()
                done.record(self._out_stream)
                slot["out_full"] = done
                if dst.device.type != "cuda":
                    self._host_out[dst.data_ptr()] = done

    def _export(self, dst, ups_out, unsat_out) -> None:
        """``msb_export`` of the lattice (into the current output staging
        slot, then ``dst``) and/or the observables (into ``_obs``, then
        ups_out / unsat_out): one kernel on the engine's stream, copies on
        the output copy stream."""
        torch = _torch()
        if (ups_out is None) != (unsat_out is None):
            raise ValueError("ups_out and unsat_out go together")
        if dst is None and ups_out is None:
            return
        self._push_host_edits()
        if dst is not None and dst.numel() * dst.element_size() != self.packed_nbytes():
            raise ValueError(f"expected {self.packed_nbytes()} bytes of packed lattices")
        slot, lin, ups, uns = self._out_begin(dst, ups_out is not None)
        if ups_out is not None:
            with torch.cuda.stream(self._stream):
                self._obs.zero_()
        call("msb_export", ctypes.byref(self._g), _p(self._spins), lin, ups, uns, self._cs)
        self._out_end(slot, dst, ups_out, unsat_out)

    def _observe(self):
        self._push_host_edits()
        if self._obs_ver != self._ver:
            if getattr(self, "_obs_copied", None) is not None:  # an observe_async copy-out may be pending
                self._stream.wait_event(self._obs_copied)
            with _torch().cuda.stream(self._stream):
                self._obs.zero_()
            ups = self._obs[: self.n_sim]
            uns = self._obs[self.n_sim:]
            call("msb_observe", ctypes.byref(self._g), _p(self._spins), _p(ups), _p(uns), self._cs)
            self._stream.synchronize()
            host = self._obs.cpu().numpy()
            self._obs_host = (host[: self.n_sim].copy(), host[self.n_sim:].copy())
            self._obs_ver = self._ver
        return self._obs_host

    def abs_magnetization(self) -> np.ndarray:
        """Per-replica |M| = |2 ups/N - 1| (engine.py:372-375)."""
        ups, _ = self._observe()
        return np.abs(2.0 * ups / self.dims.sites - 1.0)

    def energy_per_spin(self) -> np.ndarray:
        """Per-replica bond energy per spin (engine.py:377-386): bonds =
        sum s_i s_j = 2N - 2 * (unsatisfied bonds), evaluated as
        -J * bonds / N in float64 exactly as the reference."""
        _, unsat = self._observe()
        bonds = 2 * self.dims.sites - 2 * unsat
        return -self.coupling * bonds / self.dims.sites

    def halo_mismatches(self) -> int:
        """Halo/moat words of ``state`` differing from their canonical source."""
        st = self.state
        (la, lg, lw), (sa, sg, sw), (da, dg, dw) = halo_audit_index(self.dims)
        bad = int((st[:, la, lg, lw] != st[:, sa, sg, sw]).sum())
        bad += int((st[:, da, dg, dw] != 0).sum())
        return bad

    # -- driving (engine.py:401-440) -------------------------------------------

    def run(self, n_sweeps: int, measure_interval: int = 100) -> Trajectory:
        if n_sweeps < 0:
            raise ValueError("sweep count must be non-negative")
        if measure_interval < 1:
            raise ValueError("measurement interval must be positive")
        sweeps_at, abs_m, energy = [], [], []
        start_attempts = self.attempts
        t0 = time.perf_counter()
        points = []
        k = 0
        while k < n_sweeps:
            k = min((k // measure_interval + 1) * measure_interval, n_sweeps)
            points.append(k)
        self._fit_window(measure_interval, n_sweeps)
        cls = type(self)
        if points and cls.abs_magnetization is Engine.abs_magnetization and \
                cls.energy_per_spin is Engine.energy_per_spin:
            # Measurements stay on the device: each one is an msb_observe into
            # its own row of a device buffer, enqueued behind its sweeps, and
            # the host reads them all once at the end.  The sweeps never wait
            # for the host (a synchronising measurement every 8 sweeps cost
            # cfg2 11%, every sweep 57%).  The float64 expressions are those of
            # abs_magnetization / energy_per_spin (engine.py:372-386).
            torch = _torch()
            with torch.cuda.device(self.device), torch.cuda.stream(self._stream):
                obs = torch.zeros((len(points), 2, self.n_sim), dtype=torch.int64, device=self.device)
            k = 0
            for i, nxt in enumerate(points):
                self._sweeps(nxt - k)
                k = nxt
                sweeps_at.append(self.sweeps_done)
                self._push_host_edits()
                call("msb_observe", ctypes.byref(self._g), _p(self._spins), _p(obs[i, 0]), _p(obs[i, 1]), self._cs)
            self._stream.synchronize()
            host = obs.cpu().numpy()
            ups, unsat = host[:, 0, :], host[:, 1, :]
            abs_m = np.abs(2.0 * ups / self.dims.sites - 1.0)
            energy = -self.coupling * (2 * self.dims.sites - 2 * unsat) / self.dims.sites
        else:  # overridden observables (reference test wrappers): called per measurement, as the reference
            k = 0
            for nxt in points:
                self._sweeps(nxt - k)
                k = nxt
                sweeps_at.append(self.sweeps_done)
                abs_m.append(self.abs_magnetization())
                energy.append(self.energy_per_spin())
            self._stream.synchronize()
        elapsed = time.perf_counter() - t0
        return Trajectory(
            sweeps=np.array(sweeps_at, dtype=np.int64),
            abs_m=np.array(abs_m, dtype=np.float64).reshape(len(sweeps_at), self.n_sim),
            energy=np.array(energy, dtype=np.float64).reshape(len(sweeps_at), self.n_sim),
            temperatures=self.temperatures,
            meta={
                "m": self.dims.m, "n": self.dims.n, "seed": self.seed, "coupling": self.coupling,
                "init": self.init, "sim_offset": self.sim_offset, "measure_interval": measure_interval,
                "sweeps_run": n_sweeps, "attempts": self.attempts - start_attempts, "elapsed_s": elapsed,
                "device": str(self.device),
            },
        )


def run_simulations(dims: LatticeDims, temperatures, seed: int, n_sweeps: int, measure_interval: int = 100,
                    init: str = "random", coupling: float = 1.0, threads: int = 1, devices=None) -> Trajectory:
    """Replica fan-out with global stream indexing (engine.py:443-492).

    Replicas split into contiguous slices exactly as the reference does
    (np.linspace bounds, sim_offset = slice start), so any split is
    bit-identical to one engine.  Slices are assigned round-robin to
    ``devices`` (default: every visible GPU) and driven from host threads.
    """
    torch = _torch()
    temperatures = tuple(float(t) for t in temperatures)
    threads = max(1, int(threads))
    if devices is None:
        devices = list(range(torch.cuda.device_count())) if torch.cuda.is_available() else [None]
    devices = list(devices) or [None]
    t0 = time.perf_counter()
    if threads == 1 or len(temperatures) == 1:
        traj = Engine(dims, temperatures, seed, init=init, coupling=coupling, device=devices[0]).run(
            n_sweeps, measure_interval)
        traj.meta["elapsed_s"] = time.perf_counter() - t0
        traj.meta["threads"] = 1
        return traj
    threads = min(threads, len(temperatures))
    bounds = np.linspace(0, len(temperatures), threads + 1).astype(int)
    slices = [(int(a), int(b)) for a, b in zip(bounds[:-1], bounds[1:]) if b > a]

    def run_slice(i_ab):
        i, (lo, hi) = i_ab
        dev = devices[i % len(devices)]
        eng = Engine(dims, temperatures[lo:hi], seed, init=init, coupling=coupling, sim_offset=lo, device=dev)
        return eng.run(n_sweeps, measure_interval)

    with ThreadPoolExecutor(max_workers=len(slices)) as pool:
        parts = list(pool.map(run_slice, enumerate(slices)))
    merged = Trajectory(
        sweeps=parts[0].sweeps,
        abs_m=np.concatenate([p.abs_m for p in parts], axis=1),
        energy=np.concatenate([p.energy for p in parts], axis=1),
        temperatures=temperatures,
        meta=dict(parts[0].meta),
    )
    merged.meta["sim_offset"] = 0
    merged.meta["attempts"] = sum(p.meta["attempts"] for p in parts)
    merged.meta["elapsed_s"] = time.perf_counter() - t0
    merged.meta["threads"] = len(slices)
    merged.meta["devices"] = sorted({p.meta["device"] for p in parts})
    return merged
