"""Row-slab decomposition of one large lattice over several devices.

The reference runs one lattice in one process (its cell strip is emulated
in lockstep, engine.py:1-15).  Here a lattice of m rows (the reference's
cell axis c) is split into G contiguous slabs of m/G rows, one per GPU.  A
colour phase reads the other colour of rows c-1 and c+1, so each slab keeps
one ghost row per colour above and below its rows, refreshed by a one-row
exchange with the neighbouring slabs before every phase (periodic: slab 0's
upper neighbour is slab G-1).  Messages are n/16 bytes per colour row.

The random streams need no exchange: each slab generates exactly the stream
pieces that gate its own rows (jump-ahead to their offsets), so results are
bit-identical to the single-GPU Engine and to the reference for any G.

Transports:
  LocalExchange  all slabs in this process (one or several local GPUs):
                 plain device-to-device copies between the phase kernels;
  DistExchange   one slab per torch.distributed rank: batched send/recv of
                 the edge rows (NCCL over NVLink on GPUs, gloo on CPU).

FusedSlabRun drops the host from the loop: one slab per process, lookahead
windows (msb_window_sweep) whose flip warps store the slab's first/last rows
straight into the neighbours' ghost rows -- peer memory over NVLink from
symmetric memory -- and handshake every phase through flag counters in peer
memory.  One process with one slab is the periodic ring of a single slab
(its own neighbour), which runs the same kernel path.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import call, geom, SweepParams, MSB_FLIP_SLOTS, MSB_MAX_PLANES, MSB_RNG_PHILOX, MSB_RNG_XOSHIRO, RNG_MODES
from .engine import _M64, _jump_table, _p, _pow_tables, _sweep_jump_table, _torch, build_exp_table
from .layout import LatticeDims

__all__ = ["slab_bounds", "ring_plan", "SlabLattice", "LocalExchange", "DistExchange", "SlabRun", "FusedSlabRun",
           "symmetric_alloc"]


def slab_bounds(m: int, parts: int) -> list[tuple[int, int]]:
    """Contiguous even-aligned row ranges covering [0, m)."""
    if m % 2 or parts < 1:
        raise ValueError("need an even row count and at least one slab")
    pairs = m // 2
    if parts > pairs:
        raise ValueError(f"cannot split {m} rows into {parts} even slabs")
    cuts = [2 * (pairs * k // parts) for k in range(parts + 1)]
    return [(cuts[k], cuts[k + 1]) for k in range(parts)]


class SlabLattice:
    """Rows [row0, row0+rows) of n_sim replicas of an m x n lattice on one
    device, with ghost rows, RNG pieces for the owned rows and the
    accept-plane buffer."""

    def __init__(self, dims: LatticeDims, temperatures, seed: int, row0: int, rows: int, init: str = "random",
                 coupling: float = 1.0, sim_offset: int = 0, device=None, kg: int | None = None,
                 stream: str = "xoshiro", alloc=None):
        torch = _torch()
        self.dims = dims
        self.temperatures = tuple(float(t) for t in temperatures)
        self.n_sim = len(self.temperatures)
        self.seed = int(seed)
        self.coupling = float(coupling)
        self.row0, self.rows = int(row0), int(rows)
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self._stream = torch.cuda.Stream(device=self.device)
        self._cs = ctypes.c_void_p(self._stream.cuda_stream)
        self._g = geom(self.n_sim, dims.m, dims.n, row0=self.row0, rows=self.rows, ghost=1, sim_offset=sim_offset)
        call("msb_check_geom", ctypes.byref(self._g))
        L = _lib.lib()
        self.kg = int(kg) if kg is not None else int(L.msb_default_kg(ctypes.byref(self._g)))
        self.Wp = int(L.msb_row_pitch(ctypes.byref(self._g)))
        n_pieces = int(L.msb_pieces_per_phase(ctypes.byref(self._g), self.kg))
        tables = np.stack([build_exp_table(t, coupling) for t in self.temperatures])
        mode, npl = ctypes.c_int32(), ctypes.c_int32()
        codes = (ctypes.c_int8 * 16)()
        thr = np.zeros(MSB_MAX_PLANES * self.n_sim, np.uint32)
        call("msb_plan_thresholds", tables.ctypes.data_as(ctypes.c_void_p), self.n_sim, ctypes.byref(mode),
             ctypes.byref(npl), codes, thr.ctypes.data_as(ctypes.c_void_p))
        with torch.cuda.device(self.device), torch.cuda.stream(self._stream):
            nwords = int(L.msb_spin_words(ctypes.byref(self._g)))
            # alloc: e.g. symmetric_alloc(group) so peers can map the buffer (FusedSlabRun)
            self._spins = (alloc(nwords, self.device) if alloc is not None
                           else torch.empty(nwords, dtype=torch.int32, device=self.device))
            self._states = torch.empty(2 * 8 * n_pieces, dtype=torch.int32, device=self.device)
            self._planes = torch.empty(int(L.msb_plane_words(ctypes.byref(self._g), npl.value)),
                                       dtype=torch.int32, device=self.device)
            self._thr = torch.from_numpy(thr.view(np.int32)).to(self.device)
            self._work = torch.zeros(4, dtype=torch.int32, device=self.device)
            self._flips = torch.zeros(MSB_FLIP_SLOTS, dtype=torch.int64, device=self.device)
            self._obs = torch.zeros(2 * self.n_sim, dtype=torch.int64, device=self.device)
            self._edge = torch.empty(self.n_sim * 2 * self.Wp, dtype=torch.int32, device=self.device)
            self._ghost = torch.empty(self.n_sim * 2 * self.Wp, dtype=torch.int32, device=self.device)
        self._pow = _pow_tables(self.device)
        self._jump = _sweep_jump_table(self.device, dims.n)
        p = SweepParams()
        p.mode, p.n_planes = mode.value, npl.value
        p.code_plane[:] = list(codes)
        p.thr9, p.kg, p.jump, p.work = self._thr.data_ptr(), self.kg, self._jump.data_ptr(), self._work.data_ptr()
        if stream not in RNG_MODES:
            raise ValueError(f"unknown stream {stream!r}")
        self.stream = stream
        p.rng = RNG_MODES[stream]
        p.seed = self.seed & _M64
        self._params = p
        if init == "random":
            with torch.cuda.stream(self._stream):
                scratch = torch.empty(self.n_sim * self.rows * dims.n // 64, dtype=torch.int64, device=self.device)
            call("msb_init_random", ctypes.byref(self._g), ctypes.c_uint64(self.seed & _M64), _p(self._pow),
                 _p(scratch), _p(self._spins), self._cs)
            scratch.record_stream(self._stream)
        elif init == "all-up":
            call("msb_init_const", ctypes.byref(self._g), 1, _p(self._spins), self._cs)
        else:
            raise ValueError(f"unknown init mode {init!r}")
        if stream == "xoshiro":
            call("msb_rng_init", ctypes.byref(self._g), ctypes.c_uint64(self.seed & _M64), self.kg,
                 ctypes.c_uint64(0), -1, _p(self._pow), _p(self._states), self._cs)
        self.sweeps_done = 0

    # -- halo plumbing ---------------------------------------------------------

    def edges(self, colour: int):
        """[n_sim][2][Wp] int32: colour's first and last owned rows."""
        call("msb_pack_edges", ctypes.byref(self._g), colour, _p(self._spins), _p(self._edge), self._cs)
        return self._edge

    def set_ghosts(self, colour: int, ghosts) -> None:
        """ghosts: [n_sim][2][Wp] = (row above, row below) of colour."""
        call("msb_unpack_ghosts", ctypes.byref(self._g), colour, _p(ghosts), _p(self._spins), self._cs)

    # -- compute ---------------------------------------------------------------

    def rng_planes(self) -> None:
        self._params.block = 2 * self.sweeps_done
        call("msb_rng_planes", ctypes.byref(self._g), ctypes.byref(self._params), -1, _p(self._states), None,
             _p(self._planes), self._cs)

    def flip(self, colour: int) -> None:
        call("msb_flip", ctypes.byref(self._g), ctypes.byref(self._params), colour, _p(self._spins),
             _p(self._planes), _p(self._flips), self._cs)

    def observe(self):
        """Device int64 [2*n_sim]: ups and unsatisfied bonds of the owned rows
        (blue ghosts must be current)."""
        with _torch().cuda.stream(self._stream):
            self._obs.zero_()
        call("msb_observe", ctypes.byref(self._g), _p(self._spins), _p(self._obs[: self.n_sim]),
             _p(self._obs[self.n_sim:]), self._cs)
        return self._obs

    def lattice_rows(self) -> np.ndarray:
        """int8 (n_sim, rows, n) +/-1 spins of the owned rows."""
        torch = _torch()
        n = self.dims.n
        with torch.cuda.stream(self._stream):
            lin = torch.empty(self.n_sim * self.rows * n // 64, dtype=torch.int64, device=self.device)
        call("msb_to_linear", ctypes.byref(self._g), _p(self._spins), _p(lin), self._cs)
        self._stream.synchronize()
        bits = np.unpackbits(lin.cpu().numpy().view(np.uint8), bitorder="little")
        return np.where(bits == 1, 1, -1).astype(np.int8).reshape(self.n_sim, self.rows, n)

    def stream_ctx(self):
        return _torch().cuda.stream(self._stream)

    @property
    def flips(self) -> int:
        self._stream.synchronize()
        return int(self._flips.sum().item())

    def synchronize(self) -> None:
        self._stream.synchronize()


def ring_plan(m: int, world: int, rank: int) -> dict:
    """Slab rows of `rank` in a ring of `world` slabs over m rows, and its
    neighbours: the slab above (rank-1, whose last row is our upper ghost)
    and below (rank+1), with their buffer rows per colour (rows + 2)."""
    bounds = slab_bounds(m, world)
    up, down = (rank - 1) % world, (rank + 1) % world
    (a, b) = bounds[rank]
    return {"row0": a, "rows": b - a, "up": up, "down": down,
            "up_R": bounds[up][1] - bounds[up][0] + 2, "down_R": bounds[down][1] - bounds[down][0] + 2}


def symmetric_alloc(group=None):
    """Allocator for SlabLattice(alloc=...): int32 buffers in torch symmetric
    memory, so every rank of `group` can map them (FusedSlabRun)."""
    import torch.distributed._symmetric_memory as symm_mem
    torch = _torch()

    def alloc(nwords: int, device):
        return symm_mem.empty(nwords, dtype=torch.int32, device=device)
    return alloc


def _neighbour_ghosts(edges_above, edges_below, n_sim: int, Wp: int):
    """Ghost buffer [n_sim][2][Wp] from the slab above's edges (its LAST row
    becomes our upper ghost) and the slab below's edges (its FIRST row)."""
    torch = _torch()
    a = edges_above.view(n_sim, 2, Wp)
    b = edges_below.view(n_sim, 2, Wp)
    return torch.stack([a[:, 1], b[:, 0]], dim=1).reshape(-1)


class LocalExchange:
    """All slabs live in this process (same or different local GPUs): the
    edge rows move by device copies between the phase kernels."""

    def exchange(self, slabs, colour: int) -> None:
        G = len(slabs)
        edges = []
        for s in slabs:
            with s.stream_ctx():
                edges.append(s.edges(colour).clone())
            s.synchronize()
        for k, s in enumerate(slabs):
            above, below = edges[(k - 1) % G], edges[(k + 1) % G]
            with s.stream_ctx():
                g = _neighbour_ghosts(above.to(s.device), below.to(s.device), s.n_sim, s.Wp)
                s.set_ghosts(colour, g.contiguous())
            s.synchronize()


class DistExchange:
    """One slab per torch.distributed rank; the ring neighbours exchange
    their edge rows with batched point-to-point send/recv (NCCL over NVLink
    on GPUs, gloo on CPU).  Works with any slab object exposing
    edges/set_ghosts/stream_ctx/synchronize/n_sim/Wp."""

    def __init__(self, group=None):
        self.group = group

    def exchange(self, slabs, colour: int) -> None:
        import torch.distributed as dist
        torch = _torch()
        (s,) = slabs
        rank, world = dist.get_rank(self.group), dist.get_world_size(self.group)
        up, down = (rank - 1) % world, (rank + 1) % world
        with s.stream_ctx():
            e = s.edges(colour).view(s.n_sim, 2, s.Wp)
            first, last = e[:, 0].contiguous(), e[:, 1].contiguous()
            from_up, from_down = torch.empty_like(last), torch.empty_like(first)
            if world == 1:
                from_up.copy_(last)
                from_down.copy_(first)
            else:
                ops = [dist.P2POp(dist.isend, last, down, self.group),
                       dist.P2POp(dist.isend, first, up, self.group),
                       dist.P2POp(dist.irecv, from_up, up, self.group),
                       dist.P2POp(dist.irecv, from_down, down, self.group)]
                for req in dist.batch_isend_irecv(ops):
                    req.wait()
            s.set_ghosts(colour, torch.stack([from_up, from_down], dim=1).reshape(-1).contiguous())
        s.synchronize()


@dataclass
class SlabRun:
    """Drives a list of slabs (the whole lattice in LocalExchange mode, this
    rank's slab in DistExchange mode) through sweeps."""

    slabs: list
    exchange: object

    def sweep(self, n_sweeps: int = 1) -> None:
        for _ in range(n_sweeps):
            for s in self.slabs:
                s.rng_planes()           # state independent: before any exchange
            for X in (0, 1):
                self.exchange.exchange(self.slabs, 1 - X)
                for s in self.slabs:
                    s.flip(X)
            for s in self.slabs:
                s.sweeps_done += 1

    def observables(self):
        """(ups, unsat) int64 per replica, summed over this process's slabs;
        DistExchange callers all-reduce them."""
        self.exchange.exchange(self.slabs, 1)
        ups = unsat = None
        for s in self.slabs:
            o = s.observe()
            s.synchronize()
            h = o.cpu().numpy()
            u, b = h[: s.n_sim].copy(), h[s.n_sim:].copy()
            ups = u if ups is None else ups + u
            unsat = b if unsat is None else unsat + b
        return ups, unsat


class FusedSlabRun:
    """One slab per process, halos exchanged inside the window kernel.

    Per call of ``sweep(k)`` the slab runs lookahead windows of S sweeps
    (``msb_window_sweep`` with an ``msb_halo``): producer warps generate the
    next window's accept planes for the slab's own rows while the flip warps
    flip the current window phase by phase; every flip of the first / last
    owned row is also stored into the neighbour's ghost row (peer memory), and
    the slabs handshake each phase through monotonic flag counters (system-
    scope atomics on peer memory), so no host synchronisation or separate
    exchange step remains.

    world 1 (no process group): the slab is its own upper and lower
    neighbour -- the periodic single-slab ring, same kernel path.  world > 1:
    build the slab with ``alloc=symmetric_alloc(group)`` and rows from
    ``ring_plan``; spins and flags are mapped from every peer.
    """

    def __init__(self, slab: SlabLattice, group=None, window: int | None = None):
        import torch.distributed as dist
        torch = _torch()
        self.slab = slab
        L = _lib.lib()
        g = ctypes.byref(slab._g)
        if slab._params.mode == 2:
            raise ValueError("fused slab windows need FERRO/ANTI tables")
        if window is None:
            S, P = ctypes.c_int32(), ctypes.c_int32()
            call("msb_default_window", g, ctypes.byref(S), ctypes.byref(P))
            self.S, self.P = int(S.value), int(P.value)
        else:
            self.S = int(window)
            self.P = int(L.msb_window_parts(g, self.S))
        # bit-plane stream: direct sweeps (no accept planes), S sweeps per launch
        self.direct = slab.stream == "philox-bits" and bool(L.msb_direct_ok(g, ctypes.byref(slab._params)))
        self.world = dist.get_world_size(group) if (dist.is_available() and dist.is_initialized()) else 1
        self.rank = dist.get_rank(group) if self.world > 1 else 0
        if not self.direct:
            npieces = int(L.msb_window_pieces(g, self.S, self.P))
            self._words = int(L.msb_window_words(g, self.S))
            if npieces < 0 or self._words < 0:
                raise _lib.MsbError(f"slab window S={self.S} P={self.P}: {L.msb_last_error().decode()}")
            with torch.cuda.device(slab.device), slab.stream_ctx():
                self._wstates = torch.empty(8 * npieces, dtype=torch.int32, device=slab.device)
                self._wplanes = torch.empty(2 * self._words, dtype=torch.int32, device=slab.device)
            self._jump = _jump_table(slab.device, self.S * 4 * slab.dims.n)
        R = slab.rows + 2
        h = _lib.Halo()
        if self.world == 1:
            with slab.stream_ctx():
                self._flags = torch.zeros(2, dtype=torch.int32, device=slab.device)
            sp, fl = slab._spins.data_ptr(), self._flags.data_ptr()
            h.up_spins = h.down_spins = sp
            h.up_flags = h.down_flags = h.my_flags = fl
            h.up_R = h.down_R = R
            LocalExchange().exchange([slab], 0)
            LocalExchange().exchange([slab], 1)
        else:
            import torch.distributed._symmetric_memory as symm_mem
            plan = ring_plan(slab.dims.m, self.world, self.rank)
            if (plan["row0"], plan["rows"]) != (slab.row0, slab.rows):
                raise ValueError("slab rows must follow ring_plan(m, world, rank)")
            self._flags = symm_mem.empty(2, dtype=torch.int32, device=slab.device)
            self._flags.zero_()
            hs = symm_mem.rendezvous(slab._spins, group)
            hf = symm_mem.rendezvous(self._flags, group)

            def peer(hdl, t, r):  # peer r's mapping of the same buffer
                return int(hdl.buffer_ptrs[r]) + (t.data_ptr() - int(hdl.buffer_ptrs[self.rank]))
            h.up_spins, h.down_spins = peer(hs, slab._spins, plan["up"]), peer(hs, slab._spins, plan["down"])
            h.up_flags, h.down_flags = peer(hf, self._flags, plan["up"]), peer(hf, self._flags, plan["down"])
            h.my_flags = self._flags.data_ptr()
            h.up_R, h.down_R = plan["up_R"], plan["down_R"]
            DistExchange(group).exchange([slab], 0)
            DistExchange(group).exchange([slab], 1)
            torch.cuda.synchronize(slab.device)
            dist.barrier(group)
        h.phase0 = 0
        self._halo = h
        self._valid = False
        self._cur = 0
        self._wc = 0
        self._wbase = 0

    def _launch(self, first: int, count: int, produce: bool) -> None:
        s = self.slab
        w = self._words
        cur = self._wplanes[self._cur * w:(self._cur + 1) * w]
        nxt = self._wplanes[(1 - self._cur) * w:(2 - self._cur) * w]
        if count == 0:
            nxt, cur = cur, None
        s._params.jump = self._jump.data_ptr()
        s._params.block = self._wbase if count == 0 else self._wbase + 2 * self.S
        call("msb_window_sweep", ctypes.byref(s._g), ctypes.byref(s._params), self.S, self.P, _p(s._spins),
             _p(self._wstates), _p(cur) if cur is not None else None, first, count,
             _p(nxt) if produce else None, _p(s._flips), ctypes.byref(self._halo), None, s._cs)
        s._params.jump = s._jump.data_ptr()

    def sweep(self, n_sweeps: int = 1) -> None:
        s = self.slab
        k = int(n_sweeps)
        if k <= 0:
            return
        if self.direct:
            while k > 0:
                r = min(k, self.S)
                s._params.block = 2 * s.sweeps_done
                call("msb_direct_sweep", ctypes.byref(s._g), ctypes.byref(s._params), _p(s._spins), r, _p(s._flips),
                     None, ctypes.c_uint32(0), ctypes.byref(self._halo), None, s._cs)
                self._halo.phase0 += 2 * r
                s.sweeps_done += r
                k -= r
            return
        if not self._valid:
            self._wbase, self._wc, self._cur = 2 * s.sweeps_done, 0, 0
            if s.stream == "xoshiro":
                call("msb_window_init", ctypes.byref(s._g), ctypes.c_uint64(s.seed & _M64), self.S, self.P,
                     ctypes.c_uint64(self._wbase), _p(s._pow), _p(self._wstates), s._cs)
            self._launch(0, 0, True)
            self._valid = True
        while k > 0:
            r = min(k, self.S - self._wc)
            finish = self._wc + r == self.S
            self._launch(self._wc, r, finish)
            self._halo.phase0 += 2 * r
            s.sweeps_done += r
            k -= r
            if finish:
                self._cur, self._wc, self._wbase = 1 - self._cur, 0, self._wbase + 2 * self.S
            else:
                self._wc += r

    def observe_async(self):
        """Device int64 [2*n_sim] (ups, unsat) of this slab, stream-ordered: a
        device-side wait until both neighbours finished the phases so far (our
        ghost rows are current), then msb_observe.  No host synchronisation;
        callers with world > 1 all-reduce the result."""
        s = self.slab
        call("msb_window_sweep", ctypes.byref(s._g), ctypes.byref(s._params), self.S, self.P, None, None, None,
             0, 0, None, None, ctypes.byref(self._halo), None, s._cs)
        return s.observe()

    def observables(self):
        """(ups, unsat) int64 per replica of this slab (host copies)."""
        o = self.observe_async()
        self.slab.synchronize()
        h = o.cpu().numpy()
        n = self.slab.n_sim
        return h[:n].copy(), h[n:].copy()
