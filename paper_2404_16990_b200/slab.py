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

FusedSlabRun drops the host from the loop: lookahead windows
(msb_window_sweep) whose flip warps store each slab's first/last rows
straight into the neighbours' ghost rows -- peer memory over NVLink from
symmetric memory with one slab per process, or plain device memory for the
slabs of one process -- and order the phases per band group through flags
the slabs write into each other's memory, so only the edge bands ever wait
on a neighbour.  Several slabs of one process run in one cooperative launch
(msb_window_sweep_ring); one slab alone is the periodic ring of a single
slab (its own neighbour), on the same kernel path.
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
           "symmetric_alloc", "resolve_group", "peer_halo"]


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
            # phase flags (header, halo slots from the neighbour slabs, band groups):
            # written by the neighbours too, so in the same memory kind as the spins
            nflags = int(L.msb_flag_words(ctypes.byref(self._g)))
            self._flags = (alloc(nflags, self.device) if alloc is not None
                           else torch.empty(nflags, dtype=torch.int32, device=self.device))
            self._flags.zero_()
            self._edge = torch.empty(self.n_sim * 2 * self.Wp, dtype=torch.int32, device=self.device)
            self._ghost = torch.empty(self.n_sim * 2 * self.Wp, dtype=torch.int32, device=self.device)
        self._pow = _pow_tables(self.device)
        self._jump = _sweep_jump_table(self.device, dims.n)
        p = SweepParams()
        p.mode, p.n_planes = mode.value, npl.value
        p.code_plane[:] = list(codes)
        p.thr9, p.kg, p.jump, p.work = self._thr.data_ptr(), self.kg, self._jump.data_ptr(), self._work.data_ptr()
        p.flags = self._flags.data_ptr()
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


def resolve_group(group=None):
    """(group, world, rank) of a ring spanning processes: ``group`` or, when
    torch.distributed is initialised, the default group (symmetric memory
    needs a real group object: ``rendezvous(t, None)`` raises); world 1 and
    rank 0 without torch.distributed."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return None, 1, 0
    if group is None:
        group = dist.group.WORLD
    world = dist.get_world_size(group)
    return group, world, (dist.get_rank(group) if world > 1 else 0)


def peer_halo(plan: dict, rank: int, spins_handle, flags_handle, spins_ptr: int, flags_ptr: int):
    """msb_halo of ring member `rank` from the symmetric-memory handles of
    its spin and flag buffers: the neighbours' mappings of the same buffers
    (buffer_ptrs[r] is rank r's allocation as mapped here; our buffers may
    be views at an offset into the allocation)."""
    def peer(hdl, ptr, r):
        return int(hdl.buffer_ptrs[r]) + (ptr - int(hdl.buffer_ptrs[rank]))
    h = _lib.Halo()
    h.up_spins, h.down_spins = peer(spins_handle, spins_ptr, plan["up"]), peer(spins_handle, spins_ptr, plan["down"])
    h.up_flags, h.down_flags = peer(flags_handle, flags_ptr, plan["up"]), peer(flags_handle, flags_ptr, plan["down"])
    h.up_R, h.down_R = plan["up_R"], plan["down_R"]
    return h


def symmetric_alloc(group=None):
    """Allocator for SlabLattice(alloc=...): int32 buffers in torch symmetric
    memory, so every rank of `group` can map them (FusedSlabRun).  Symmetric
    buffers must have one size on every rank, and slabs of an uneven split
    differ by a row or two: each allocation is the group's largest request
    (one MAX all-reduce per buffer; every rank allocates the same buffers in
    the same order), returned as a view of the requested length."""
    import torch.distributed as dist
    import torch.distributed._symmetric_memory as symm_mem
    torch = _torch()

    def alloc(nwords: int, device):
        top = int(nwords)
        if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
            t = torch.tensor([top], dtype=torch.int64, device=device)
            dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
            top = int(t.item())
        return symm_mem.empty(top, dtype=torch.int32, device=device)[:nwords]
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
    """Slabs whose halos are exchanged inside the flip kernels.

    Per call of ``sweep(k)`` every slab runs lookahead windows of S sweeps
    (``msb_window_sweep`` with an ``msb_halo``; the bit-plane stream: direct
    sweeps): producer warps generate the next window's accept planes for the
    slab's own rows while the flip warps flip the current window; every flip
    of a slab's first / last row is also stored into the neighbour's ghost
    row, and phases are ordered per band group -- interior bands wait only
    for their neighbours on the same GPU, the edge bands also for the
    neighbour slab's edge band (flags written into each other's memory) --
    so no host synchronisation or separate exchange step remains and the
    halo traffic overlaps the interior flips.

    ``slabs``: one SlabLattice, or a list of them forming the whole ring on
    this process's device (consecutive ring_plan / slab_bounds slabs of one
    lattice).  With one process, the slabs are each other's neighbours (a
    single slab is its own: the periodic ring of one slab); several slabs run
    in ONE cooperative launch per window (msb_window_sweep_ring), the CTAs
    split between them.  With a process group of world > 1: exactly one slab
    per rank, built with ``alloc=symmetric_alloc(group)`` and rows from
    ``ring_plan``; spins and flags of the ring neighbours are mapped from
    symmetric memory (NVLink peer memory).
    """

    def __init__(self, slabs, group=None, window: int | None = None):
        import torch.distributed as dist
        torch = _torch()
        self.slabs = list(slabs) if isinstance(slabs, (list, tuple)) else [slabs]
        s0 = self.slab = self.slabs[0]
        L = _lib.lib()
        g = ctypes.byref(s0._g)
        for s in self.slabs:
            if s._params.mode == 2:
                raise ValueError("fused slab windows need FERRO/ANTI tables")
            if s.stream != s0.stream or s.device != s0.device or s.dims != s0.dims or s.n_sim != s0.n_sim:
                raise ValueError("the slabs of a ring share the lattice, stream kind and device")
        if window is None:
            S, P = ctypes.c_int32(), ctypes.c_int32()
            call("msb_default_window", g, ctypes.byref(S), ctypes.byref(P))
            self.S, self.P = int(S.value), int(P.value)
        else:
            self.S = int(window)
            self.P = int(L.msb_window_parts(g, self.S))
        # bit-plane stream: direct sweeps (no accept planes), S sweeps per launch
        self.direct = s0.stream == "philox-bits" and all(
            bool(L.msb_direct_ok(ctypes.byref(s._g), ctypes.byref(s._params))) for s in self.slabs)
        self.group, self.world, self.rank = resolve_group(group)
        if self.world > 1 and len(self.slabs) != 1:
            raise ValueError("one slab per rank when the ring spans processes")
        self._wb = []
        if not self.direct:
            for s in self.slabs:
                sg = ctypes.byref(s._g)
                npieces = int(L.msb_window_pieces(sg, self.S, self.P))
                words = int(L.msb_window_words(sg, self.S))
                if npieces < 0 or words < 0:
                    raise _lib.MsbError(f"slab window S={self.S} P={self.P}: {L.msb_last_error().decode()}")
                with torch.cuda.device(s.device), s.stream_ctx():
                    self._wb.append((torch.empty(8 * npieces, dtype=torch.int32, device=s.device),
                                     torch.empty(2 * words, dtype=torch.int32, device=s.device), words))
            self._jump = _jump_table(s0.device, self.S * 4 * s0.dims.n)
        self._halos = []
        if self.world == 1:
            V = len(self.slabs)
            for v, s in enumerate(self.slabs):
                up, dn = self.slabs[(v - 1) % V], self.slabs[(v + 1) % V]
                if (up.row0 + up.rows) % s.dims.m != s.row0 or (s.row0 + s.rows) % s.dims.m != dn.row0:
                    raise ValueError("the slabs must be consecutive row ranges covering the lattice")
                h = _lib.Halo()
                h.up_spins, h.down_spins = up._spins.data_ptr(), dn._spins.data_ptr()
                h.up_flags, h.down_flags = up._flags.data_ptr(), dn._flags.data_ptr()
                h.up_R, h.down_R = up.rows + 2, dn.rows + 2
                self._halos.append(h)
            for X in (0, 1):
                LocalExchange().exchange(self.slabs, X)
        else:
            import torch.distributed._symmetric_memory as symm_mem
            plan = ring_plan(s0.dims.m, self.world, self.rank)
            if (plan["row0"], plan["rows"]) != (s0.row0, s0.rows):
                raise ValueError("slab rows must follow ring_plan(m, world, rank)")

            def base(t):
                return t._base if t._base is not None else t
            hs = symm_mem.rendezvous(base(s0._spins), self.group)
            hf = symm_mem.rendezvous(base(s0._flags), self.group)
            self._halos.append(peer_halo(plan, self.rank, hs, hf, s0._spins.data_ptr(), s0._flags.data_ptr()))
            self._handles = (hs, hf)
            DistExchange(self.group).exchange([s0], 0)
            DistExchange(self.group).exchange([s0], 1)
            torch.cuda.synchronize(s0.device)
            dist.barrier(self.group)
        if len(self.slabs) > 1:
            with torch.cuda.device(s0.device), s0.stream_ctx():
                self._ctx = torch.empty(int(L.msb_ring_ctx_bytes(len(self.slabs))), dtype=torch.uint8,
                                        device=s0.device)
            # one launch runs every slab: the slabs share the first slab's stream
            # from here on (their construction work, on their own streams, first)
            for s in self.slabs[1:]:
                s.synchronize()
                s._stream, s._cs = s0._stream, s0._cs
        self._valid = False
        self._cur = 0
        self._wc = 0
        self._wbase = 0

    def _ring(self, first: int, count: int, produce: bool):
        arr = (_lib.RingSlab * len(self.slabs))()
        for v, s in enumerate(self.slabs):
            r = arr[v]
            r.g, r.p = ctypes.pointer(s._g), ctypes.pointer(s._params)
            r.spins, r.flips, r.halo = s._spins.data_ptr(), s._flips.data_ptr(), ctypes.pointer(self._halos[v])
            if not self.direct:
                states, planes, w = self._wb[v]
                cur = planes[self._cur * w:(self._cur + 1) * w]
                nxt = planes[(1 - self._cur) * w:(2 - self._cur) * w]
                if count == 0:
                    nxt, cur = cur, None
                r.states = states.data_ptr()
                r.cur = cur.data_ptr() if cur is not None else None
                r.next = nxt.data_ptr() if produce else None
        return arr

    def _launch(self, first: int, count: int, produce: bool) -> None:
        s0 = self.slab
        for s in self.slabs:
            s._params.jump = self._jump.data_ptr()
            s._params.block = self._wbase if count == 0 else self._wbase + 2 * self.S
        if len(self.slabs) == 1:
            states, planes, w = self._wb[0]
            cur = planes[self._cur * w:(self._cur + 1) * w]
            nxt = planes[(1 - self._cur) * w:(2 - self._cur) * w]
            if count == 0:
                nxt, cur = cur, None
            call("msb_window_sweep", ctypes.byref(s0._g), ctypes.byref(s0._params), self.S, self.P, _p(s0._spins),
                 _p(states), _p(cur) if cur is not None else None, first, count, _p(nxt) if produce else None,
                 _p(s0._flips), ctypes.byref(self._halos[0]), None, s0._cs)
        else:
            arr = self._ring(first, count, produce)
            call("msb_window_sweep_ring", len(self.slabs), arr, self.S, self.P, first, count, _p(self._ctx), s0._cs)
        for s in self.slabs:
            s._params.jump = s._jump.data_ptr()

    def sweep(self, n_sweeps: int = 1) -> None:
        s0 = self.slab
        k = int(n_sweeps)
        if k <= 0:
            return
        if self.direct:
            while k > 0:
                r = min(k, self.S)
                for s in self.slabs:
                    s._params.block = 2 * s.sweeps_done
                if len(self.slabs) == 1:
                    call("msb_direct_sweep", ctypes.byref(s0._g), ctypes.byref(s0._params), _p(s0._spins), r,
                         _p(s0._flips), ctypes.byref(self._halos[0]), None, s0._cs)
                else:
                    call("msb_direct_sweep_ring", len(self.slabs), self._ring(0, r, False), r, _p(self._ctx), s0._cs)
                for s in self.slabs:
                    s.sweeps_done += r
                k -= r
            return
        if not self._valid:
            self._wbase, self._wc, self._cur = 2 * s0.sweeps_done, 0, 0
            if s0.stream == "xoshiro":
                for s, (states, _, _) in zip(self.slabs, self._wb):
                    call("msb_window_init", ctypes.byref(s._g), ctypes.c_uint64(s.seed & _M64), self.S, self.P,
                         ctypes.c_uint64(self._wbase), _p(s._pow), _p(states), s0._cs)
            self._launch(0, 0, True)
            self._valid = True
        while k > 0:
            r = min(k, self.S - self._wc)
            finish = self._wc + r == self.S
            self._launch(self._wc, r, finish)
            for s in self.slabs:
                s.sweeps_done += r
            k -= r
            if finish:
                self._cur, self._wc, self._wbase = 1 - self._cur, 0, self._wbase + 2 * self.S
            else:
                self._wc += r

    def observe_async(self):
        """Device int64 [2*n_sim] (ups, unsat) of this process's slabs,
        stream-ordered: a device-side wait until the neighbours finished the
        phases so far (our ghost rows are current), then msb_observe.  No
        host synchronisation; callers with world > 1 all-reduce the result."""
        s0 = self.slab
        total = None
        for v, s in enumerate(self.slabs):
            call("msb_window_sweep", ctypes.byref(s._g), ctypes.byref(s._params), self.S, self.P, None, None, None,
                 0, 0, None, None, ctypes.byref(self._halos[v]), None, s0._cs)
            with s0.stream_ctx():
                s._obs.zero_()
            call("msb_observe", ctypes.byref(s._g), _p(s._spins), _p(s._obs[: s.n_sim]), _p(s._obs[s.n_sim:]), s0._cs)
            # the sum over the slabs on the slabs' stream too: on the caller's
            # current stream it could read a slab's counters before msb_observe
            # has written them
            with s0.stream_ctx():
                total = s._obs if total is None else total + s._obs
        return total

    def observables(self):
        """(ups, unsat) int64 per replica of this process's slabs (host copies)."""
        o = self.observe_async()
        self.slab.synchronize()
        h = o.cpu().numpy()
        n = self.slab.n_sim
        return h[:n].copy(), h[n:].copy()

    def synchronize(self) -> None:
        self.slab.synchronize()
