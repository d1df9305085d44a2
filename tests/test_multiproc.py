"""Multi-process host logic on CPU with the gloo backend (world size 2):
the slab ghost exchange and the replica fan-out.  The GPU kernels are
replaced by CPU stand-ins with the same interface; the transport code is
the product code."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class FakeSlab:
    """CPU stand-in exposing the slab transport interface."""

    def __init__(self, rank, n_sim=2, Wp=16):
        self.n_sim, self.Wp, self.rank = n_sim, Wp, rank
        self.got = {}

    def stream_ctx(self):
        import contextlib
        return contextlib.nullcontext()

    def synchronize(self):
        pass

    def edges(self, colour):
        # first row tagged 1000*rank + 10*colour + 1, last row ... + 2
        e = torch.zeros(self.n_sim, 2, self.Wp, dtype=torch.int32)
        e[:, 0] = 1000 * self.rank + 10 * colour + 1
        e[:, 1] = 1000 * self.rank + 10 * colour + 2
        return e.reshape(-1)

    def set_ghosts(self, colour, ghosts):
        self.got[colour] = ghosts.view(self.n_sim, 2, self.Wp).clone()


def _exchange_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2404_16990_b200.slab import DistExchange
    s = FakeSlab(rank)
    ex = DistExchange()
    for colour in (0, 1):
        ex.exchange([s], colour)
    up, down = (rank - 1) % world, (rank + 1) % world
    ok = True
    for colour in (0, 1):
        g = s.got[colour]
        ok &= bool((g[:, 0] == 1000 * up + 10 * colour + 2).all())    # neighbour above: its LAST row
        ok &= bool((g[:, 1] == 1000 * down + 10 * colour + 1).all())  # neighbour below: its FIRST row
    out[rank] = int(ok)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_slab_ghost_exchange_ring(world):
    out = mp.Manager().dict()
    mp.spawn(_exchange_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    assert all(out[r] == 1 for r in range(world))


class OracleEngineFactory:
    """Runs the CPU oracle behind the Engine.run() interface."""

    def __call__(self, dims, temperatures, seed, init, coupling, sim_offset):
        from oracle import oracle as orc
        e = orc.OracleEngine(dims.m, dims.n, temperatures, seed, init=init, coupling=coupling,
                             sim_offset=sim_offset)

        class Run:
            def run(self, n, mi):
                from paper_2404_16990_b200.observables import Trajectory
                sw, am, en = e.run(n, mi)
                return Trajectory(sw, am, en, tuple(temperatures), meta={"attempts": e.attempts})
        return Run()


def _replica_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2404_16990_b200 import LatticeDims
    from paper_2404_16990_b200.distributed import run_replicas_distributed
    temps = (1.5, 2.0, 2.5, 3.0, 3.5)
    traj = run_replicas_distributed(LatticeDims(12, 96), temps, 77, 30, measure_interval=10,
                                    engine_factory=OracleEngineFactory())
    out[rank] = (traj.abs_m.tolist(), traj.energy.tolist(), traj.meta["attempts"])
    dist.destroy_process_group()


def test_replica_fanout_matches_one_process(golden):
    from oracle import oracle as orc
    world = 2
    out = mp.Manager().dict()
    mp.spawn(_replica_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    e = orc.OracleEngine(12, 96, (1.5, 2.0, 2.5, 3.0, 3.5), 77)
    _, am, en = e.run(30, 10)
    for r in range(world):
        got_m, got_e, att = out[r]
        assert np.array_equal(np.array(got_m), am) and np.array_equal(np.array(got_e), en)
        assert att == e.attempts


def test_replica_slices_match_reference_split():
    from paper_2404_16990_b200.distributed import replica_slices
    assert replica_slices(754, 8) == [(0, 94), (94, 188), (188, 282), (282, 377), (377, 471), (471, 565),
                                      (565, 659), (659, 754)]
    assert replica_slices(4, 3) == [(0, 1), (1, 2), (2, 4)]


def _group_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2404_16990_b200.slab import resolve_group
    g, w, r = resolve_group(None)
    out[rank] = (g is dist.group.WORLD, w, r)
    dist.destroy_process_group()


def test_fused_ring_resolves_the_default_group():
    """FusedSlabRun(group=None) under torch.distributed uses the default
    group (round 1 passed None to symm_mem.rendezvous, which raises)."""
    from paper_2404_16990_b200.slab import resolve_group
    assert resolve_group(None) == (None, 1, 0)
    out = mp.Manager().dict()
    mp.spawn(_group_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    assert out[0] == (True, 2, 0) and out[1] == (True, 2, 1)


class _Handle:
    def __init__(self, bases):
        self.buffer_ptrs = bases


@pytest.mark.parametrize("world", [2, 3, 8])
def test_peer_halo_pointers(world):
    """The halo a rank builds from symmetric-memory handles points at the
    ring neighbours' mappings of the same buffers, offsets included."""
    from paper_2404_16990_b200.slab import peer_halo, ring_plan
    m = 14336
    spin_bases = [0x7000_0000_0000 + 0x1_0000_0000 * r for r in range(world)]
    flag_bases = [0x9000_0000_0000 + 0x10_0000 * r for r in range(world)]
    for rank in range(world):
        plan = ring_plan(m, world, rank)
        h = peer_halo(plan, rank, _Handle(spin_bases), _Handle(flag_bases), spin_bases[rank] + 4096,
                      flag_bases[rank])
        up, down = (rank - 1) % world, (rank + 1) % world
        assert (h.up_spins, h.down_spins) == (spin_bases[up] + 4096, spin_bases[down] + 4096)
        assert (h.up_flags, h.down_flags) == (flag_bases[up], flag_bases[down])
        assert h.up_R == ring_plan(m, world, up)["rows"] + 2 and h.down_R == ring_plan(m, world, down)["rows"] + 2
