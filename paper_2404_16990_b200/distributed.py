"""Replica parallelism across torch.distributed ranks (one process per GPU).

The reference fans replicas out over threads with contiguous slices and a
global stream offset (run_simulations, engine.py:469-479), so any split is
bit-identical.  Here each rank takes the slice np.linspace bounds assign it
(engine.py:470) and runs its own Engine with sim_offset = slice start.
Replicas never interact: there is no data-path collective; the per-rank
Trajectories are gathered once at the end (host objects).
"""

from __future__ import annotations

import numpy as np

from .observables import Trajectory

__all__ = ["replica_slices", "run_replicas_distributed"]


def replica_slices(n_total: int, parts: int) -> list[tuple[int, int]]:
    """Contiguous [lo, hi) slices exactly as run_simulations (engine.py:470)."""
    parts = max(1, min(int(parts), int(n_total)))
    bounds = np.linspace(0, n_total, parts + 1).astype(int)
    return [(int(a), int(b)) for a, b in zip(bounds[:-1], bounds[1:])]


def run_replicas_distributed(dims, temperatures, seed: int, n_sweeps: int, measure_interval: int = 100,
                             init: str = "random", coupling: float = 1.0, group=None, engine_factory=None,
                             device=None) -> Trajectory:
    """Every rank runs its replica slice; every rank returns the merged
    Trajectory (replicas in global order)."""
    import torch.distributed as dist

    temperatures = tuple(float(t) for t in temperatures)
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    slices = replica_slices(len(temperatures), world)
    if engine_factory is None:
        from .engine import Engine
        engine_factory = lambda **kw: Engine(device=device, **kw)  # noqa: E731
    part = None
    if rank < len(slices):
        lo, hi = slices[rank]
        eng = engine_factory(dims=dims, temperatures=temperatures[lo:hi], seed=seed, init=init,
                             coupling=coupling, sim_offset=lo)
        traj = eng.run(n_sweeps, measure_interval)
        part = (lo, traj.sweeps, traj.abs_m, traj.energy, traj.meta)
    parts = [None] * world
    dist.all_gather_object(parts, part, group=group)
    parts = sorted((p for p in parts if p is not None), key=lambda p: p[0])
    meta = dict(parts[0][4])
    meta.update(sim_offset=0, attempts=sum(p[4]["attempts"] for p in parts), ranks=len(parts))
    return Trajectory(sweeps=parts[0][1], abs_m=np.concatenate([p[2] for p in parts], axis=1),
                      energy=np.concatenate([p[3] for p in parts], axis=1), temperatures=temperatures, meta=meta)
