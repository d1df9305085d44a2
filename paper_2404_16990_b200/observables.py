"""Trajectory container returned by ``Engine.run`` / ``run_simulations``.

Boundary type of the drop-in API, restating the reference's dataclass
(pkg/src/multispin/observables.py:27-61): ``abs_m[k, s]`` and
``energy[k, s]`` are measurement k (taken at sweep ``sweeps[k]``) of replica
s; ``meta`` echoes the configuration plus counters.  The reference's
post-processing statistics (equilibration detection, Onsager summary) are
host-side analysis outside the hot path and are not part of this package.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

__all__ = ["Trajectory"]


@dataclass
class Trajectory:
    sweeps: np.ndarray
    abs_m: np.ndarray
    energy: np.ndarray
    temperatures: tuple
    meta: dict = field(default_factory=dict)

    def __post_init__(self) -> None:
        n_sim = len(self.temperatures)
        if self.abs_m.shape != (self.sweeps.size, n_sim):
            raise ValueError("abs_m shape does not match sweeps x simulations")
        if self.energy.shape != self.abs_m.shape:
            raise ValueError("energy shape does not match abs_m")
        if self.sweeps.size and (np.diff(self.sweeps) <= 0).any():
            raise ValueError("measurement sweep indices must be strictly increasing")

    @property
    def n_measurements(self) -> int:
        return int(self.sweeps.size)

    @property
    def n_sim(self) -> int:
        return len(self.temperatures)

    def series(self, sim: int) -> np.ndarray:
        return self.abs_m[:, sim]
