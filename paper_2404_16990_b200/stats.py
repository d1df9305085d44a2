"""Equilibration statistics of |M| series, for the CLI's ``validate`` command.

Restates the reference's host post-processing (pkg/src/multispin/
observables.py:64-153) with the same float64 numpy expressions, so reports
built from bit-identical trajectories are identical too:

* ``statistical_inefficiency`` -- g = 1 + 2 sum_k rho(k), summed up to the
  first non-positive normalised autocorrelation (observables.py:64-83);
* ``detect_equilibration`` -- the origin on a geometric grid over the first
  three quarters that maximises the effective sample count (N - t0) / g
  (observables.py:86-109);
* ``summarize`` -- equilibrated mean, its standard error from the effective
  sample count, and the deviation from Onsager's |M| (observables.py:112-153).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .layout import onsager_magnetization

__all__ = ["statistical_inefficiency", "detect_equilibration", "Summary", "summarize"]


def statistical_inefficiency(series) -> float:
    x = np.asarray(series, dtype=np.float64).ravel()
    if x.size < 10:
        raise ValueError(f"need at least 10 samples, got {x.size}")
    dev = x - x.mean()
    variance = float((dev * dev).mean())
    if variance == 0.0:
        return 1.0
    g = 1.0
    for lag in range(1, x.size):
        rho = float((dev[:-lag] * dev[lag:]).mean()) / variance
        if rho <= 0.0:
            break
        g += 2.0 * rho
    return max(1.0, g)


def detect_equilibration(series, n_origins: int = 10) -> tuple[int, float, float]:
    x = np.asarray(series, dtype=np.float64).ravel()
    if x.size < 20:
        raise ValueError(f"equilibration detection needs at least 20 measurements, got {x.size}")
    if x.std() == 0.0:
        return 0, 1.0, float(x.size)
    top = max(1, (3 * x.size) // 4)
    origins = [0] + [int(t) for t in np.unique(np.geomspace(1, top, n_origins - 1).astype(int))
                     if x.size - t >= 10]
    best_neff, best_t0, best_g = -1.0, 0, 1.0
    for t0 in origins:
        g = statistical_inefficiency(x[t0:])
        neff = (x.size - t0) / g
        if neff > best_neff:
            best_neff, best_t0, best_g = neff, t0, g
    return best_t0, best_g, best_neff


@dataclass(frozen=True)
class Summary:
    temperature: float
    mean_abs_m: float
    stderr: float
    onsager_abs_m: float
    deviation: float
    t0: int
    g: float
    n_eff: float
    n_used: int


def summarize(series, temperature: float, coupling: float = 1.0) -> Summary:
    x = np.asarray(series, dtype=np.float64).ravel()
    if x.size == 0:
        raise ValueError("empty trajectory: run longer or measure more often")
    t0, g, n_eff = detect_equilibration(x)
    tail = x[t0:]
    if tail.size == 0:
        raise ValueError("no post-equilibration data: run longer")
    mean = float(tail.mean())
    spread = float(tail.std(ddof=1)) if tail.size > 1 else 0.0
    exact = onsager_magnetization(temperature, coupling)
    return Summary(temperature=float(temperature), mean_abs_m=mean, stderr=float(spread / np.sqrt(n_eff)),
                   onsager_abs_m=exact, deviation=mean - exact, t0=t0, g=g, n_eff=n_eff, n_used=int(tail.size))
