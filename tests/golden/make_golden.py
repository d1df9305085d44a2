"""Generate golden fixtures by running the UNMODIFIED reference `multispin`.

Run in the build container (the reference is importable only there):

    python tests/golden/make_golden.py

It imports the reference from /root/reference/pkg/src (read-only), runs the
configurations below through its own public API (Engine / run_simulations /
record_engine_randoms / Xoshiro256pp), and writes small compressed fixtures
to tests/golden/reference_runs.npz.  The GPU box never needs the reference:
tests compare against these vectors.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
OUT = Path(__file__).resolve().parent / "reference_runs.npz"

# (name, m, n, temperatures, seed, init, coupling, sim_offset, n_sweeps, measure_interval, table_override)
ENGINE_CASES = [
    ("a_12x96_T2", 12, 96, [2.0], 31, "random", 1.0, 0, 60, 1, None),
    ("b_4x32", 4, 32, [2.0], 37, "random", 1.0, 0, 30, 1, None),
    ("c_16x96", 16, 96, [2.0], 37, "random", 1.0, 0, 30, 1, None),
    ("d_8x64", 8, 64, [2.0], 37, "random", 1.0, 0, 30, 1, None),
    ("e_cfg1_128x128", 128, 128, [2.269], 2024, "random", 1.0, 0, 200, 1, None),
    ("f_multi4", 12, 96, [1.5, 2.0, 2.5, 3.0], 77, "random", 1.0, 0, 30, 10, None),
    ("g_slice_off2", 12, 96, [2.5, 3.0], 77, "random", 1.0, 2, 30, 10, None),
    ("h_antiferro", 8, 64, [1.5], 11, "random", -1.0, 0, 20, 5, None),
    ("i_J0", 4, 32, [2.0], 5, "random", 0.0, 0, 3, 1, None),
    ("j_allup_2T", 32, 64, [1.0, 3.0], 9, "all-up", 1.0, 0, 40, 8, None),
    ("k_table_half", 12, 96, [2.0], 4, "random", 1.0, 0, 10, 5, 0.5),
    ("l_table_zero", 12, 96, [2.0], 3, "random", 1.0, 0, 2, 1, 0.0),
    ("m_table_one", 12, 96, [2.0], 3, "random", 1.0, 0, 2, 1, 1.0),
    ("n_bigseed", 8, 96, [2.269], (1 << 64) - 3, "random", 1.0, 0, 10, 5, None),
    ("o_64x256x3", 64, 256, [1.8, 2.269, 2.7], 123, "random", 1.0, 0, 6, 3, None),
    ("p_coupling2", 16, 128, [3.0], 8, "random", 2.0, 0, 12, 4, None),
    ("q_lowT", 12, 96, [0.5], 31, "random", 1.0, 0, 20, 10, None),
    ("r_highT", 12, 96, [5.0], 31, "random", 1.0, 0, 20, 10, None),
]


# (name, m, n, temperatures, seed, init, coupling, sim_offset, n_sweeps, measure_interval)
PHILOX_CASES = [
    ("px_12x96", 12, 96, [2.0], 31, "random", 1.0, 0, 30, 1),
    ("px_128x128", 128, 128, [2.269], 2024, "random", 1.0, 0, 50, 5),
    ("px_multi", 16, 256, [1.5, 2.269, 3.0], 7, "random", 1.0, 3, 12, 4),
    ("px_anti", 8, 64, [1.5], 11, "random", -1.0, 0, 10, 5),
    ("px_bigseed", 4, 32, [2.0], (1 << 64) - 3, "all-up", 1.0, 0, 10, 10),
]

# Bit-plane counter stream (PhiloxBitStreams): full 32-draw chunks, 16-draw
# chunks (n = 512), and chunks straddling 32-draw groups (n/32 = 3, 5).
PBITS_CASES = [
    ("pb_12x96", 12, 96, [2.0], 31, "random", 1.0, 0, 30, 1),
    ("pb_32x1024", 32, 1024, [1.8, 2.6], 5, "random", 1.0, 1, 12, 4),
    ("pb_16x512", 16, 512, [2.269], 9, "random", 1.0, 0, 10, 5),
    ("pb_8x160", 8, 160, [2.5], 3, "random", 1.0, 0, 8, 4),
    ("pb_anti", 8, 64, [1.5], 11, "random", -1.0, 0, 10, 5),
    ("pb_bigseed", 4, 32, [2.0], (1 << 64) - 3, "all-up", 1.0, 0, 10, 10),
]


def main() -> None:
    sys.path.insert(0, REF)
    from multispin import Engine, LatticeDims, Xoshiro256pp
    from multispin.reference import record_engine_randoms

    data: dict[str, np.ndarray] = {}
    manifest = []

    # RNG known-answer vectors (test_rng.py:63-73 pins 2024/0 and 2024/1).
    rng_cases = [(2024, 0), (2024, 1), (7, 13), (0xDEADBEEF, 999), (5, (1 << 48) + 3),
                 ((1 << 64) - 3, 17), (0, 0)]
    data["rng_cases"] = np.array([[s & ((1 << 64) - 1), st] for s, st in rng_cases], np.uint64)
    gens = [Xoshiro256pp(s, st) for s, st in rng_cases]
    data["rng_out"] = np.stack([np.array([g.next_raw64() for _ in range(64)], np.uint64)
                                for g in gens])

    for (name, m, n, temps, seed, init, J, off, sweeps, mi, table) in ENGINE_CASES:
        dims = LatticeDims(m, n)
        eng = Engine(dims, temps, seed, init=init, coupling=J, sim_offset=off)
        if table is not None:
            eng._tables[:] = table
        start = np.stack([eng.lattice(s) for s in range(eng.n_sim)])
        traj = eng.run(sweeps, measure_interval=mi)
        final = np.stack([eng.lattice(s) for s in range(eng.n_sim)])
        data[f"{name}/start"] = np.packbits(start > 0, axis=-1)
        data[f"{name}/final"] = np.packbits(final > 0, axis=-1)
        data[f"{name}/sweeps"] = traj.sweeps
        data[f"{name}/abs_m"] = traj.abs_m
        data[f"{name}/energy"] = traj.energy
        data[f"{name}/flips"] = np.array([eng.flips], np.int64)
        data[f"{name}/attempts"] = np.array([eng.attempts], np.int64)
        data[f"{name}/state"] = eng.state.copy()
        manifest.append(dict(name=name, m=m, n=n, temperatures=temps, seed=str(seed), init=init,
                             coupling=J, sim_offset=off, n_sweeps=sweeps, measure_interval=mi,
                             table=table))
        print(f"{name}: flips={eng.flips}", flush=True)

    # Draw map recorded through the reference's own recorder hook.
    dims = LatticeDims(12, 96)
    eng = Engine(dims, [2.0], 21, init="random")
    rmap = record_engine_randoms(eng, 3)
    data["drawmap_12x96_seed21"] = np.round(rmap.draws * (1 << 23)).astype(np.uint32)

    # from_lattices start (test_engine.py random_spins pattern).
    spins = np.random.default_rng(2).choice(np.array([-1, 1], np.int8), size=(12, 96))
    eng = Engine.from_lattices([spins], [2.0], seed=1)
    traj = eng.run(10, measure_interval=5)
    data["fromlat/start"] = np.packbits(spins > 0, axis=-1)
    data["fromlat/final"] = np.packbits(eng.lattice(0) > 0, axis=-1)
    data["fromlat/abs_m"] = traj.abs_m
    data["fromlat/energy"] = traj.energy
    data["fromlat/flips"] = np.array([eng.flips], np.int64)

    # Counter-based stream: the reference Engine itself, handed a
    # PhiloxStreams as its duck-typed `streams` (engine.py:259-261, 336).
    sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
    from paper_2404_16990_b200.rng import PhiloxStreams
    philox_manifest = []
    for (name, m, n, temps, seed, init, J, off, sweeps, mi) in PHILOX_CASES:
        dims = LatticeDims(m, n)
        eng = Engine(dims, temps, seed, init=init, coupling=J, sim_offset=off)
        eng.streams = PhiloxStreams(seed, len(temps) * dims.cells, off * dims.cells)
        traj = eng.run(sweeps, measure_interval=mi)
        final = np.stack([eng.lattice(s) for s in range(eng.n_sim)])
        data[f"{name}/final"] = np.packbits(final > 0, axis=-1)
        data[f"{name}/abs_m"] = traj.abs_m
        data[f"{name}/energy"] = traj.energy
        data[f"{name}/flips"] = np.array([eng.flips], np.int64)
        philox_manifest.append(dict(name=name, m=m, n=n, temperatures=temps, seed=str(seed), init=init,
                                    coupling=J, sim_offset=off, n_sweeps=sweeps, measure_interval=mi))
        print(f"{name}: flips={eng.flips}", flush=True)
    data["philox_manifest"] = np.frombuffer(json.dumps(philox_manifest).encode(), np.uint8)

    # Bit-plane counter stream, the same way (the reference Engine fed a
    # PhiloxBitStreams; the GPU compares these draws plane by plane, lazily).
    from paper_2404_16990_b200.rng import PhiloxBitStreams
    pbits_manifest = []
    for (name, m, n, temps, seed, init, J, off, sweeps, mi) in PBITS_CASES:
        dims = LatticeDims(m, n)
        eng = Engine(dims, temps, seed, init=init, coupling=J, sim_offset=off)
        eng.streams = PhiloxBitStreams(seed, len(temps) * dims.cells, off * dims.cells)
        traj = eng.run(sweeps, measure_interval=mi)
        final = np.stack([eng.lattice(s) for s in range(eng.n_sim)])
        data[f"{name}/final"] = np.packbits(final > 0, axis=-1)
        data[f"{name}/abs_m"] = traj.abs_m
        data[f"{name}/energy"] = traj.energy
        data[f"{name}/flips"] = np.array([eng.flips], np.int64)
        pbits_manifest.append(dict(name=name, m=m, n=n, temperatures=temps, seed=str(seed), init=init,
                                   coupling=J, sim_offset=off, n_sweeps=sweeps, measure_interval=mi))
        print(f"{name}: flips={eng.flips}", flush=True)
    data["pbits_manifest"] = np.frombuffer(json.dumps(pbits_manifest).encode(), np.uint8)

    data["manifest"] = np.frombuffer(json.dumps(manifest).encode(), np.uint8)
    np.savez_compressed(OUT, **data)
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes)")


if __name__ == "__main__":
    main()
