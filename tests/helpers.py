"""Shared test helpers (fixture decoding)."""
import numpy as np


def unpack_lattice(packed: np.ndarray, n: int) -> np.ndarray:
    """Inverse of np.packbits(spins > 0, axis=-1): +/-1 int8 lattices."""
    bits = np.unpackbits(packed, axis=-1)[..., :n]
    return np.where(bits == 1, 1, -1).astype(np.int8)


def case(golden, name):
    for c in golden["_manifest"]:
        if c["name"] == name:
            return c
    raise KeyError(name)
