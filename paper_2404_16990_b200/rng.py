"""Host-side view of the reference RNG stream (pkg/src/multispin/rng.py:53-236).

The sweep kernels generate the reference's xoshiro256++ streams on the GPU
(csrc/msb_kernels.cu).  This module keeps the host API the reference exports
-- scalar ``Xoshiro256pp``, lock-step ``XoshiroStreams`` and
``shape_unit_float`` -- for callers that draw on the host (e.g. custom
streams handed to ``Engine.streams``).  It is not on the hot path.
"""

from __future__ import annotations

import numpy as np

__all__ = ["Xoshiro256pp", "XoshiroStreams", "stream_state", "shape_unit_float", "DeviceStreams"]

_M64 = (1 << 64) - 1
_PHI = 0x9E3779B97F4B7C15


def _mix(z: int) -> int:
    z &= _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def stream_state(master_seed: int, stream: int) -> list[int]:
    """256-bit state of stream `stream`: the 4 splitmix64 outputs following
    seed mix64(master + (stream+1)*phi); the all-zero state is patched."""
    z = _mix(master_seed + (stream + 1) * _PHI)
    out = []
    for _ in range(4):
        z = (z + _PHI) & _M64
        out.append(_mix(z))
    if not any(out):
        out[0] = _PHI
    return out


def _step(s: list[int]) -> int:
    s0, s1, s2, s3 = s
    x = (s0 + s3) & _M64
    res = ((((x << 23) | (x >> 41)) & _M64) + s0) & _M64
    t = (s1 << 17) & _M64
    s2 ^= s0
    s3 ^= s1
    s1 ^= s2
    s0 ^= s3
    s2 ^= t
    s3 = ((s3 << 45) | (s3 >> 19)) & _M64
    s[:] = [s0, s1, s2, s3]
    return res


class Xoshiro256pp:
    def __init__(self, master_seed: int, stream: int = 0):
        self.master_seed = int(master_seed)
        self.stream = int(stream)
        self._s = stream_state(self.master_seed, self.stream)

    def next_raw64(self) -> int:
        return _step(self._s)

    def next_bits(self, k: int) -> int:
        if not 1 <= k <= 64:
            raise ValueError(f"bit count {k} outside [1, 64]")
        return self.next_raw64() >> (64 - k)

    def next_unit_float(self) -> float:
        return ((self.next_raw64() >> 32) & 0x7FFFFF) * 2.0 ** -23

    def raw64(self, count: int) -> np.ndarray:
        return np.array([_step(self._s) for _ in range(count)], dtype=np.uint64)

    def unit_floats(self, count: int) -> np.ndarray:
        return ((self.raw64(count) >> np.uint64(32)) & np.uint64(0x7FFFFF)) * 2.0 ** -23

    def bits(self, count: int) -> np.ndarray:
        raw = self.raw64(-(-count // 64))
        return np.unpackbits(raw.astype(">u8").view(np.uint8))[:count]


class XoshiroStreams:
    """Lock-step streams; column j of a block is stream first_stream + j."""

    def __init__(self, master_seed: int, n_streams: int, first_stream: int = 0):
        if n_streams < 1:
            raise ValueError("need at least one stream")
        self.master_seed = int(master_seed)
        self.n_streams = int(n_streams)
        self.first_stream = int(first_stream)
        st = np.array([stream_state(self.master_seed, self.first_stream + j)
                       for j in range(self.n_streams)], dtype=np.uint64)
        self._s = [st[:, i].copy() for i in range(4)]

    def raw_block(self, count: int, _force_numpy: bool = True) -> np.ndarray:
        s0, s1, s2, s3 = self._s
        out = np.empty((count, self.n_streams), np.uint64)
        u = lambda k: np.uint64(k)
        for k in range(count):
            x = s0 + s3
            out[k] = ((x << u(23)) | (x >> u(41))) + s0
            t = s1 << u(17)
            s2 = s2 ^ s0
            s3 = s3 ^ s1
            s1 = s1 ^ s2
            s0 = s0 ^ s3
            s2 = s2 ^ t
            s3 = (s3 << u(45)) | (s3 >> u(19))
        self._s = [s0, s1, s2, s3]
        return out

    def unit_block(self, count: int) -> np.ndarray:
        return ((self.raw_block(count) >> np.uint64(32)) & np.uint64(0x7FFFFF)) * 2.0 ** -23


def shape_unit_float(raw32):
    raw = np.atleast_1d(np.asarray(raw32, dtype=np.uint32))
    pattern = (raw & np.uint32(0x007FFFFF)) | np.uint32(0x3F800000)
    shaped = (pattern.view(np.float32) - np.float32(1.0)).astype(np.float64)
    return float(shaped[0]) if np.ndim(raw32) == 0 else shaped


class DeviceStreams:
    """Descriptor of an engine's device-resident flip streams.

    Stands in for the reference's ``Engine.streams`` (engine.py:259-261):
    stream ``first_stream + j`` of ``master_seed`` for j < n_streams.  The
    draws live on the GPU as per-piece xoshiro states; assigning any other
    object with a ``unit_block(count)`` method to ``Engine.streams`` switches
    the engine to host-supplied draws (the reference's duck-typed seam).
    """

    def __init__(self, master_seed: int, n_streams: int, first_stream: int):
        self.master_seed = int(master_seed)
        self.n_streams = int(n_streams)
        self.first_stream = int(first_stream)

    def __repr__(self) -> str:
        return (f"DeviceStreams(master_seed={self.master_seed}, n_streams={self.n_streams}, "
                f"first_stream={self.first_stream})")
