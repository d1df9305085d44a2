"""Host-side view of the reference RNG stream (pkg/src/multispin/rng.py:53-236).

The sweep kernels generate the reference's xoshiro256++ streams on the GPU
(csrc/msb_sweep.cu, csrc/msb_common.cuh).  This module keeps the host API the reference exports
-- scalar ``Xoshiro256pp``, lock-step ``XoshiroStreams`` and
``shape_unit_float`` -- for callers that draw on the host (e.g. custom
streams handed to ``Engine.streams``).  It is not on the hot path.
"""

from __future__ import annotations

import numpy as np

__all__ = ["Xoshiro256pp", "XoshiroStreams", "stream_state", "shape_unit_float", "DeviceStreams",
           "philox4x32_10", "PhiloxStreams", "PhiloxBitStreams", "PBITS_PLANES", "PBITS_CALLS"]

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


# ---------------------------------------------------------------------------
# Counter-based stream
# ---------------------------------------------------------------------------

_PM0, _PM1, _PW0, _PW1 = 0xD2511F53, 0xCD9E8D57, 0x9E3779B9, 0xBB67AE85


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11) on numpy uint32
    arrays (or ints); returns the four output words."""
    u32 = np.uint32
    c0, c1, c2, c3 = (np.asarray(v, dtype=np.uint64) for v in (c0, c1, c2, c3))
    k0 = np.uint64(int(k0) & 0xFFFFFFFF)
    k1 = np.uint64(int(k1) & 0xFFFFFFFF)
    m32 = np.uint64(0xFFFFFFFF)
    for _ in range(10):
        p0 = c0 * np.uint64(_PM0)
        p1 = c2 * np.uint64(_PM1)
        n0 = (p1 >> np.uint64(32)) ^ c1 ^ k0
        n2 = (p0 >> np.uint64(32)) ^ c3 ^ k1
        c1 = p1 & m32
        c3 = p0 & m32
        c0, c2 = n0 & m32, n2 & m32
        k0 = (k0 + np.uint64(_PW0)) & m32
        k1 = (k1 + np.uint64(_PW1)) & m32
    return tuple(v.astype(u32) for v in (c0, c1, c2, c3))


class PhiloxStreams:
    """Counter-based replacement for ``XoshiroStreams`` (rng.py:150-220).

    Draw d of stream S (= first_stream + column) is the low 23 bits of word
    d & 3 of Philox4x32-10 with counter (d >> 2 as 64 bits, S as 64 bits)
    and key = master_seed (64 bits), shaped to k * 2**-23 like every
    reference draw (rng.py:180-183).  ``unit_block(count)`` has the
    reference's semantics: every stream advances by ``count`` draws, so the
    reference ``Engine`` accepts it as ``engine.streams`` unchanged; the GPU
    kernels generate the same draws from (seed, stream, draw index) alone.
    """

    def __init__(self, master_seed: int, n_streams: int, first_stream: int = 0, position: int = 0):
        if n_streams < 1:
            raise ValueError("need at least one stream")
        self.master_seed = int(master_seed) & ((1 << 64) - 1)
        self.n_streams = int(n_streams)
        self.first_stream = int(first_stream)
        self.position = int(position)

    def raw_block(self, count: int) -> np.ndarray:
        """(count, n_streams) uint32: the 32-bit Philox output word of each draw."""
        d = self.position + np.arange(count, dtype=np.uint64)[:, None]
        sid = (self.first_stream + np.arange(self.n_streams, dtype=np.uint64))[None, :]
        c = d >> np.uint64(2)
        shape = np.broadcast_shapes(d.shape, sid.shape)
        m32 = np.uint64(0xFFFFFFFF)
        words = philox4x32_10(np.broadcast_to(c & m32, shape), np.broadcast_to(c >> np.uint64(32), shape),
                              np.broadcast_to(sid & m32, shape), np.broadcast_to(sid >> np.uint64(32), shape),
                              self.master_seed & 0xFFFFFFFF, self.master_seed >> 32)
        e = np.broadcast_to((d & np.uint64(3)).astype(np.intp), shape)
        out = np.choose(e, words)
        self.position += count
        return out.astype(np.uint32)

    def unit_block(self, count: int) -> np.ndarray:
        return (self.raw_block(count) & np.uint32(0x7FFFFF)).astype(np.float64) * 2.0 ** -23

    def __repr__(self) -> str:
        return (f"PhiloxStreams(master_seed={self.master_seed}, n_streams={self.n_streams}, "
                f"first_stream={self.first_stream}, position={self.position})")


PBITS_PLANES = 23   # bit planes of a draw (u23, most significant first)
PBITS_CALLS = 6     # Philox blocks per 32-draw group: 4 planes each, the 24th word unused
PBITS_DOMAIN = 0x80000000  # set in the stream's high counter word: separates these blocks from PhiloxStreams'


class PhiloxBitStreams:
    """Counter-based stream defined by bit planes, for lazy comparison on the
    GPU (SURVEY F1 option).

    Draws come in groups of 32 consecutive draws of a stream: group g holds
    draws 32g .. 32g+31.  Philox4x32-10 block j (0..5) of group g, with
    counter (g lo, (g hi << 3) | j, S lo, S hi | 2^31) and key = master_seed,
    gives four plane words, planes 4j .. 4j+3.  Draw d = 32g + i is the
    23-bit number whose bit 22-b is bit i of plane b (b = 0..22), shaped to
    u23 * 2**-23 like every reference draw (rng.py:180-183).

    A Metropolis test u < K reads u from the most significant plane down and
    stops at the first bit where u and K differ, so 32 draws (one plane word)
    resolve after ~7 planes instead of 23 bits each.  The GPU generates only
    the planes its 32 comparisons need (``Engine(stream="philox-bits")``).
    The comparison results are the same, so this class replays it exactly
    through the reference ``Engine`` (as ``engine.streams``, like
    ``PhiloxStreams``).
    """

    def __init__(self, master_seed: int, n_streams: int, first_stream: int = 0, position: int = 0):
        if n_streams < 1:
            raise ValueError("need at least one stream")
        self.master_seed = int(master_seed) & ((1 << 64) - 1)
        self.n_streams = int(n_streams)
        self.first_stream = int(first_stream)
        self.position = int(position)

    def planes(self, g0: int, groups: int) -> np.ndarray:
        """(groups, n_streams, 24) uint32 plane words of groups g0 .. g0+groups-1."""
        g = (int(g0) + np.arange(groups, dtype=np.uint64))[:, None]
        sid = (self.first_stream + np.arange(self.n_streams, dtype=np.uint64))[None, :]
        shape = (groups, self.n_streams)
        m32 = np.uint64(0xFFFFFFFF)
        out = np.empty(shape + (4 * PBITS_CALLS,), np.uint32)
        for j in range(PBITS_CALLS):
            words = philox4x32_10(np.broadcast_to(g & m32, shape),
                                  np.broadcast_to(((g >> np.uint64(32)) << np.uint64(3)) | np.uint64(j), shape),
                                  np.broadcast_to(sid & m32, shape),
                                  np.broadcast_to((sid >> np.uint64(32)) | np.uint64(PBITS_DOMAIN), shape),
                                  self.master_seed & 0xFFFFFFFF, self.master_seed >> 32)
            for e in range(4):
                out[:, :, 4 * j + e] = words[e]
        return out

    def raw_block(self, count: int) -> np.ndarray:
        """(count, n_streams) uint32: the 23-bit value of each draw."""
        d = self.position + np.arange(count, dtype=np.int64)
        g0 = int(self.position) >> 5
        groups = ((int(self.position) + count - 1) >> 5) - g0 + 1 if count > 0 else 0
        pl = self.planes(g0, max(groups, 1))                  # (groups, streams, 24)
        gi = (d >> 5) - g0
        bit = (d & 31).astype(np.uint32)
        u = np.zeros((count, self.n_streams), np.uint32)
        for b in range(PBITS_PLANES):
            u |= ((pl[gi, :, b] >> bit[:, None]) & np.uint32(1)) << np.uint32(PBITS_PLANES - 1 - b)
        self.position += count
        return u

    def unit_block(self, count: int) -> np.ndarray:
        return self.raw_block(count).astype(np.float64) * 2.0 ** -23

    def __repr__(self) -> str:
        return (f"PhiloxBitStreams(master_seed={self.master_seed}, n_streams={self.n_streams}, "
                f"first_stream={self.first_stream}, position={self.position})")
