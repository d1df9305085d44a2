"""Out-of-bounds writes, checked without compute-sanitizer (closed on this
GPU pool): every device buffer the engine and the slabs allocate comes
from a guard allocator -- the buffer sits between two 4 KiB bands of a
sentinel byte -- and after sweeps through every kernel family each band must
be intact.  The same runs are compared with the oracle, so a kernel that
wrote outside its rows would also show as a parity failure."""
import numpy as np
import pytest

from tests.conftest import cuda_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]

SENTINEL = 0xA5
GUARD_BYTES = 4096  # keeps the interior 16-byte aligned (uint4 accesses)


class GuardTorch:
    """Stand-in for the torch module inside engine.py / slab.py: CUDA
    empty/zeros come with guard bands, everything else is torch."""

    def __init__(self, torch):
        self._t = torch
        self.allocs = []

    def __getattr__(self, name):
        return getattr(self._t, name)

    def empty(self, *size, dtype=None, device=None, **kw):
        t = self._t
        if device is None or t.device(device).type != "cuda" or kw.get("pin_memory"):
            return t.empty(*size, dtype=dtype, device=device, **kw)
        shape = tuple(size[0]) if len(size) == 1 and isinstance(size[0], (tuple, list)) else tuple(size)
        n = int(np.prod(shape)) if shape else 1
        es = t.empty((), dtype=dtype).element_size()
        g = GUARD_BYTES // es
        buf = t.empty(n + 2 * g, dtype=dtype, device=device)
        raw = buf.view(t.uint8)
        raw[: g * es].fill_(SENTINEL)
        raw[(g + n) * es:].fill_(SENTINEL)
        self.allocs.append((buf, g * es, (g + n) * es))
        return buf[g:g + n].view(shape)

    def zeros(self, *size, dtype=None, device=None, **kw):
        out = self.empty(*size, dtype=dtype, device=device, **kw)
        out.zero_()
        return out

    def check(self):
        self._t.cuda.synchronize()
        bad = []
        for i, (buf, a, b) in enumerate(self.allocs):
            raw = buf.view(self._t.uint8)
            head, tail = raw[:a], raw[b:]
            if not bool((head == SENTINEL).all()) or not bool((tail == SENTINEL).all()):
                bad.append((i, buf.numel(), int((head != SENTINEL).sum()), int((tail != SENTINEL).sum())))
        return bad


@pytest.fixture
def guard(monkeypatch):
    import torch
    from paper_2404_16990_b200 import engine, slab
    g = GuardTorch(torch)
    monkeypatch.setattr(engine, "_torch", lambda: g)
    monkeypatch.setattr(slab, "_torch", lambda: g)
    return g


@pytest.mark.parametrize("m,n,n_sim,stream", [
    (64, 1024, 3, "xoshiro"), (32, 512, 5, "xoshiro"), (16, 2048, 2, "philox"), (64, 1024, 3, "philox-bits"),
    (32, 512, 5, "philox-bits"), (16, 14336, 1, "philox-bits"), (12, 96, 2, "xoshiro"), (16, 160, 2, "philox-bits"),
])
def test_engine_paths_stay_in_bounds(guard, m, n, n_sim, stream):
    import torch
    from oracle import oracle as orc
    from paper_2404_16990_b200 import Engine, LatticeDims
    temps = list(np.linspace(1.7, 3.1, n_sim))
    e = Engine(LatticeDims(m, n), temps, 9, sim_offset=4, stream=stream)
    o = orc.OracleEngine(m, n, temps, 9, sim_offset=4, stream=stream)
    k = e.window + 3
    e.run(k, measure_interval=2)                       # windows / direct launches, partial and full
    o.sweep(k)
    e.flip_red()                                       # per-phase kernels
    e.flip_blue()
    o.sweep(1)
    if (m * -(-n // 1024)) % 4 == 0:                   # host I/O inside the flip launch
        buf = torch.empty(e.packed_nbytes(), dtype=torch.uint8, pin_memory=True)
        e.store_packed(buf)
        e.step_packed(buf, 2, buf)
        e.synchronize()
        o.sweep(2)
    _ = e.state                                        # interop conversions
    assert (e.lattices() == o.spins).all()
    assert e.flips == o.flips
    e._tables[:] = 0.5                                 # generic tables: per-sweep / per-phase path
    e.sweep()
    assert guard.check() == [], "a kernel wrote outside its buffer"
    assert len(guard.allocs) >= 8


@pytest.mark.parametrize("m,n,V,stream", [
    (64, 1024, 1, "xoshiro"), (64, 1024, 2, "philox-bits"), (60, 1024, 3, "xoshiro"), (128, 14336, 2, "xoshiro"),
    (96, 512, 3, "philox-bits"),
])
def test_slab_rings_stay_in_bounds(guard, m, n, V, stream):
    from oracle import oracle as orc
    from paper_2404_16990_b200 import LatticeDims
    from paper_2404_16990_b200.slab import FusedSlabRun, SlabLattice, slab_bounds
    slabs = [SlabLattice(LatticeDims(m, n), [2.2, 2.6], 3, a, b - a, stream=stream) for a, b in slab_bounds(m, V)]
    run = FusedSlabRun(slabs if V > 1 else slabs[0], window=3)
    run.sweep(7)
    run.observables()
    o = orc.OracleEngine(m, n, [2.2, 2.6], 3, stream=stream)
    o.sweep(7)
    assert (np.concatenate([s.lattice_rows() for s in slabs], axis=1) == o.spins).all()
    assert guard.check() == [], "a kernel wrote outside its buffer"


def test_guard_detects_an_overrun(guard):
    """The check itself: a write one word past an interior is reported."""
    t = guard.empty(100, dtype=guard.int32, device="cuda")
    t.fill_(7)
    assert guard.check() == []
    buf, a, b = guard.allocs[-1]
    buf.view(guard.uint8)[b:b + 4].fill_(0)
    assert len(guard.check()) == 1
