"""The ctypes binding a reference maintainer would add,
as a module the tests exercise: ``B200Sweeper`` keeps the reference's own
``multispin.Engine`` object and replaces only its sweep loop
(pkg/src/multispin/engine.py:353-360) with libmsb200 calls through the C
ABI (include/msb200.h), reading the device state back into ``eng.state`` on
request.  Nothing of this package's Python Engine is used."""
import ctypes

import numpy as np
import torch

from paper_2404_16990_b200 import _lib  # loads libmsb200.so, declares argtypes

L = _lib.lib()


class B200Sweeper:
    """Device twin of one reference Engine (same dims, temps, seed, offset)."""

    def __init__(self, eng, device="cuda:0"):
        self.g = _lib.geom(eng.n_sim, eng.dims.m, eng.dims.n, sim_offset=eng.sim_offset)
        self.stream = torch.cuda.Stream(device=device)
        cs = ctypes.c_void_p(self.stream.cuda_stream)
        words = L.msb_spin_words(ctypes.byref(self.g))
        kg = L.msb_default_kg(ctypes.byref(self.g))
        pieces = L.msb_pieces_per_phase(ctypes.byref(self.g), kg)
        dev = torch.device(device)
        self.spins = torch.empty(words, dtype=torch.int32, device=dev)
        self.states = torch.empty(16 * pieces, dtype=torch.int32, device=dev)
        self.planes = torch.empty(2 * L.msb_plane_words(ctypes.byref(self.g), 10), dtype=torch.int32, device=dev)
        self.flips = torch.zeros(256, dtype=torch.int64, device=dev)
        self.work = torch.zeros(4, dtype=torch.int32, device=dev)
        # tables -> integer keys (engine.py:257, 321-331)
        mode, npl, codes = ctypes.c_int32(), ctypes.c_int32(), (ctypes.c_int8 * 16)()
        thr = np.zeros(10 * eng.n_sim, np.uint32)
        tab = np.ascontiguousarray(eng._tables)
        _lib.check(L.msb_plan_thresholds(tab.ctypes.data, eng.n_sim, ctypes.byref(mode), ctypes.byref(npl), codes,
                                         thr.ctypes.data), "msb_plan_thresholds")
        self.thr = torch.from_numpy(thr.view(np.int32)).to(dev)
        pw = np.empty(64 * 8192, np.uint32)
        _lib.check(L.msb_rng_power_tables(pw.ctypes.data), "msb_rng_power_tables")
        jt = np.empty(8192, np.uint32)
        _lib.check(L.msb_rng_jump_table(4 * eng.dims.n, jt.ctypes.data), "msb_rng_jump_table")
        self.pow = torch.from_numpy(pw.view(np.int32)).to(dev)
        self.jump = torch.from_numpy(jt.view(np.int32)).to(dev)
        p = _lib.SweepParams()
        p.mode, p.n_planes, p.kg = mode.value, npl.value, kg
        p.code_plane[:] = list(codes)
        p.thr9, p.jump, p.work = self.thr.data_ptr(), self.jump.data_ptr(), self.work.data_ptr()
        self.p = p
        # upload the reference state (interop layout, engine.py:262) and position the streams
        st = torch.from_numpy(np.ascontiguousarray(eng.state).view(np.int16).reshape(-1)).to(dev)
        _lib.check(L.msb_from_ref16(ctypes.byref(self.g), ctypes.c_void_p(st.data_ptr()),
                                    ctypes.c_void_p(self.spins.data_ptr()), cs), "msb_from_ref16")
        _lib.check(L.msb_rng_init(ctypes.byref(self.g), eng.seed & (2**64 - 1), kg, 2 * eng.sweeps_done, -1,
                                  ctypes.c_void_p(self.pow.data_ptr()), ctypes.c_void_p(self.states.data_ptr()), cs),
                   "msb_rng_init")
        self.cs = cs
        self.flips0 = eng.flips

    def sweep(self, eng, n=1):  # replaces Engine.sweep (engine.py:353-360)
        cur = ctypes.c_int32(0)
        st = L.msb_sweep(ctypes.byref(self.g), ctypes.byref(self.p), ctypes.c_void_p(self.spins.data_ptr()),
                         ctypes.c_void_p(self.states.data_ptr()), ctypes.c_void_p(self.planes.data_ptr()),
                         n, 0, ctypes.byref(cur), ctypes.c_void_p(self.flips.data_ptr()), self.cs)
        _lib.check(st, "msb_sweep")
        eng.sweeps_done += n
        eng.attempts += eng.dims.sites * eng.n_sim * n

    def pull_state(self, eng):  # device -> eng.state (halos refreshed)
        out = torch.empty(eng.state.size, dtype=torch.int16, device=self.spins.device)
        _lib.check(L.msb_to_ref16(ctypes.byref(self.g), ctypes.c_void_p(self.spins.data_ptr()),
                                  ctypes.c_void_p(out.data_ptr()), self.cs), "msb_to_ref16")
        self.stream.synchronize()
        eng.state[...] = out.cpu().numpy().view(np.uint16).reshape(eng.state.shape)
        eng.flips = self.flips0 + int(self.flips.sum().item())
