// Cross-translation-unit entry points of the window / direct launch drivers
// (msb_window.cuh), one translation unit per stream kind so the kernel
// instantiations compile in parallel.  Plain ABI types only.
#pragma once
#include "../../include/msb200.h"

namespace msbk {
int window_run_xoshiro(int nslabs, const msb_ring_slab* slabs, bool ring, int S, int P, int first, int count,
                       const msb_window_io* io, void* ctx, void* stream);
int window_run_philox(int nslabs, const msb_ring_slab* slabs, bool ring, int S, int P, int first, int count,
                      const msb_window_io* io, void* ctx, void* stream);
int window_run_pbits(int nslabs, const msb_ring_slab* slabs, bool ring, int S, int P, int first, int count,
                     const msb_window_io* io, void* ctx, void* stream);
int direct_run(int nslabs, const msb_ring_slab* slabs, bool ring, int n_sweeps, const msb_window_io* io, void* ctx,
               void* stream);
}  // namespace msbk
