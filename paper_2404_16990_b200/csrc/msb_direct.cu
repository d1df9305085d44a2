// Direct-sweep kernels (bit-plane Philox stream, no accept planes); see msb_window.cuh.
#include "msb_window.cuh"

namespace msbk {
int direct_run(int nslabs, const msb_ring_slab* slabs, bool ring, int n_sweeps, const msb_window_io* io, void* ctx,
               void* stream) {
  return direct_run_impl<>(nslabs, slabs, ring, n_sweeps, io, ctx, stream);
}
}  // namespace msbk
