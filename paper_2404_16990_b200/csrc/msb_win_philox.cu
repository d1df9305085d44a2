// Window-launch kernels of one stream kind (kSrcPhilox); see msb_window.cuh.
#include "msb_window.cuh"

namespace msbk {
int window_run_philox(int nslabs, const msb_ring_slab* slabs, bool ring, int S, int P, int first, int count,
         const msb_window_io* io, void* ctx, void* stream) {
  return window_run<kSrcPhilox>(nslabs, slabs, ring, S, P, first, count, io, ctx, stream);
}
}  // namespace msbk
