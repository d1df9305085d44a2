// Window-launch kernels of one stream kind (kSrcPbits); see msb_window.cuh.
#include "msb_window.cuh"

namespace msbk {
int window_run_pbits(int nslabs, const msb_ring_slab* slabs, bool ring, int S, int P, int first, int count,
         const msb_window_io* io, void* ctx, void* stream) {
  return window_run<kSrcPbits>(nslabs, slabs, ring, S, P, first, count, io, ctx, stream);
}
}  // namespace msbk
