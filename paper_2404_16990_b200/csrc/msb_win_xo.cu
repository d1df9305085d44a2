// Window-launch kernels of one stream kind (kSrcXoshiro); see msb_window.cuh.
#include "msb_window.cuh"

namespace msbk {
int window_run_xoshiro(int nslabs, const msb_ring_slab* slabs, bool ring, int S, int P, int first, int count,
         const msb_window_io* io, void* ctx, void* stream) {
  return window_run<kSrcXoshiro>(nslabs, slabs, ring, S, P, first, count, io, ctx, stream);
}
}  // namespace msbk

using namespace msbk;

extern "C" {
#ifdef MSB_TRACE
int msb_debug_trace_win(uint64_t* host_out, int32_t n) {
  if (n > kTraceWarps * 8) n = kTraceWarps * 8;
  CUDA_TRY(cudaDeviceSynchronize());
  CUDA_TRY(cudaMemcpyFromSymbol(host_out, g_trace, (size_t)n * 8));
  return MSB_OK;
}
#endif
}
