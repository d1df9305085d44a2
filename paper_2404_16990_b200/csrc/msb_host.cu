// libmsb200 host-side ABI: status/error reporting, geometry queries,
// threshold planning (the reference's float64 tables -> exact integer keys),
// the GF(2) jump tables and the INT32 issue-peak microbenchmark.
#include "msb_common.cuh"

namespace msbk {

thread_local std::string g_last_error;

int fail(int code, const std::string& why) {
  g_last_error = why;
  return code;
}

int check_geom(const msb_geom* g) {
  if (!g) return fail(MSB_ERR_ARG, "null geometry");
  if (g->m < 4 || g->m % 4)
    return fail(MSB_ERR_ARG, "m=" + std::to_string(g->m) + ": the cell-axis extent must be a multiple of 4 (and >= 4)");
  if (g->n < 32 || g->n % 32)
    return fail(MSB_ERR_ARG, "n=" + std::to_string(g->n) + ": the memory-axis extent must be a multiple of 32 (and >= 32)");
  if (g->n_sim < 1) return fail(MSB_ERR_ARG, "need at least one replica");
  if (g->ghost != 0 && g->ghost != 1) return fail(MSB_ERR_ARG, "ghost must be 0 or 1");
  if (g->rows < 2 || g->row0 < 0 || g->row0 + g->rows > g->m || (g->rows % 2) || (g->row0 % 2))
    return fail(MSB_ERR_ARG, "held rows must be an even-aligned, even-sized range inside [0, m)");
  if (!g->ghost && (g->row0 != 0 || g->rows != g->m))
    return fail(MSB_ERR_ARG, "a buffer without ghost rows must hold the whole lattice");
  if (g->sim_offset < 0) return fail(MSB_ERR_ARG, "sim_offset must be non-negative");
  return MSB_OK;
}

int check_params(const msb_sweep_params* p) {
  // (piece and quad counts are checked against 2^31 where launched)
  if (!p) return fail(MSB_ERR_ARG, "null sweep parameters");
  const int kg = p->kg;
  if (kg != 1 && kg != 2 && kg != 4 && kg != 8 && kg != 16) return fail(MSB_ERR_ARG, "kg must be 1, 2, 4, 8 or 16");
  if (p->n_planes < 0 || p->n_planes > MSB_MAX_PLANES) return fail(MSB_ERR_ARG, "bad plane count");
  if (p->mode != MSB_MODE_GENERIC && p->n_planes != 2) return fail(MSB_ERR_ARG, "ferro/anti modes use exactly 2 planes");
  if (p->mode < 0 || p->mode > 2) return fail(MSB_ERR_ARG, "bad mode");
  if (p->n_planes > 0 && !p->thr9) return fail(MSB_ERR_ARG, "null thresholds");
  if (!p->work) return fail(MSB_ERR_ARG, "null work counter (4 zeroed uint32 per engine)");
  if (p->rng != MSB_RNG_XOSHIRO && p->rng != MSB_RNG_PHILOX && p->rng != MSB_RNG_PHILOX_BITS) return fail(MSB_ERR_ARG, "unknown rng");
  return MSB_OK;
}

namespace {
// Issue-bound INT32 peak: independent LOP3 (ALU pipe) and IMAD (FMA pipe)
// chains, 1:1, no cross-chain dependences.
constexpr int kPeakChains = 8;
__global__ void k_int_peak(uint32_t* out, uint32_t seed, int iters) {
  uint32_t a[kPeakChains], b[kPeakChains];
#pragma unroll
  for (int i = 0; i < kPeakChains; i++) {
    a[i] = seed * (threadIdx.x + i + 1);
    b[i] = a[i] ^ 0x9e3779b9u;
  }
  const uint32_t k1 = seed | 1u, k2 = seed >> 3, k3 = seed * 7u;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < kPeakChains; i++) {
      asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[i]) : "r"(k3), "r"(k1));
      asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(b[i]) : "r"(k1), "r"(k2));
    }
  }
  uint32_t acc = 0;
#pragma unroll
  for (int i = 0; i < kPeakChains; i++) acc ^= a[i] ^ b[i];
  if (acc == 0x12345678u) out[threadIdx.x] = acc;
}
}  // namespace
}  // namespace msbk

using namespace msbk;

extern "C" {

const char* msb_status_string(int status) {
  switch (status) {
    case MSB_OK: return "ok";
    case MSB_ERR_ARG: return "invalid argument";
    case MSB_ERR_CUDA: return "CUDA error";
    case MSB_ERR_UNSUPPORTED: return "unsupported";
    default: return "unknown status";
  }
}

const char* msb_last_error(void) { return g_last_error.c_str(); }

int msb_abi_version(void) { return 2; }

int msb_check_geom(const msb_geom* g) { return check_geom(g); }

int64_t msb_spin_words(const msb_geom* g) {
  if (check_geom(g)) return -1;
  const Geo G = make_geo(g);
  return (int64_t)G.n_sim * 2 * G.R * G.Wp;
}

int32_t msb_row_pitch(const msb_geom* g) {
  if (check_geom(g)) return -1;
  return make_geo(g).Wp;
}

int64_t msb_pieces_per_phase(const msb_geom* g, int32_t kg) {
  if (check_geom(g)) return -1;
  return (int64_t)g->n_sim * g->rows * kg;
}

int32_t msb_default_kg(const msb_geom* g) {
  if (check_geom(g)) return -1;
  // Smallest split giving ~one warp-unit (32 pieces) per producer warp of
  // every SM (148 SMs x 28 warps); longer pieces amortise the per-sweep
  // jump (64 table lookups) better.
  const long long rows2 = 2LL * g->n_sim * g->rows;
  int kg = 1;
  while (kg < 16 && rows2 * kg < 118000) kg *= 2;
  return kg;
}

int msb_plan_thresholds(const double* tables, int32_t n_sim, int32_t* mode, int32_t* n_planes,
                        int8_t code_plane[16], uint32_t* thr9) {
  if (!tables || n_sim < 1 || !mode || !n_planes || !code_plane || !thr9)
    return fail(MSB_ERR_ARG, "msb_plan_thresholds: null argument");
  constexpr uint32_t kFull = 1u << 23;
  auto K = [&](int s, int code) -> uint32_t {
    const double v = tables[(size_t)s * 16 + code];
    if (!(v > 0.0)) return 0u;  // also NaN: u < NaN is false
    const double x = v * 8388608.0;
    if (!(x < 8388608.0)) return kFull;
    return (uint32_t)std::ceil(x);  // #{k : k 2^-23 < v}
  };
  auto key = [&](uint32_t k) -> uint32_t { return k >= kFull ? kKeyAlways : (k << 9); };
  // J>0 / J<0 structure: codes with >= 2 disagreeing neighbours always flip,
  // exactly-one and none share one threshold each across own = 0/1.
  for (int anti = 0; anti < 2; anti++) {
    bool ok = true;
    for (int s = 0; s < n_sim && ok; s++) {
      for (int own = 0; own < 2 && ok; own++)
        for (int u = 0; u < 5 && ok; u++) {
          const int d = (own ^ anti) ? 4 - u : u;
          if (d >= 2 && K(s, 8 * own + u) != kFull) ok = false;
        }
      const int e4a = anti ? 3 : 1, e4b = anti ? 9 : 11, e8a = anti ? 4 : 0, e8b = anti ? 8 : 12;
      if (K(s, e4a) != K(s, e4b) || K(s, e8a) != K(s, e8b)) ok = false;
    }
    if (!ok) continue;
    *mode = anti ? MSB_MODE_ANTI : MSB_MODE_FERRO;
    *n_planes = 2;
    for (int code = 0; code < 16; code++) {
      const int own = code >> 3, u = code & 7;
      if (u > 4) { code_plane[code] = -1; continue; }
      const int d = (own ^ anti) ? 4 - u : u;
      code_plane[code] = (int8_t)(d >= 2 ? -2 : d == 1 ? 0 : 1);
    }
    for (int s = 0; s < n_sim; s++) {
      thr9[0 * n_sim + s] = key(K(s, anti ? 3 : 1));
      thr9[1 * n_sim + s] = key(K(s, anti ? 4 : 0));
    }
    return MSB_OK;
  }
  // generic: one plane per distinct per-replica threshold vector
  int np = 0;
  int rep[MSB_MAX_PLANES];
  for (int code = 0; code < 16; code++) {
    const int u = code & 7;
    if (u > 4) { code_plane[code] = -1; continue; }
    bool all_full = true, all_zero = true;
    for (int s = 0; s < n_sim; s++) {
      const uint32_t k = K(s, code);
      all_full &= k == kFull;
      all_zero &= k == 0;
    }
    if (all_full) { code_plane[code] = -2; continue; }
    if (all_zero) { code_plane[code] = -1; continue; }
    int found = -1;
    for (int p = 0; p < np && found < 0; p++) {
      bool same = true;
      for (int s = 0; s < n_sim && same; s++) same = K(s, rep[p]) == K(s, code);
      if (same) found = p;
    }
    if (found < 0) {
      found = np;
      rep[np++] = code;
    }
    code_plane[code] = (int8_t)found;
  }
  for (int p = 0; p < np; p++)
    for (int s = 0; s < n_sim; s++) thr9[p * n_sim + s] = key(K(s, rep[p]));
  *mode = MSB_MODE_GENERIC;
  *n_planes = np;
  return MSB_OK;
}

int msb_rng_power_tables(uint32_t* host_out) {
  if (!host_out) return fail(MSB_ERR_ARG, "null output");
  msb::power_tables(host_out);
  return MSB_OK;
}

int msb_rng_jump_table(uint64_t jump, uint32_t* host_out) {
  if (!host_out) return fail(MSB_ERR_ARG, "null output");
  msb::jump_table(jump, host_out);
  return MSB_OK;
}

int msb_bench_int_peak(int32_t blocks, int32_t iters, double* ops_out, float* ms_out, void* stream) {
  if (blocks < 1 || iters < 1 || !ops_out || !ms_out) return fail(MSB_ERR_ARG, "bad arguments");
  cudaStream_t st = as_stream(stream);
  uint32_t* d = nullptr;
  CUDA_TRY(cudaMalloc(&d, 4096));
  cudaEvent_t e0, e1;
  CUDA_TRY(cudaEventCreate(&e0));
  CUDA_TRY(cudaEventCreate(&e1));
  k_int_peak<<<blocks, 256, 0, st>>>(d, 7u, iters);  // warm-up
  CUDA_TRY(cudaEventRecord(e0, st));
  k_int_peak<<<blocks, 256, 0, st>>>(d, 7u, iters);
  CUDA_TRY(cudaEventRecord(e1, st));
  CUDA_TRY(cudaEventSynchronize(e1));
  CUDA_TRY(cudaEventElapsedTime(ms_out, e0, e1));
  *ops_out = (double)blocks * 256 * iters * kPeakChains * 2;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d);
  return MSB_OK;
}

}  // extern "C"
