// libmsb200 state kernels: stream positioning, lattice initialisation,
// layout conversions (linear / reference interop), observables, draw export
// and slab halo packing, with their ABI entry points.
#include "msb_io.cuh"

namespace msbk {
namespace {

// ---------------------------------------------------------------------------
// device: state initialisation and layout conversions
// ---------------------------------------------------------------------------

// Piece start states.  Colour X's pieces are positioned at stream block
// `blockX` (one block = the 2n draws a stream spends on one colour phase,
// engine.py:336): piece (row c, kgi) starts at draw
// blockX*2n + q*(n/2) + kgi*(16/kg)*(n/32) of stream (sim_offset+s)*(m/4) + gamma-1.
__global__ void k_rng_init(Geo G, uint64_t seed, int kg, int kr, long long npieces, uint64_t block0,
                           int colour, const uint4* __restrict__ pow, uint32_t* states) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int ncol = colour < 0 ? 2 : 1;
  if (i >= ncol * npieces) return;
  const int X = colour < 0 ? (int)(i / npieces) : colour;
  const uint64_t block = colour < 0 ? block0 + (uint64_t)X : block0;
  const long long gp = i % npieces;
  const long long gr = gp / kg;
  const int kgi = (int)(gp % kg);
  const int s = (int)(gr / G.rows), lr = (int)(gr % G.rows);
  const int c = G.row0 + lr;
  const RowStream rs = row_stream(G.m, c, X);
  const uint64_t cells = (uint64_t)(G.m / 4);
  const uint64_t stream = ((uint64_t)G.sim_offset + (uint64_t)s) * cells + (uint64_t)(rs.gamma - 1);
  const uint64_t n = (uint64_t)G.n;
  const uint64_t offset = block * 2 * n + (uint64_t)rs.q * (n / 2) + (uint64_t)kgi * kr * (uint64_t)G.words;
  XState st = jump_by(stream_state(seed, stream), offset, pow);
  store_state(st, states + (size_t)X * 8 * npieces, npieces, gp);
}

// Reference-stream order outputs of init="random" (engine.py:279-281):
// linear word o of replica s = brev64(output (row0*n/64 + o) of stream
// 2^48 + sim_offset + s), i.e. bit i%64 <-> site i (little-endian order).
constexpr int kInitPiece = 2048;
__global__ void k_init_linear(Geo G, uint64_t seed, long long words_per_sim, const uint4* __restrict__ pow,
                              unsigned long long* lin) {
  const long long per_sim = (words_per_sim + kInitPiece - 1) / kInitPiece;
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= per_sim * G.n_sim) return;
  const int s = (int)(i / per_sim);
  const long long o0 = (i % per_sim) * kInitPiece;
  const long long o1 = min(o0 + kInitPiece, words_per_sim);
  const uint64_t first = (uint64_t)G.row0 * (uint64_t)G.n / 64;
  XState st = stream_state(seed, (1ULL << 48) + (uint64_t)G.sim_offset + (uint64_t)s);
  st = jump_by(st, first + (uint64_t)o0, pow);
  unsigned long long* out = lin + (size_t)s * words_per_sim;
  for (long long o = o0; o < o1; o++) {
    // full 64-bit output needed here (rng.py:139-147 uses all 64 bits)
    const uint64_t a = ((uint64_t)st.a1 << 32) | st.a0, d = ((uint64_t)st.d1 << 32) | st.d0;
    const uint64_t x = a + d;
    const uint64_t r = ((x << 23) | (x >> 41)) + a;
    xstep(st);
    out[o] = __brevll(r);
  }
}

// Linear <-> colour-split and the observables, one warp per group of CPW
// consecutive chunks (msb_io.cuh).
constexpr int kConvThreads = 256;

template <int CPW>
__global__ void __launch_bounds__(kConvThreads) k_from_linear(Geo G, const uint32_t* __restrict__ lin,
                                                               uint32_t* __restrict__ spins, unsigned nwarps) {
  const unsigned wq = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (wq < nwarps) from_linear_group<CPW>(G, lin, spins, wq);  // warp-uniform
}

// The observables are reduced per warp, then per CTA: one atomic per CTA and
// replica run (a CTA's warps are consecutive chunk groups, so it spans one
// replica or the boundary of two).  Per-warp atomics on the n_sim counters
// serialised (35 us at 2 chunks per warp for cfg2).
template <int CPW, bool LIN, bool OBS>
__global__ void __launch_bounds__(kConvThreads) k_export(Geo G, const uint32_t* __restrict__ spins,
                                                          uint32_t* __restrict__ lin, long long* ups,
                                                          long long* unsat, unsigned nwarps) {
  const unsigned wq = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int s = -1;
  uint32_t u = 0, b = 0;
  if (wq < nwarps) s = export_group<CPW, LIN, OBS, false>(G, spins, lin, wq, u, b);  // warp-uniform
  if (OBS) {
    u = __reduce_add_sync(0xFFFFFFFFu, u);
    b = __reduce_add_sync(0xFFFFFFFFu, b);
    constexpr int kW = kConvThreads / 32;
    __shared__ int ss[kW];
    __shared__ uint32_t su[kW], sb[kW];
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
      ss[w] = s;
      su[w] = u;
      sb[w] = b;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int cur = -1;
      unsigned long long tu = 0, tb = 0;
      for (int i = 0; i <= kW; i++) {
        const int si = i < kW ? ss[i] : -1;
        if (si != cur) {
          if (cur >= 0) {
            atomicAdd(reinterpret_cast<unsigned long long*>(ups + cur), tu);
            atomicAdd(reinterpret_cast<unsigned long long*>(unsat + cur), tb);
          }
          cur = si;
          tu = tb = 0;
        }
        if (i < kW) {
          tu += su[i];
          tb += sb[i];
        }
      }
    }
  }
}

__global__ void k_init_const(Geo G, uint32_t up, uint32_t* spins) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long total = (long long)G.n_sim * 2 * G.R * G.Wp;
  if (i >= total) return;
  const int wd = (int)(i % G.Wp);
  const int br = (int)((i / G.Wp) % G.R);
  const bool ghost_row = G.ghost && (br == 0 || br == G.R - 1);
  spins[i] = (up && !ghost_row) ? chunk_mask(G, wd >> 4) : 0u;
}

// Canonical source of a state element (lattice.py:283-329), evaluated per
// element; codes in ALL_CODES order RFE RBO RBE RFO BFE BBO BBE BFO.
__global__ void k_to_ref16(Geo G, const uint32_t* __restrict__ spins, uint16_t* state) {
  const int cells = G.m / 4, words = G.words;
  const int cols = cells + 2, vec = words + 2;
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long total = (long long)G.n_sim * 8 * cols * vec;
  if (i >= total) return;
  int e = (int)(i % vec);
  int g = (int)((i / vec) % cols);
  int a = (int)((i / ((long long)vec * cols)) % 8);
  const int s = (int)(i / (8LL * vec * cols));
  const bool in_moat = g == 0 || g == cols - 1, in_halo = e == 0 || e == vec - 1;
  uint16_t val = 0;
  bool live = true;
  if (in_moat && in_halo) {
    live = false;
  } else if (in_moat) {
    const bool red = a < 4, fill_right = red ? (a % 4) < 2 : (a % 4) >= 2;
    if (fill_right && g == cols - 1) { a ^= 2; g = cells; }
    else if (!fill_right && g == 0) { a ^= 2; g = 1; }
    else live = false;
  } else if (in_halo) {
    const bool copy_top = (a % 2) == 0;
    if (copy_top && e == vec - 1) e = 1;
    else if (!copy_top && e == 0) e = words;
    else live = false;
  }
  if (live) {
    const bool red = a < 4, fwd = (a % 4) == 0 || (a % 4) == 3, even = (a % 2) == 0;
    const int p0 = even ? 0 : 1, cpar = red ? p0 : 1 - p0;
    const int c = fwd ? 2 * (g - 1) + cpar : G.m - 2 * g + cpar;  // lattice.py:190-196
    const int X = red ? 0 : 1;
    const int w = e - 1;
    const uint32_t* row = spins + row_off(G, s, X, c) + (w >> 5) * 16;
    uint32_t v = 0;
#pragma unroll
    for (int t = 0; t < 16; t++) v |= ((row[t] >> (w & 31)) & 1u) << t;
    val = (uint16_t)v;
  }
  state[i] = val;
}

__global__ void k_from_ref16(Geo G, const uint16_t* __restrict__ state, uint32_t* spins) {
  const int cells = G.m / 4, words = G.words;
  const int cols = cells + 2, vec = words + 2;
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long total = (long long)G.n_sim * 2 * G.m * G.Wp;
  if (i >= total) return;
  const int wd = (int)(i % G.Wp);
  const int c = (int)((i / G.Wp) % G.m);
  const int X = (int)((i / ((long long)G.Wp * G.m)) % 2);
  const int s = (int)(i / (2LL * G.Wp * G.m));
  const int ch = wd >> 4, t = wd & 15;
  const RowStream rs = row_stream(G.m, c, X);
  const int a = 4 * X + rs.q;
  const uint16_t* col = state + (((size_t)s * 8 + a) * cols + rs.gamma) * vec + 1 + 32 * ch;
  const int nb = chunk_bits(G, ch);
  uint32_t v = 0;
  for (int b = 0; b < nb; b++) v |= ((uint32_t)(col[b] >> t) & 1u) << b;
  spins[row_off(G, s, X, c) + wd] = v;
}

// ---------------------------------------------------------------------------
// device: observables (engine.py:372-386)
// ---------------------------------------------------------------------------

// (observables: k_export above)

// ---------------------------------------------------------------------------
// device: record/replay, slab halos, INT microbenchmark
// ---------------------------------------------------------------------------

__global__ void k_draws(Geo G, int X, int kg, int kr, long long npieces, const uint32_t* __restrict__ states,
                        int philox, uint32_t seed_lo, uint32_t seed_hi, unsigned long long block, uint32_t* out) {
  const long long gp = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gp >= npieces) return;
  const long long gr = gp / kg;
  const int kgi = (int)(gp % kg);
  const int s = (int)(gr / G.rows), c = (int)(gr % G.rows);
  const RowStream rs = row_stream(G.m, c, X);
  uint32_t* o = out + (((size_t)s * (G.m / 4) + rs.gamma - 1) * 4 + rs.q) * 16 * G.words;
  if (!philox) {
    XState st;
    load_state(st, states + (size_t)X * 8 * npieces, npieces, gp);
    for (int k = kgi * kr; k < (kgi + 1) * kr; k++)
      for (int w = 0; w < G.words; w++) o[(size_t)k * G.words + w] = xstep(st) & 0x7FFFFFu;
    return;
  }
  const unsigned long long sid = ((unsigned long long)G.sim_offset + s) * (unsigned long long)(G.m / 4) + rs.gamma - 1;
  const unsigned long long n = (unsigned long long)G.n;
  const unsigned long long d0 = block * 2 * n + (unsigned long long)rs.q * (n / 2);
  if (philox == 2) {  // bit-plane form
    for (int k = kgi * kr; k < (kgi + 1) * kr; k++)
      for (int w = 0; w < G.words; w++)
        o[(size_t)k * G.words + w] =
            pbits_draw(d0 + (unsigned long long)k * G.words + w, (uint32_t)sid, (uint32_t)(sid >> 32), seed_lo, seed_hi);
    return;
  }
  for (int k = kgi * kr; k < (kgi + 1) * kr; k++)
    for (int w = 0; w < G.words; w++) {
      const unsigned long long d = d0 + (unsigned long long)k * G.words + w, cc = d >> 2;
      uint32_t x0 = (uint32_t)cc, x1 = (uint32_t)(cc >> 32), x2 = (uint32_t)sid, x3 = (uint32_t)(sid >> 32);
      philox10(x0, x1, x2, x3, seed_lo, seed_hi);
      const int e = (int)(d & 3);
      o[(size_t)k * G.words + w] = (e == 0 ? x0 : e == 1 ? x1 : e == 2 ? x2 : x3) & 0x7FFFFFu;
    }
}

__global__ void k_pack_edges(Geo G, int X, const uint32_t* __restrict__ spins, uint32_t* edge) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= G.n_sim * 2 * G.Wp) return;
  const int j = i % G.Wp, which = (i / G.Wp) % 2, s = i / (2 * G.Wp);
  const int br = which == 0 ? G.ghost : G.ghost + G.rows - 1;
  edge[i] = spins[row_off(G, s, X, br) + j];
}

__global__ void k_unpack_ghosts(Geo G, int X, const uint32_t* __restrict__ ghost_rows, uint32_t* spins) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= G.n_sim * 2 * G.Wp) return;
  const int j = i % G.Wp, which = (i / G.Wp) % 2, s = i / (2 * G.Wp);
  const int br = which == 0 ? 0 : G.R - 1;
  spins[row_off(G, s, X, br) + j] = ghost_rows[i];
}


// Chunks per warp of the conversion kernels: the largest of 8, 4, 2, 1 that
// divides a replica's chunk count, so a warp never spans two replicas.
int conv_cpw(const Geo& G, int cap) {
  const long long per = (long long)G.rows * G.nch;
  for (int c = cap; c > 1; c >>= 1)
    if (per % c == 0) return c;
  return 1;
}

int check_conv(const Geo& G) {
  if (32LL * G.n_sim * G.rows * G.nch >= (1LL << 31)) return fail(MSB_ERR_UNSUPPORTED, "too many chunks for one launch");
  return MSB_OK;
}

template <int CPW>
void launch_from_linear(const Geo& G, const uint32_t* lin, uint32_t* spins, cudaStream_t st) {
  const unsigned nw = (unsigned)((long long)G.n_sim * G.rows * G.nch / CPW);
  k_from_linear<CPW><<<blocks_for(32LL * nw, kConvThreads), kConvThreads, 0, st>>>(G, lin, spins, nw);
}

template <int CPW, bool LIN, bool OBS>
void launch_export(const Geo& G, const uint32_t* spins, uint32_t* lin, long long* ups, long long* unsat,
                          cudaStream_t st) {
  const unsigned nw = (unsigned)((long long)G.n_sim * G.rows * G.nch / CPW);
  k_export<CPW, LIN, OBS><<<blocks_for(32LL * nw, kConvThreads), kConvThreads, 0, st>>>(G, spins, lin, ups, unsat,
                                                                                        nw);
}

template <bool LIN, bool OBS>
void export_cpw(const Geo& G, const uint32_t* spins, uint32_t* lin, long long* ups, long long* unsat,
                       cudaStream_t st) {
  switch (conv_cpw(G, 4)) {  // 4 beats 8 with the observables (registers: 40 vs 80)
    case 4: launch_export<4, LIN, OBS>(G, spins, lin, ups, unsat, st); break;
    case 2: launch_export<2, LIN, OBS>(G, spins, lin, ups, unsat, st); break;
    default: launch_export<1, LIN, OBS>(G, spins, lin, ups, unsat, st); break;
  }
}


}  // namespace
}  // namespace msbk

using namespace msbk;

extern "C" {

int msb_rng_init(const msb_geom* g, uint64_t seed, int32_t kg, uint64_t block, int32_t colour,
                 const uint32_t* pow_tables, uint32_t* states, void* stream) {
  if (int r = check_geom(g)) return r;
  if (kg != 1 && kg != 2 && kg != 4 && kg != 8 && kg != 16) return fail(MSB_ERR_ARG, "kg must be 1, 2, 4, 8 or 16");
  if (colour < -1 || colour > 1) return fail(MSB_ERR_ARG, "colour must be -1 (both), 0 or 1");
  if (!pow_tables || !states) return fail(MSB_ERR_ARG, "null buffer");
  const Geo G = make_geo(g);
  const long long np = (long long)g->n_sim * g->rows * kg;
  const long long n = (colour < 0 ? 2 : 1) * np;
  k_rng_init<<<blocks_for(n, 128), 128, 0, as_stream(stream)>>>(
      G, seed, kg, 16 / kg, np, block, colour, reinterpret_cast<const uint4*>(pow_tables), states);
  CUDA_TRY(cudaGetLastError());
  return MSB_OK;
}

int msb_init_random(const msb_geom* g, uint64_t seed, const uint32_t* pow_tables, uint64_t* scratch,
                    uint32_t* spins, void* stream) {
  if (int r = check_geom(g)) return r;
  if (!pow_tables || !scratch || !spins) return fail(MSB_ERR_ARG, "null buffer");
  const Geo G = make_geo(g);
  const long long wps = (long long)g->rows * g->n / 64;
  const long long pieces = (wps + kInitPiece - 1) / kInitPiece * g->n_sim;
  k_init_linear<<<blocks_for(pieces, 64), 64, 0, as_stream(stream)>>>(
      G, seed, wps, reinterpret_cast<const uint4*>(pow_tables), reinterpret_cast<unsigned long long*>(scratch));
  CUDA_TRY(cudaGetLastError());
  if (int r = msb_init_const(g, 0, spins, stream)) return r;
  return msb_from_linear(g, scratch, spins, stream);
}

int msb_init_const(const msb_geom* g, int32_t up, uint32_t* spins, void* stream) {
  if (int r = check_geom(g)) return r;
  if (!spins) return fail(MSB_ERR_ARG, "null buffer");
  const Geo G = make_geo(g);
  const long long total = (long long)G.n_sim * 2 * G.R * G.Wp;
  k_init_const<<<blocks_for(total, 256), 256, 0, as_stream(stream)>>>(G, up ? 1u : 0u, spins);
  CUDA_TRY(cudaGetLastError());
  return MSB_OK;
}

int msb_from_linear(const msb_geom* g, const uint64_t* lin, uint32_t* spins, void* stream) {
  if (int r = check_geom(g)) return r;
  if (!lin || !spins) return fail(MSB_ERR_ARG, "null buffer");
  const Geo G = make_geo(g);
  if (int r = check_conv(G)) return r;
  const uint32_t* l = reinterpret_cast<const uint32_t*>(lin);
  switch (conv_cpw(G, 8)) {
    case 8: launch_from_linear<8>(G, l, spins, as_stream(stream)); break;
    case 4: launch_from_linear<4>(G, l, spins, as_stream(stream)); break;
    case 2: launch_from_linear<2>(G, l, spins, as_stream(stream)); break;
    default: launch_from_linear<1>(G, l, spins, as_stream(stream)); break;
  }
  CUDA_TRY(cudaGetLastError());
  return MSB_OK;
}

int msb_export(const msb_geom* g, const uint32_t* spins, uint64_t* lin, int64_t* ups, int64_t* unsat,
               void* stream) {
  if (int r = check_geom(g)) return r;
  if (!spins) return fail(MSB_ERR_ARG, "null buffer");
  if ((ups == nullptr) != (unsat == nullptr)) return fail(MSB_ERR_ARG, "ups and unsat go together");
  const Geo G = make_geo(g);
  if (int r = check_conv(G)) return r;
  uint32_t* l = reinterpret_cast<uint32_t*>(lin);
  long long *u = reinterpret_cast<long long*>(ups), *b = reinterpret_cast<long long*>(unsat);
  const cudaStream_t st = as_stream(stream);
  if (lin && ups) export_cpw<true, true>(G, spins, l, u, b, st);
  else if (lin) export_cpw<true, false>(G, spins, l, u, b, st);
  else if (ups) export_cpw<false, true>(G, spins, l, u, b, st);
  else return MSB_OK;
  CUDA_TRY(cudaGetLastError());
  return MSB_OK;
}

int msb_to_linear(const msb_geom* g, const uint32_t* spins, uint64_t* lin, void* stream) {
  if (!lin) return fail(MSB_ERR_ARG, "null buffer");
  return msb_export(g, spins, lin, nullptr, nullptr, stream);
}

int msb_to_ref16(const msb_geom* g, const uint32_t* spins, uint16_t* state, void* stream) {
  if (int r = check_geom(g)) return r;
  if (g->ghost) return fail(MSB_ERR_UNSUPPORTED, "ref16 interop needs a whole lattice");
  if (!spins || !state) return fail(MSB_ERR_ARG, "null buffer");
  const Geo G = make_geo(g);
  const long long total = (long long)G.n_sim * 8 * (G.m / 4 + 2) * (G.words + 2);
  k_to_ref16<<<blocks_for(total, 256), 256, 0, as_stream(stream)>>>(G, spins, state);
  CUDA_TRY(cudaGetLastError());
  return MSB_OK;
}

int msb_from_ref16(const msb_geom* g, const uint16_t* state, uint32_t* spins, void* stream) {
  if (int r = check_geom(g)) return r;
  if (g->ghost) return fail(MSB_ERR_UNSUPPORTED, "ref16 interop needs a whole lattice");
  if (!spins || !state) return fail(MSB_ERR_ARG, "null buffer");
  const Geo G = make_geo(g);
  const long long total = (long long)G.n_sim * 2 * G.m * G.Wp;
  k_from_ref16<<<blocks_for(total, 256), 256, 0, as_stream(stream)>>>(G, state, spins);
  CUDA_TRY(cudaGetLastError());
  return MSB_OK;
}

int msb_observe(const msb_geom* g, const uint32_t* spins, int64_t* ups, int64_t* unsat, void* stream) {
  if (!ups || !unsat) return fail(MSB_ERR_ARG, "null buffer");
  return msb_export(g, spins, nullptr, ups, unsat, stream);
}

int msb_draws(const msb_geom* g, const msb_sweep_params* p, int32_t phase, const uint32_t* states, uint32_t* out,
              void* stream) {
  if (int r = check_geom(g)) return r;
  if (g->ghost) return fail(MSB_ERR_UNSUPPORTED, "draw export needs a whole lattice");
  if (!p) return fail(MSB_ERR_ARG, "null parameters");
  const int kg = p->kg;
  if (kg != 1 && kg != 2 && kg != 4 && kg != 8 && kg != 16) return fail(MSB_ERR_ARG, "kg must be 1, 2, 4, 8 or 16");
  if (phase != 0 && phase != 1) return fail(MSB_ERR_ARG, "phase must be 0 or 1");
  if (!out || (p->rng == MSB_RNG_XOSHIRO && !states)) return fail(MSB_ERR_ARG, "null buffer");
  const Geo G = make_geo(g);
  const long long np = (long long)g->n_sim * g->rows * kg;
  k_draws<<<blocks_for(np, 128), 128, 0, as_stream(stream)>>>(G, phase, kg, 16 / kg, np, states,
                                                              p->rng == MSB_RNG_PHILOX ? 1 : p->rng == MSB_RNG_PHILOX_BITS ? 2 : 0, (uint32_t)p->seed,
                                                              (uint32_t)(p->seed >> 32), p->block, out);
  CUDA_TRY(cudaGetLastError());
  return MSB_OK;
}

int msb_pack_edges(const msb_geom* g, int32_t colour, const uint32_t* spins, uint32_t* edge, void* stream) {
  if (int r = check_geom(g)) return r;
  if (!g->ghost) return fail(MSB_ERR_ARG, "edge exchange needs a slab buffer (ghost = 1)");
  if (!spins || !edge) return fail(MSB_ERR_ARG, "null buffer");
  const Geo G = make_geo(g);
  k_pack_edges<<<blocks_for((long long)G.n_sim * 2 * G.Wp, 256), 256, 0, as_stream(stream)>>>(G, colour & 1, spins, edge);
  CUDA_TRY(cudaGetLastError());
  return MSB_OK;
}

int msb_unpack_ghosts(const msb_geom* g, int32_t colour, const uint32_t* ghost_rows, uint32_t* spins, void* stream) {
  if (int r = check_geom(g)) return r;
  if (!g->ghost) return fail(MSB_ERR_ARG, "ghost rows need a slab buffer (ghost = 1)");
  if (!spins || !ghost_rows) return fail(MSB_ERR_ARG, "null buffer");
  const Geo G = make_geo(g);
  k_unpack_ghosts<<<blocks_for((long long)G.n_sim * 2 * G.Wp, 256), 256, 0, as_stream(stream)>>>(G, colour & 1,
                                                                                                  ghost_rows, spins);
  CUDA_TRY(cudaGetLastError());
  return MSB_OK;
}

}  // extern "C"
