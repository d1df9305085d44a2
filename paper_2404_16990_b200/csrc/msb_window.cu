// libmsb200 lookahead windows: accept planes for S sweeps per launch.
//
// The reference consumes each cell stream in sweep order: sweep k takes
// draws [4n k, 4n (k+1)) of stream (sim_offset+s)*(m/4)+gamma-1 -- block 2k
// (red) then block 2k+1 (blue), each four quarters of n/2 draws in FLIP_RED /
// FLIP_BLUE order (engine.py:334-343, 57-68).  The per-sweep path
// (msb_sweep.cu) gives each stream piece one quarter (or less) and jumps it
// 4n draws ahead every sweep: one 64-lookup GF(2) jump per n/2 draws.
//
// Here a piece is (window slot j, part p, stream): it runs its stream
// CONTIGUOUSLY through 1/P of sweep j of the window -- P = 1 is the whole
// sweep, 8 quarter-segments in a row -- and jumps S*4n ahead once, to the same
// place in the next window.  With S = 8, P = 1 that is one jump per 32 n
// draws instead of per n/2.  The planes of a window live in one buffer
// [S][2 colours][2 planes][n_sim][m][Wp] (same per-slot layout as the
// per-sweep planes), so the flip pass is unchanged.
//
// k_win is the steady state, one cooperative launch per window: producer
// warps fill the NEXT window's buffer while the consumer warps of every CTA
// flip the S sweeps of the CURRENT one (red, grid barrier, blue, grid
// barrier, ...; band walk or quad walk, msb_sweep.cuh).  Launch, start-up and
// tail are paid once per S sweeps.  Row slabs (msb_halo) additionally push
// their edge rows into the neighbours' ghost rows and handshake every phase.
#include "msb_window.cuh"

using namespace msbk;

extern "C" {


int32_t msb_window_parts(const msb_geom* g, int32_t S) {
  long long np = 0;
  if (check_window(g, S, g && g->ghost ? 8 : 1, &np)) return -1;
  // smallest split giving ~one warp-unit (32 pieces) per producer warp of
  // every SM (148 SMs x 28 warps), as msb_default_kg; slabs need P >= 8
  const long long rows2 = 2LL * g->n_sim * g->rows;  // (replica, colour, row) segments per sweep
  auto pieces = [&](int p) { return (long long)S * rows2 * p / 8; };
  int p = g->ghost ? 8 : 1;
  while (p < 128 && pieces(p) < 118000) p *= 2;
  // Rows being written concurrently stay L2-resident: a piece completes its
  // row's plane words one t-word per k, so ~140k pieces in flight write
  // 140k / max(1, P/8) rows of 8*Wp bytes (P > 8: the P/8 parts of a row run
  // side by side).  Keep that under ~100 MB (measured: cfg4 best at P = 32,
  // the 32768-wide cfg5 rows at P = 32-64; P = 8 cost 9-19%).
  const long long row_bytes = 8LL * make_geo(g).Wp;
  while (p < 128 && 140000LL / std::max(1, p / 8) * row_bytes > (100LL << 20)) p *= 2;
  static const int env_p = [] { const char* e = getenv("MSB_WINDOW_PARTS"); return e ? atoi(e) : 0; }();
  if (env_p > 0 && env_p <= 128 && !(env_p & (env_p - 1)) && (env_p >= 8 || !g->ghost)) p = env_p;  // tuning
  while (p > (g->ghost ? 8 : 1) && pieces(p) >= (1LL << 31)) p >>= 1;
  return p;
}

int msb_default_window(const msb_geom* g, int32_t* S, int32_t* P) {
  if (!S || !P) return fail(MSB_ERR_ARG, "null output");
  long long np = 0;
  if (int r = check_window(g, 1, g && g->ghost ? 8 : 1, &np)) return r;
  // Whole lattices: S = 64 sweeps per window launch (fewer launches, jumps,
  // start-up and tail costs per sweep: cfg2 0.934 -> 0.965 T, cfg3 0.936 ->
  // 0.963 T at S = 32; end to end, one host round trip per 64 sweeps), slabs
  // S = 32; halved while the two window buffers would exceed 8 GiB of planes
  // (cfg3: S = 32, 6.3 GB).
  const long long slot_bytes = 4LL * (long long)slot_words(g);
  int s = g->ghost ? 32 : 64;  // slabs: cfg4 S = 8 0.940, 16 0.955, 32 0.958 T (ring of 8: 0.853, 0.872, 0.877)
  while (s > 1 && 2LL * s * slot_bytes > (8LL << 30)) s >>= 1;
  *S = s;
  *P = msb_window_parts(g, s);
  return MSB_OK;
}

int64_t msb_window_pieces(const msb_geom* g, int32_t S, int32_t P) {
  long long np = 0;
  if (check_window(g, S, P, &np)) return -1;
  return np;
}

int64_t msb_window_words(const msb_geom* g, int32_t S) {
  long long np = 0;
  if (check_window(g, S, g && g->ghost ? 8 : 1, &np)) return -1;
  return (int64_t)S * (int64_t)slot_words(g);
}

int msb_window_init(const msb_geom* g, uint64_t seed, int32_t S, int32_t P, uint64_t block, const uint32_t* pow_tables,
                    uint32_t* states, void* stream) {
  long long np = 0;
  if (int r = check_window(g, S, P, &np)) return r;
  if (!pow_tables || !states) return fail(MSB_ERR_ARG, "null buffer");
  msb_sweep_params p = {};
  p.block = block;
  WinArgs wa;
  fill_win_args(wa, g, &p, S, P, np, states, nullptr);
  k_win_init<<<blocks_for(np, 128), 128, 0, as_stream(stream)>>>(wa, seed,
                                                                 reinterpret_cast<const uint4*>(pow_tables));
  CUDA_TRY(cudaGetLastError());
  return MSB_OK;
}

namespace {
int window_run_any(int rng, int nslabs, const msb_ring_slab* slabs, bool ring, int S, int P, int first, int count,
                   const msb_window_io* io, void* ctx, void* stream) {
  if (rng == MSB_RNG_PHILOX) return window_run_philox(nslabs, slabs, ring, S, P, first, count, io, ctx, stream);
  if (rng == MSB_RNG_PHILOX_BITS) return window_run_pbits(nslabs, slabs, ring, S, P, first, count, io, ctx, stream);
  return window_run_xoshiro(nslabs, slabs, ring, S, P, first, count, io, ctx, stream);
}
}  // namespace

int msb_window_sweep(const msb_geom* g, const msb_sweep_params* p, int32_t S, int32_t P, uint32_t* spins,
                     uint32_t* states, const uint32_t* cur, int32_t first, int32_t count, uint32_t* next,
                     uint64_t* flips, const msb_halo* halo, const msb_window_io* io, void* stream) {
  if (!next && count == 0) {
    WinArgs wa;
    FlipArgs fa;
    HaloArgs ha;
    WinIO wio;
    long long np = 0;
    if (int r = plan_window(g, p, S, P, spins, states, cur, first, count, next, flips, halo, io, wa, fa, ha, wio, np))
      return r;
    if (halo) {  // until the neighbours' pushes into our ghost rows landed
      k_halo_wait<<<1, 32, 0, as_stream(stream)>>>(wa.flags, wa.nslot);
      CUDA_TRY(cudaGetLastError());
    }
    return MSB_OK;
  }
  if (int r = check_params(p)) return r;
  const msb_ring_slab one = {g, p, spins, states, cur, next, flips, halo};
  return window_run_any(p->rng, 1, &one, false, S, P, first, count, io, nullptr, stream);
}

int msb_direct_ok(const msb_geom* g, const msb_sweep_params* p) {
  if (check_geom(g) || check_params(p)) return 0;
  if (p->rng != MSB_RNG_PHILOX_BITS || p->mode == MSB_MODE_GENERIC) return 0;
  const Geo G = make_geo(g);
  if (G.words % 32 != 0 && G.words != 16) return 0;
  FlipArgs fa;
  fill_flip_args(fa, g, p, 0, nullptr, nullptr, nullptr);
  return direct_band(fa, g) ? 1 : 0;
}

int64_t msb_flag_words(const msb_geom* g) {
  if (check_geom(g)) return -1;
  msb_sweep_params p = {};
  p.mode = MSB_MODE_FERRO;
  p.n_planes = 2;
  FlipArgs fa;
  fill_flip_args(fa, g, &p, 0, nullptr, nullptr, nullptr);
  const long long nslot = g_nslot(fa);
  // the direct walk's 2-row bands give the most groups of any band walk
  const long long groups = direct_band(fa, g) ? (long long)fa.band_groups : 0;
  return 1 + 2 * nslot + groups;
}

int msb_direct_sweep(const msb_geom* g, const msb_sweep_params* p, uint32_t* spins, int32_t n_sweeps, uint64_t* flips,
                     const msb_halo* halo, const msb_window_io* io, void* stream) {
  const msb_ring_slab one = {g, p, spins, nullptr, nullptr, nullptr, flips, halo};
  return direct_run(1, &one, false, n_sweeps, io, nullptr, stream);
}

int64_t msb_ring_ctx_bytes(int32_t nslabs) {
  if (nslabs < 1 || nslabs > MSB_RING_MAX) return -1;
  return (int64_t)nslabs * (int64_t)sizeof(SlabCtx);
}

int msb_window_sweep_ring(int32_t nslabs, const msb_ring_slab* slabs, int32_t S, int32_t P, int32_t first,
                          int32_t count, void* ctx, void* stream) {
  if (nslabs < 1 || nslabs > MSB_RING_MAX || !slabs) return fail(MSB_ERR_ARG, "ring of 1..MSB_RING_MAX slabs");
  for (int v = 0; v < nslabs; v++) {
    if (!slabs[v].p) return fail(MSB_ERR_ARG, "null sweep parameters");
    if (slabs[v].p->rng != slabs[0].p->rng) return fail(MSB_ERR_ARG, "ring slabs must share the stream kind");
  }
  if (count == 0) {  // production only: no phases, the slabs need not run together
    for (int v = 0; v < nslabs; v++) {
      const msb_ring_slab& r = slabs[v];
      if (int e = msb_window_sweep(r.g, r.p, S, P, r.spins, r.states, r.cur, first, 0, r.next, r.flips, r.halo,
                                   nullptr, stream))
        return e;
    }
    return MSB_OK;
  }
  if (!ctx) return fail(MSB_ERR_ARG, "null ring context buffer");
  return window_run_any(slabs[0].p->rng, nslabs, slabs, true, S, P, first, count, nullptr, ctx, stream);
}

int msb_direct_sweep_ring(int32_t nslabs, const msb_ring_slab* slabs, int32_t n_sweeps, void* ctx, void* stream) {
  if (nslabs < 1 || nslabs > MSB_RING_MAX || !slabs) return fail(MSB_ERR_ARG, "ring of 1..MSB_RING_MAX slabs");
  if (!ctx) return fail(MSB_ERR_ARG, "null ring context buffer");
  return direct_run(nslabs, slabs, true, n_sweeps, nullptr, ctx, stream);
}

}  // extern "C"
