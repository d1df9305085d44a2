// libmsb200 hot path: accept-plane generation (the RNG half of a sweep), the
// per-colour flip pass, the persistent fused sweep kernel and their ABI
// entry points (msb_rng_planes / msb_flip / msb_phase / msb_sweep).
#include "msb_sweep.cuh"

namespace msbk {
namespace {

// ---------------------------------------------------------------------------
// device: accept-plane generation (the RNG half of a sweep)
// ---------------------------------------------------------------------------
//
// The reference's draws never depend on the spins (engine.py:336-341 draws a
// whole block before any flip), so a sweep splits into
//   (1) k_rng_planes: every stream piece generates its draws and reduces each
//       to NP accept bits (u23 < K_p), accumulated per (k, chunk) straight
//       into planes[X][p][s][lr][ch*16 + t(k)] (same layout as the spins);
//   (2) k_flip (per colour): bit-sliced neighbour classes select the plane.
// (1) is INT-pipe bound and state independent; (2) is a light pass over L2.

struct RngArgs {
  Geo G;
  uint32_t* states;
  const uint32_t* thr9;
  const uint4* jump;
  const uint32_t* ext;
  uint32_t* planes;
  unsigned* work;
  long long npieces;
  int colour0, ncol, kg, kr, np, kg_shift;
  FastDiv pieces_div;
  uint32_t seed_lo, seed_hi;  // Philox key
  unsigned long long block0;  // Philox: stream block of colour0's phase
  PhiloxKeys pk;              // Philox round keys
};

// static (interleaved across CTAs), later ones come from work[0].
template <int NPMAX, int SRC, bool FULL>
__device__ __forceinline__ void rng_produce(const RngArgs& a, const uint4* __restrict__ jt, int role_warp,
                                            int role_warps) {
  // FULL: n/32 is a multiple of 32, so every chunk holds 32 draws
  constexpr bool EXT = SRC == kSrcExt;
  constexpr bool XO = SRC == kSrcXoshiro;
  const Geo& G = a.G;
  const int np = NPMAX == 2 ? 2 : a.np;
  const int lane = threadIdx.x & 31;
  const long long total = a.npieces * a.ncol;
  const long long units = (total + 31) / 32;
  const size_t pstride = (size_t)G.n_sim * G.rows * G.Wp;
  const long long nwarps = (long long)role_warps * gridDim.x;
  long long u = (long long)role_warp * gridDim.x + blockIdx.x;
#ifdef MSB_TRACE
  unsigned long long done_units = 0;
#endif
  for (;;) {
    if (u >= units) break;
#ifdef MSB_TRACE
    done_units++;
#endif
    const long long gi = u * 32 + lane;
    if (gi < total) {
    const unsigned xi = a.pieces_div.div((unsigned)gi);
    const int X = a.colour0 + (int)xi;
    const long long gp = gi - (long long)xi * a.npieces;
    const unsigned gr = (unsigned)gp >> a.kg_shift;
    const int kgi = (int)(gp - ((long long)gr << a.kg_shift));
    const int s = (int)G.rows_div.div(gr), lr = (int)(gr - (unsigned)s * G.rows);
    uint32_t key[NPMAX];
#pragma unroll
    for (int p = 0; p < NPMAX; p++) key[p] = p < np ? a.thr9[p * G.n_sim + s] : 0u;
    uint32_t* out = a.planes + plane_off(G, np, X, 0, s, lr);
    XState st;
    const uint32_t* ext = nullptr;
    uint32_t* sp = a.states + (size_t)X * 8 * a.npieces;
    // jump bookkeeping: the piece's start state, consumed 4 bits at a time
    uint32_t jw0 = 0, jw1 = 0, jw2 = 0, jw3 = 0, jw4 = 0, jw5 = 0, jw6 = 0, jw7 = 0;
    uint32_t r0 = 0, r1 = 0, r2 = 0, r3 = 0, r4 = 0, r5 = 0, r6 = 0, r7 = 0;
    int nib = 0;
    uint32_t ps0 = 0, ps1 = 0;              // Philox: stream id
    unsigned long long pd0 = 0;             // Philox: draw index of this piece's first draw
    if (XO) {
      load_state(st, sp, a.npieces, gp);
      jw0 = st.a0; jw1 = st.a1; jw2 = st.b0; jw3 = st.b1; jw4 = st.c0; jw5 = st.c1; jw6 = st.d0; jw7 = st.d1;
    } else {
      const RowStream rsd = row_stream(G.m, G.row0 + lr, X);
      if (EXT) {
        ext = a.ext + ((((size_t)s * (G.m / 4) + rsd.gamma - 1) * 4 + rsd.q) * 16) * G.words;
      } else {
        const unsigned long long sid =
            ((unsigned long long)G.sim_offset + (unsigned long long)s) * (unsigned long long)(G.m / 4) +
            (unsigned long long)(rsd.gamma - 1);
        ps0 = (uint32_t)sid;
        ps1 = (uint32_t)(sid >> 32);
        const unsigned long long n = (unsigned long long)G.n;
        pd0 = (a.block0 + (unsigned long long)(X - a.colour0)) * 2 * n + (unsigned long long)rsd.q * (n / 2);
      }
    }
    for (int kk = 0; kk < a.kr; kk++) {
      const int k = kgi * a.kr + kk;
      const int t = t_of_k(k);
      uint32_t* outk = out + t;
      if (FULL && XO) {
        // fast path: whole chunks, reverse + invert straight into the plane words
        for (int ch = 0; ch < G.nch; ch++) {
          uint32_t acc0 = 0, acc1 = 0;
#pragma unroll kChunkUnroll
          for (int i = 0; i < 32; i++) {
            const uint32_t h9 = xstep(st) << 9;
            acc_reject(acc0, h9, key[0]);
            if (np > 1) acc_reject(acc1, h9, key[NPMAX > 1 ? 1 : 0]);
          }
#ifdef MSB_TRACE_NOSTORE
          if ((acc0 ^ acc1) == 0x9E3779B9u) outk[ch * 16] = acc0;  // timing experiment only
#else
          outk[ch * 16] = ~__brev(acc0);
          if (np > 1) outk[pstride + ch * 16] = ~__brev(acc1);
#endif
        }
      } else
      for (int ch = 0; ch < G.nch; ch++) {
        const int L = FULL ? 32 : chunk_bits(G, ch);
        uint32_t acc[NPMAX];
#pragma unroll
        for (int p = 0; p < NPMAX; p++) acc[p] = 0;
        if (SRC == kSrcPbits) {  // accept bits straight from the bit planes
          pbits_chunk<NPMAX>(pd0 + (unsigned long long)k * G.words + 32 * ch, L, pbits_lane(ps0, ps1), a.pk, key, np,
                             acc);
#pragma unroll
          for (int p = 0; p < NPMAX; p++)
            if (p < np) out[p * pstride + ch * 16 + t] = acc[p];
          continue;
        } else if (SRC == kSrcPhilox) {
          const unsigned long long d0 = pd0 + (unsigned long long)k * G.words + 32 * ch;
          if ((d0 & 3) == 0 && (L & 3) == 0) {
            for (int i = 0; i < L; i += 4) {
              const unsigned long long c = (d0 + i) >> 2;
              uint32_t x0 = (uint32_t)c, x1 = (uint32_t)(c >> 32), x2 = ps0, x3 = ps1;
              philox10k(x0, x1, x2, x3, a.pk);
              const uint32_t xs[4] = {x0, x1, x2, x3};
#pragma unroll
              for (int j = 0; j < 4; j++) {
                const uint32_t h9 = xs[j] << 9;
#pragma unroll
                for (int p = 0; p < NPMAX; p++)
                  if (p < np) acc_reject(acc[p], h9, key[p]);
              }
            }
          } else {  // draw groups straddle the piece: one block per draw
            for (int i = 0; i < L; i++) {
              const unsigned long long d = d0 + i, c = d >> 2;
              uint32_t x0 = (uint32_t)c, x1 = (uint32_t)(c >> 32), x2 = ps0, x3 = ps1;
              philox10k(x0, x1, x2, x3, a.pk);
              const int e = (int)(d & 3);
              const uint32_t h9 = (e == 0 ? x0 : e == 1 ? x1 : e == 2 ? x2 : x3) << 9;
#pragma unroll
              for (int p = 0; p < NPMAX; p++)
                if (p < np) acc_reject(acc[p], h9, key[p]);
            }
          }
        } else if (!EXT) {
          if (L == 32) {
#pragma unroll kChunkUnroll
            for (int i = 0; i < 32; i++) {
              const uint32_t h9 = xstep(st) << 9;
#pragma unroll
              for (int p = 0; p < NPMAX; p++)
                if (p < np) acc_reject(acc[p], h9, key[p]);
            }
            // full chunk: reverse + invert straight into the plane words
#pragma unroll
            for (int p = 0; p < NPMAX; p++)
              if (p < np) outk[p * pstride + ch * 16] = ~__brev(acc[p]);
            continue;
          } else {
            for (int i = 0; i < L; i++) {
              const uint32_t h9 = xstep(st) << 9;
#pragma unroll
              for (int p = 0; p < NPMAX; p++)
                if (p < np) acc_reject(acc[p], h9, key[p]);
            }
          }
        } else {
          const uint32_t* e = ext + (size_t)k * G.words + 32 * ch;
          for (int i = 0; i < L; i++) {
            const uint32_t h9 = e[i] << 9;
#pragma unroll
            for (int p = 0; p < NPMAX; p++)
              if (p < np) acc_reject(acc[p], h9, key[p]);
          }
        }
        // acc holds REJECT bits, newest draw in bit 0: reverse and invert
#pragma unroll
        for (int p = 0; p < NPMAX; p++)
          if (p < np) out[p * pstride + ch * 16 + t] = (~__brev(acc[p])) >> (32 - L);
      }
      // jump lookups: one 32-bit state word (8 nibbles, 64 lookups in all)
      // after every second k-segment when kr == 16, else 8/kr words per segment
#ifdef MSB_TRACE_NOJUMP
      if (false) {  // timing experiment only: no jump lookups
#else
      if (XO) {
#endif
        const int nwords = a.kr >= 16 ? (kk & 1) : 8 / a.kr;
        for (int wcount = 0; wcount < nwords; wcount++) {
          // entry (position nib+j, value v) lives at byte (nib+j)*512 + v*32
          const char* e = reinterpret_cast<const char*>(jt) + nib * 512;
#pragma unroll
          for (int j = 0; j < 8; j += 2) {
            const uint32_t oa = j == 0 ? ((jw0 << 5) & 0x1E0u) : ((jw0 >> (4 * j - 5)) & 0x1E0u);
            const uint32_t ob = j == 0 ? ((jw0 << 1) & 0x1E0u) : ((jw0 >> (4 * j - 1)) & 0x1E0u);
            const uint4* ea = reinterpret_cast<const uint4*>(e + j * 512 + oa);
            const uint4* eb = reinterpret_cast<const uint4*>(e + (j + 1) * 512 + ob);
            const uint4 la = ea[0], ha = ea[1], lb = eb[0], hb = eb[1];
            r0 = xor3(r0, la.x, lb.x); r1 = xor3(r1, la.y, lb.y); r2 = xor3(r2, la.z, lb.z); r3 = xor3(r3, la.w, lb.w);
            r4 = xor3(r4, ha.x, hb.x); r5 = xor3(r5, ha.y, hb.y); r6 = xor3(r6, ha.z, hb.z); r7 = xor3(r7, ha.w, hb.w);
          }
          nib += 8;
          jw0 = jw1; jw1 = jw2; jw2 = jw3; jw3 = jw4; jw4 = jw5; jw5 = jw6; jw6 = jw7;
        }
      }
    }
    if (XO) {
      XState nx;
      nx.a0 = r0; nx.a1 = r1; nx.b0 = r2; nx.b1 = r3; nx.c0 = r4; nx.c1 = r5; nx.d0 = r6; nx.d1 = r7;
      store_state(nx, sp, a.npieces, gp);  // next sweep's start
    }
    }
    long long nu = 0;
    if (lane == 0) nu = nwarps + (long long)atomicAdd(a.work, 1u);
    u = __shfl_sync(0xFFFFFFFFu, nu, 0);
  }
#ifdef MSB_TRACE
  unsigned smid;
  asm("mov.u32 %0, %smid;" : "=r"(smid));
  MSB_TRACE_PUT(3, smid | (done_units << 32));
#endif
}

template <int NPMAX, int SRC, bool FULL>
__global__ void __launch_bounds__(kRngThreads, 1) k_rng_planes(const RngArgs a) {
  extern __shared__ uint4 jt[];  // nibble table of A^(4n), 32 KiB
#ifdef MSB_TRACE
  MSB_TRACE_PUT(0, gtimer());
  MSB_TRACE_PUT(4, clock64());
#endif
  if (SRC == kSrcXoshiro) {
    for (int i = threadIdx.x; i < kJumpWords / 4; i += blockDim.x) jt[i] = a.jump[i];
    __syncthreads();
  }
#ifdef MSB_TRACE
  MSB_TRACE_PUT(1, gtimer());
#endif
  rng_produce<NPMAX, SRC, FULL>(a, jt, threadIdx.x >> 5, blockDim.x >> 5);
#ifdef MSB_TRACE
  MSB_TRACE_PUT(2, gtimer());
  MSB_TRACE_PUT(5, clock64());
#endif
  finish_warp(a.work, gridDim.x * (blockDim.x >> 5));
}



// ---------------------------------------------------------------------------
// device: fused sweep -- flips of sweep k overlapped with the planes of k+1
// ---------------------------------------------------------------------------
//
// Cooperative persistent kernel, one 1024-thread CTA per SM.  Warps
// [0, kProducerWarps) generate sweep k+1's accept planes (rng_produce) into
// one buffer; the other warps flip sweep k from the other buffer: red quads,
// a grid barrier among flip warps, then blue quads.  The flip pass is
// latency-bound and the RNG ALU-bound, so sharing the SMs hides the flips.
// flip warps per CTA: FlipArgs::cwarps (the rest produce planes)


template <int NPMAX, int SRC, bool FULL>
__global__ void __launch_bounds__(kRngThreads, 1) k_sweep_fused(const RngArgs ra, const FlipArgs fa) {
  const int kFlipWarps = fa.cwarps;
  const int kProducerWarps = (kRngThreads >> 5) - kFlipWarps;
  extern __shared__ uint4 jt[];
#ifdef MSB_TRACE
  MSB_TRACE_PUT(0, gtimer());
  MSB_TRACE_PUT(4, clock64());
#endif
  if (SRC == kSrcXoshiro) {
    for (int i = threadIdx.x; i < kJumpWords / 4; i += blockDim.x) jt[i] = ra.jump[i];
    __syncthreads();
  }
#ifdef MSB_TRACE
  MSB_TRACE_PUT(1, gtimer());
#endif
  const int warp = threadIdx.x >> 5;
  const unsigned total_warps = gridDim.x * (blockDim.x >> 5);
  if (warp < kProducerWarps) {
    rng_produce<NPMAX, SRC, FULL>(ra, jt, warp, kProducerWarps);
  } else {
    const unsigned total = (unsigned)fa.G.n_sim * (unsigned)fa.G.rows * ((unsigned)fa.G.Wp >> 2);  // quads
    const unsigned nc = gridDim.x * kFlipWarps;
    const unsigned cw = (warp - kProducerWarps) * gridDim.x + blockIdx.x;
    const unsigned per = ((total + nc - 1) / nc + 31) & ~31u;  // quads per consumer warp
    const unsigned lo = min(total, cw * per), hi = min(total, lo + per);
    const unsigned i0 = lo + (threadIdx.x & 31);
    unsigned cnt = 0;
    for (int X = 0; X < 2; X++) {
      if (X == 0) {
        cnt += flip_run<false>(fa, i0, hi, 0);
      } else {
        cnt += flip_run<true>(fa, i0, hi, 1);
      }
      if (X == 0) {  // grid barrier among the flip warps
        __syncwarp();
        if ((threadIdx.x & 31) == 0) {
          __threadfence();
          atomicAdd(ra.work + 1, 1u);
          const unsigned need = gridDim.x * kFlipWarps;
          while (ld_acquire(ra.work + 1) < need) __nanosleep(1000);
        }
        __syncwarp();
        __threadfence();
#ifdef MSB_TRACE
        MSB_TRACE_PUT(6, gtimer());
#endif
      }
    }
    add_flips(fa.flips, cnt);
#ifdef MSB_TRACE
    unsigned smid;
    asm("mov.u32 %0, %smid;" : "=r"(smid));
    MSB_TRACE_PUT(3, smid | (1ull << 63));
#endif
  }
#ifdef MSB_TRACE
  MSB_TRACE_PUT(2, gtimer());
  MSB_TRACE_PUT(5, clock64());
#endif
  finish_warp(ra.work, total_warps);
}



void fill_rng_args(RngArgs& a, const msb_geom* g, const msb_sweep_params* p, int colour, uint32_t* states,
                   const uint32_t* ext, uint32_t* planes) {
  a.G = make_geo(g);
  a.states = states;
  a.thr9 = p->thr9;
  a.jump = reinterpret_cast<const uint4*>(p->jump);
  a.ext = ext;
  a.planes = planes;
  a.kg = p->kg;
  a.kr = 16 / p->kg;
  a.npieces = (long long)g->n_sim * g->rows * p->kg;
  a.np = p->n_planes;
  a.colour0 = colour < 0 ? 0 : colour;
  a.ncol = colour < 0 ? 2 : 1;
  a.work = p->work;
  a.kg_shift = p->kg == 1 ? 0 : p->kg == 2 ? 1 : p->kg == 4 ? 2 : p->kg == 8 ? 3 : 4;
  a.pieces_div.init((uint32_t)a.npieces);
  a.seed_lo = (uint32_t)p->seed;
  a.seed_hi = (uint32_t)(p->seed >> 32);
  a.block0 = p->block;
  a.pk = philox_keys(p->seed);
}


int rng_planes(const msb_geom* g, const msb_sweep_params* p, int colour, uint32_t* states, const uint32_t* ext,
               uint32_t* planes, cudaStream_t st) {
  if (2LL * g->n_sim * g->rows * p->kg >= (1LL << 31)) return fail(MSB_ERR_UNSUPPORTED, "too many stream pieces");
  RngArgs a;
  fill_rng_args(a, g, p, colour, states, ext, planes);
  int dev = 0, sms = 148;
  CUDA_TRY(cudaGetDevice(&dev));
  CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const long long units = (a.npieces * a.ncol + 31) / 32;
  const long long per_cta = kRngThreads / 32;
  (void)per_cta;
  const unsigned grid = (unsigned)std::max(1LL, std::min<long long>(sms, units));
  const size_t smem = (ext || p->rng != MSB_RNG_XOSHIRO) ? 0 : (size_t)kJumpWords * 4;
#define MSB_LAUNCH_RNG(NP, SRC, FULL)                                         \
  do {                                                                        \
    static std::once_flag o;                                                  \
    static cudaError_t e;                                                     \
    if (int r = set_smem_attr(k_rng_planes<NP, SRC, FULL>, o, e)) return r;   \
    k_rng_planes<NP, SRC, FULL><<<grid, kRngThreads, smem, st>>>(a);          \
  } while (0)
  const int src = ext ? kSrcExt
                      : (p->rng == MSB_RNG_PHILOX ? kSrcPhilox
                                                  : (p->rng == MSB_RNG_PHILOX_BITS ? kSrcPbits : kSrcXoshiro));
  const bool full = (a.G.words % 32) == 0;
  if (p->mode != MSB_MODE_GENERIC) {
    if (src == kSrcExt) MSB_LAUNCH_RNG(2, kSrcExt, false);
    else if (src == kSrcPhilox) MSB_LAUNCH_RNG(2, kSrcPhilox, false);
    else if (src == kSrcPbits) MSB_LAUNCH_RNG(2, kSrcPbits, false);
    else if (full) MSB_LAUNCH_RNG(2, kSrcXoshiro, true);
    else MSB_LAUNCH_RNG(2, kSrcXoshiro, false);
  } else {
    if (src == kSrcExt) MSB_LAUNCH_RNG(MSB_MAX_PLANES, kSrcExt, false);
    else if (src == kSrcPhilox) MSB_LAUNCH_RNG(MSB_MAX_PLANES, kSrcPhilox, false);
    else if (src == kSrcPbits) MSB_LAUNCH_RNG(MSB_MAX_PLANES, kSrcPbits, false);
    else MSB_LAUNCH_RNG(MSB_MAX_PLANES, kSrcXoshiro, false);
  }
#undef MSB_LAUNCH_RNG
  CUDA_TRY(cudaGetLastError());
  return MSB_OK;
}



// flips of the sweep whose planes are in `cur` + planes of the next sweep
// into `next`, one cooperative launch (FERRO/ANTI whole lattices).
int fused_sweep(const msb_geom* g, const msb_sweep_params* p, uint32_t* spins, uint32_t* states, const uint32_t* cur,
                uint32_t* next, uint64_t* flips, cudaStream_t st) {
  if (int r = check_flip_extent(g, p->n_planes)) return r;
  RngArgs ra;
  fill_rng_args(ra, g, p, -1, states, nullptr, next);
  FlipArgs fa;
  fill_flip_args(fa, g, p, 0, spins, cur, flips);
  fa.cwarps = flip_warps_for((2LL * g->n_sim * g->rows * p->kg + 31) / 32);
  int dev = 0, sms = 148;
  CUDA_TRY(cudaGetDevice(&dev));
  CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const bool philox = p->rng == MSB_RNG_PHILOX, pbits = p->rng == MSB_RNG_PHILOX_BITS;
  const bool full = (fa.G.words % 32) == 0;
  static std::once_flag o, o2, o3, o4;
  static cudaError_t e, e2, e3, e4;
  if (int r = set_smem_attr(k_sweep_fused<2, kSrcXoshiro, false>, o, e)) return r;
  if (int r = set_smem_attr(k_sweep_fused<2, kSrcPhilox, false>, o2, e2)) return r;
  if (int r = set_smem_attr(k_sweep_fused<2, kSrcXoshiro, true>, o3, e3)) return r;
  if (int r = set_smem_attr(k_sweep_fused<2, kSrcPbits, false>, o4, e4)) return r;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)sms);
  cfg.blockDim = dim3(kRngThreads);
  cfg.dynamicSmemBytes = (philox || pbits) ? 0 : (size_t)kJumpWords * 4;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (philox) CUDA_TRY(cudaLaunchKernelEx(&cfg, k_sweep_fused<2, kSrcPhilox, false>, ra, fa));
  else if (pbits) CUDA_TRY(cudaLaunchKernelEx(&cfg, k_sweep_fused<2, kSrcPbits, false>, ra, fa));
  else if (full) CUDA_TRY(cudaLaunchKernelEx(&cfg, k_sweep_fused<2, kSrcXoshiro, true>, ra, fa));
  else CUDA_TRY(cudaLaunchKernelEx(&cfg, k_sweep_fused<2, kSrcXoshiro, false>, ra, fa));
  return MSB_OK;
}
}  // namespace
}  // namespace msbk

using namespace msbk;

extern "C" {

#ifdef MSB_TRACE
int msb_debug_trace(uint64_t* host_out, int32_t n) {
  if (n > kTraceWarps * 8) n = kTraceWarps * 8;
  CUDA_TRY(cudaDeviceSynchronize());
  CUDA_TRY(cudaMemcpyFromSymbol(host_out, g_trace, (size_t)n * 8));
  return MSB_OK;
}
#endif

int64_t msb_plane_words(const msb_geom* g, int32_t n_planes) {
  if (check_geom(g)) return -1;
  if (n_planes < 0 || n_planes > MSB_MAX_PLANES) return -1;
  const Geo G = make_geo(g);
  return 2LL * std::max(n_planes, 1) * g->n_sim * g->rows * G.Wp;
}

int msb_rng_planes(const msb_geom* g, const msb_sweep_params* p, int32_t colour, uint32_t* states,
                   const uint32_t* ext_draws, uint32_t* planes, void* stream) {
  if (int r = check_geom(g)) return r;
  if (int r = check_params(p)) return r;
  if (colour < -1 || colour > 1) return fail(MSB_ERR_ARG, "colour must be -1 (both), 0 or 1");
  if (!planes) return fail(MSB_ERR_ARG, "null planes buffer");
  if (ext_draws && (g->ghost || colour < 0)) return fail(MSB_ERR_UNSUPPORTED, "external draws: one colour of a whole lattice");
  if (!ext_draws && p->rng == MSB_RNG_XOSHIRO && (!states || !p->jump))
    return fail(MSB_ERR_ARG, "null RNG state or jump table");
  return rng_planes(g, p, colour, states, ext_draws, planes, as_stream(stream));
}

int msb_flip(const msb_geom* g, const msb_sweep_params* p, int32_t colour, uint32_t* spins, const uint32_t* planes,
             uint64_t* flips, void* stream) {
  if (int r = check_geom(g)) return r;
  if (int r = check_params(p)) return r;
  if (colour != 0 && colour != 1) return fail(MSB_ERR_ARG, "colour must be 0 (red) or 1 (blue)");
  if (!spins || !planes || !flips) return fail(MSB_ERR_ARG, "null buffer");
  return flip(g, p, colour, spins, planes, flips, as_stream(stream));
}

int msb_phase(const msb_geom* g, const msb_sweep_params* p, int32_t phase, uint32_t* spins, uint32_t* states,
              const uint32_t* ext_draws, uint32_t* planes, uint64_t* flips, void* stream) {
  if (phase != 0 && phase != 1) return fail(MSB_ERR_ARG, "phase must be 0 (red) or 1 (blue)");
  if (int r = msb_rng_planes(g, p, phase, states, ext_draws, planes, stream)) return r;
  return msb_flip(g, p, phase, spins, planes, flips, stream);
}

int msb_sweep(const msb_geom* g, const msb_sweep_params* p, uint32_t* spins, uint32_t* states, uint32_t* planes,
              int32_t n_sweeps, int32_t flags, int32_t* cur_io, uint64_t* flips, void* stream) {
  if (int r = check_geom(g)) return r;
  if (int r = check_params(p)) return r;
  if (n_sweeps < 0) return fail(MSB_ERR_ARG, "sweep count must be non-negative");
  if (!spins || !planes || !flips) return fail(MSB_ERR_ARG, "null buffer");
  if (p->rng == MSB_RNG_XOSHIRO && (!states || !p->jump)) return fail(MSB_ERR_ARG, "null RNG state or jump table");
  if (g->ghost) return fail(MSB_ERR_UNSUPPORTED, "msb_sweep runs whole lattices; slabs use the per-phase calls");
  if ((flags & (MSB_SWEEP_AHEAD_IN | MSB_SWEEP_AHEAD_OUT)) && !cur_io)
    return fail(MSB_ERR_ARG, "lookahead flags need cur_io");
  cudaStream_t st = as_stream(stream);
  const int64_t pw = msb_plane_words(g, p->n_planes);
  // p->block: stream block of the red phase of the first sweep whose planes
  // this call generates (Philox); advanced by 2 per generated sweep
  msb_sweep_params q = *p;
  p = &q;
  int cur = (flags & MSB_SWEEP_AHEAD_IN) ? (*cur_io & 1) : 0;
  const bool fused_ok = p->mode != MSB_MODE_GENERIC && !(flags & MSB_SWEEP_SERIAL);
  if (n_sweeps == 0) {
    if ((flags & MSB_SWEEP_AHEAD_OUT) && !(flags & MSB_SWEEP_AHEAD_IN)) {
      if (int r = rng_planes(g, p, -1, states, nullptr, planes + (size_t)cur * pw, st)) return r;
      q.block += 2;
    }
    if (cur_io) *cur_io = cur;
    return MSB_OK;
  }
  if (!(flags & MSB_SWEEP_AHEAD_IN)) {
    if (int r = rng_planes(g, p, -1, states, nullptr, planes + (size_t)cur * pw, st)) return r;
    q.block += 2;
  }
  for (int k = 0; k < n_sweeps; k++) {
    uint32_t* bc = planes + (size_t)cur * pw;
    uint32_t* bn = planes + (size_t)(1 - cur) * pw;
    const bool last = k + 1 == n_sweeps;
    if (last && !(flags & MSB_SWEEP_AHEAD_OUT)) {
      if (int r = flip(g, p, 0, spins, bc, flips, st)) return r;
      if (int r = flip(g, p, 1, spins, bc, flips, st)) return r;
    } else if (fused_ok) {
      if (int r = fused_sweep(g, p, spins, states, bc, bn, flips, st)) return r;
      q.block += 2;
      cur = 1 - cur;
    } else {
      if (int r = flip(g, p, 0, spins, bc, flips, st)) return r;
      if (int r = flip(g, p, 1, spins, bc, flips, st)) return r;
      if (int r = rng_planes(g, p, -1, states, nullptr, bn, st)) return r;
      q.block += 2;
      cur = 1 - cur;
    }
  }
  if (cur_io) *cur_io = cur;
  return MSB_OK;
}

}  // extern "C"
