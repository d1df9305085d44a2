// libmsb200: sm_100a kernels for the bit-packed checkerboard Metropolis hot
// path of the reference `multispin` package (see include/msb200.h for the
// ABI and DESIGN.md for the layout / roofline discussion).
//
// Reference algorithm being reproduced bit-exactly (pkg/src/multispin/...):
//   stream seeding       rng.py:53-82     splitmix64 -> xoshiro256 state
//   xoshiro256++ step    rng.py:93-105
//   23-bit shaping       rng.py:113-115, 180-183
//   draw consumption     engine.py:334-343 (quarter, k = 4i+ii, word)
//   bit gated by draw    engine.py:321-331 (bit 4ii+i of the target word)
//   quarter targets      engine.py:57-68  (FLIP_RED / FLIP_BLUE)
//   Metropolis test      engine.py:78-94, 325-330 (float64 u < table[code])
//   observables          engine.py:372-386
//
// Layout here is NOT the reference's eight folded uint16 arrays: spins are
// split by checkerboard colour into rows of 32 same-colour sites per uint32
// (include/msb200.h).  The fold/moat/halo structure of the WSE mapping is an
// interop format only (msb_to_ref16 / msb_from_ref16).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>

#include "../../include/msb200.h"
#include "gf2_jump.h"

namespace {

constexpr uint64_t kGolden = 0x9E3779B97F4B7C15ULL;
constexpr int kJumpWords = 8192;  // one nibble table = 32 KiB
constexpr uint32_t kKeyAlways = 0xFFFFFFFFu;

thread_local std::string g_last_error;

int fail(int code, const std::string& why) {
  g_last_error = why;
  return code;
}

#define CUDA_TRY(expr)                                                                 \
  do {                                                                                 \
    cudaError_t e_ = (expr);                                                           \
    if (e_ != cudaSuccess) return fail(MSB_ERR_CUDA, std::string(#expr ": ") + cudaGetErrorString(e_)); \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// ---------------------------------------------------------------------------
// device: RNG
// ---------------------------------------------------------------------------

struct XState {
  uint32_t a0, a1, b0, b1, c0, c1, d0, d1;  // s0..s3 as (lo, hi) halves
};

__device__ __forceinline__ uint32_t xor3(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

// One xoshiro256++ step (rng.py:93-105); returns the HIGH 32 bits of the
// output, the only bits the reference shapes into a draw (rng.py:115).
// 64-bit adds are carry chains (IADD3 + IMAD.X), rotations funnel shifts,
// the XOR network four 3-input LOP3 pairs.
__device__ __forceinline__ uint32_t xstep(XState& s) {
  uint32_t x0, x1, o1;
  asm("add.cc.u32 %0, %2, %3;\n\taddc.u32 %1, %4, %5;"
      : "=r"(x0), "=r"(x1)
      : "r"(s.a0), "r"(s.d0), "r"(s.a1), "r"(s.d1));
  const uint32_t r1 = __funnelshift_l(x0, x1, 23), r0 = __funnelshift_l(x1, x0, 23);
  asm("{.reg .b32 t;\n\tadd.cc.u32 t, %1, %2;\n\taddc.u32 %0, %3, %4;}"
      : "=r"(o1)
      : "r"(r0), "r"(s.a0), "r"(r1), "r"(s.a1));
  // t = s1 << 17 through IMAD.WIDE (FMA pipe): lo = b0 << 17, hi = b0 >> 15
  uint64_t w17;
  asm("mul.wide.u32 %0, %1, 131072;" : "=l"(w17) : "r"(s.b0));
  const uint32_t t0 = (uint32_t)w17, t1 = s.b1 * 131072u + (uint32_t)(w17 >> 32);
  const uint32_t nc0 = xor3(s.c0, s.a0, t0), nc1 = xor3(s.c1, s.a1, t1);
  const uint32_t nd0 = s.d0 ^ s.b0, nd1 = s.d1 ^ s.b1;
  const uint32_t nb0 = xor3(s.b0, s.c0, s.a0), nb1 = xor3(s.b1, s.c1, s.a1);
  const uint32_t na0 = xor3(s.a0, s.d0, s.b0), na1 = xor3(s.a1, s.d1, s.b1);
  s.a0 = na0; s.a1 = na1; s.b0 = nb0; s.b1 = nb1; s.c0 = nc0; s.c1 = nc1;
  s.d1 = __funnelshift_l(nd1, nd0, 13);  // rotl64(nd, 45)
  s.d0 = __funnelshift_l(nd0, nd1, 13);
  return o1;
}

// acc = 2*acc + [h9 >= key]  (h9 = draw << 9): one carry-out compare plus
// one carry-in add.  [h9 >= key] is the REJECT bit of u23 < K (key = K<<9,
// or 0xFFFFFFFF when K == 2^23).
__device__ __forceinline__ void acc_reject(uint32_t& acc, uint32_t h9, uint32_t key) {
  asm("{.reg .b32 t;\n\tsub.cc.u32 t, %1, %2;\n\taddc.u32 %0, %0, %0;}" : "+r"(acc) : "r"(h9), "r"(key));
}

// Philox4x32-10 (Salmon et al., SC'11), the counter-based stream of
// paper_2404_16990_b200.rng.PhiloxStreams: counter (c0..c3), key (k0, k1).
// Each round is two IMAD.WIDE (FMA pipe) and two 3-input XORs (ALU); the
// round keys are warp-uniform.
__device__ __forceinline__ void philox10(uint32_t& c0, uint32_t& c1, uint32_t& c2, uint32_t& c3, uint32_t k0,
                                         uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; r++) {
    const uint64_t p0 = (uint64_t)c0 * 0xD2511F53u, p1 = (uint64_t)c2 * 0xCD9E8D57u;
    const uint32_t n0 = xor3((uint32_t)(p1 >> 32), c1, k0), n2 = xor3((uint32_t)(p0 >> 32), c3, k1);
    c1 = (uint32_t)p1;
    c3 = (uint32_t)p0;
    c0 = n0;
    c2 = n2;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

__device__ __forceinline__ uint64_t mix64(uint64_t z) {  // rng.py:53-58
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

__device__ __forceinline__ XState stream_state(uint64_t seed, uint64_t stream) {  // rng.py:71-82
  uint64_t z = mix64(seed + (stream + 1) * kGolden);
  uint64_t s[4];
#pragma unroll
  for (int i = 0; i < 4; i++) {
    z += kGolden;
    s[i] = mix64(z);
  }
  if (!(s[0] | s[1] | s[2] | s[3])) s[0] = kGolden;
  XState x;
  x.a0 = (uint32_t)s[0]; x.a1 = (uint32_t)(s[0] >> 32);
  x.b0 = (uint32_t)s[1]; x.b1 = (uint32_t)(s[1] >> 32);
  x.c0 = (uint32_t)s[2]; x.c1 = (uint32_t)(s[2] >> 32);
  x.d0 = (uint32_t)s[3]; x.d1 = (uint32_t)(s[3] >> 32);
  return x;
}

// s <- M s with M given as a nibble table T[64][16][8 words] (uint4 pairs).
__device__ __forceinline__ XState jump_apply(const XState& s, const uint4* __restrict__ T) {
  const uint32_t w[8] = {s.a0, s.a1, s.b0, s.b1, s.c0, s.c1, s.d0, s.d1};
  uint32_t r[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
  for (int q = 0; q < 8; q++) {
#pragma unroll
    for (int nib = 0; nib < 8; nib++) {
      const int p = q * 8 + nib;
      const uint32_t v = (w[q] >> (4 * nib)) & 15u;
      const uint4 lo = T[(p * 16 + v) * 2], hi = T[(p * 16 + v) * 2 + 1];
      r[0] ^= lo.x; r[1] ^= lo.y; r[2] ^= lo.z; r[3] ^= lo.w;
      r[4] ^= hi.x; r[5] ^= hi.y; r[6] ^= hi.z; r[7] ^= hi.w;
    }
  }
  XState o;
  o.a0 = r[0]; o.a1 = r[1]; o.b0 = r[2]; o.b1 = r[3];
  o.c0 = r[4]; o.c1 = r[5]; o.d0 = r[6]; o.d1 = r[7];
  return o;
}

__device__ __forceinline__ XState jump_by(XState s, uint64_t J, const uint4* __restrict__ pow) {
  for (int b = 0; b < 64; b++)
    if ((J >> b) & 1) s = jump_apply(s, pow + (size_t)b * (kJumpWords / 4));
  return s;
}

__device__ __forceinline__ void load_state(XState& s, const uint32_t* st, long long np, long long gp) {
  s.a0 = st[0 * np + gp]; s.a1 = st[1 * np + gp]; s.b0 = st[2 * np + gp]; s.b1 = st[3 * np + gp];
  s.c0 = st[4 * np + gp]; s.c1 = st[5 * np + gp]; s.d0 = st[6 * np + gp]; s.d1 = st[7 * np + gp];
}
__device__ __forceinline__ void store_state(const XState& s, uint32_t* st, long long np, long long gp) {
  st[0 * np + gp] = s.a0; st[1 * np + gp] = s.a1; st[2 * np + gp] = s.b0; st[3 * np + gp] = s.b1;
  st[4 * np + gp] = s.c0; st[5 * np + gp] = s.c1; st[6 * np + gp] = s.d0; st[7 * np + gp] = s.d1;
}

// ---------------------------------------------------------------------------
// device: geometry of the reference stream <-> colour-split rows
// ---------------------------------------------------------------------------

// For lattice row c and colour X: the reference cell (1-based gamma) whose
// stream gates it and the quarter q (position of the target array in
// FLIP_RED / FLIP_BLUE, engine.py:57-68).  Targets: (F,E)->0, (B,O)->1,
// (B,E)->2, (F,O)->3 for both colours, E/O = parity of the rows r of the
// colour's sites, (c+X)&1 (lattice.py:156-175).
struct RowStream {
  int gamma, q;
};
__device__ __host__ __forceinline__ RowStream row_stream(int m, int c, int X) {
  const bool fwd = c < m / 2;
  const int odd = (c + X) & 1;
  RowStream r;
  r.gamma = fwd ? c / 2 + 1 : (m - 1 - c) / 2 + 1;
  r.q = fwd ? (odd ? 3 : 0) : (odd ? 1 : 2);
  return r;
}

// ---------------------------------------------------------------------------
// device: the interleaved colour-split layout
// ---------------------------------------------------------------------------
//
// Row (c, X) holds the n/2 sites of colour X (X = 0 red: (c+r) even), site
// index i = r >> 1, split as i = 16 w + t (w < n/32, t < 16) -- exactly the
// reference's packing of a column vector into uint16 words, word w bit t
// (lattice.py:199-202).  Our uint32 word (ch, t) of the row holds bit t of
// the reference words w = 32 ch + b, b = 0..31: a 32-way transpose of the
// reference words, so the draws a stream consumes for one k (= one t, every
// w in order, engine.py:321-330) accumulate straight into one word per
// chunk.  Row pitch Wp = 16 * nch words, nch = ceil((n/32) / 32).

// Division by a run-time invariant 32-bit divisor with a multiply-high
// (round-up method): q = (t + ((x - t) >> s1)) >> s2, t = umulhi(x, m).
struct FastDiv {
  uint32_t d, m, s1, s2;
  __host__ void init(uint32_t div) {
    d = div;
    uint32_t l = 0;
    while (l < 32 && (1ull << l) < div) l++;
    m = (uint32_t)(((1ull << 32) * ((1ull << l) - div)) / div + 1);
    s1 = l < 1 ? l : 1;
    s2 = l > 0 ? l - 1 : 0;
  }
  __device__ __forceinline__ uint32_t div(uint32_t x) const {
    const uint32_t t = __umulhi(x, m);
    return (t + ((x - t) >> s1)) >> s2;
  }
};

struct Geo {
  int n_sim, m, n, rows, row0, ghost, R, Wp, words, nch;
  long long sim_offset;
  FastDiv rows_div, quads_div;
};

__host__ Geo make_geo(const msb_geom* g) {
  Geo o;
  o.n_sim = g->n_sim; o.m = g->m; o.n = g->n; o.rows = g->rows; o.row0 = g->row0; o.ghost = g->ghost;
  o.R = g->rows + 2 * g->ghost;
  o.words = g->n / 32;
  o.nch = (o.words + 31) / 32;
  o.Wp = 16 * o.nch;
  o.sim_offset = g->sim_offset;
  o.rows_div.init((uint32_t)o.rows);
  o.quads_div.init((uint32_t)(o.Wp / 4));
  return o;
}

// valid bits of chunk ch (w = 32 ch + b < n/32)
__device__ __forceinline__ int chunk_bits(const Geo& G, int ch) {
  const int b = G.words - 32 * ch;
  return b >= 32 ? 32 : b;
}
__device__ __forceinline__ uint32_t chunk_mask(const Geo& G, int ch) {
  const int b = chunk_bits(G, ch);
  return b >= 32 ? 0xFFFFFFFFu : ((1u << b) - 1u);
}
__device__ __forceinline__ size_t row_off(const Geo& G, int s, int X, int br) {
  return ((size_t)(s * 2 + X) * G.R + br) * G.Wp;
}
// buffer rows of the vertical neighbours (c-1, c+1) of buffer row br
__device__ __forceinline__ void vert_rows(const Geo& G, int br, int& bu, int& bd) {
  if (G.ghost) {
    bu = br - 1; bd = br + 1;
  } else {
    bu = br == 0 ? G.R - 1 : br - 1;
    bd = br + 1 == G.R ? 0 : br + 1;
  }
}

// The second horizontal neighbour (site i+1 when p=1, i-1 when p=0, periodic
// in n/2) of word (ch, t), read from the other colour's row y.  Interior t
// just uses word t+-1; t = 15 / t = 0 wrap into the next / previous w.
__device__ __forceinline__ uint32_t h_second(const Geo& G, const uint32_t* y, int ch, int t, int p) {
  if (p) {
    if (t < 15) return y[ch * 16 + t + 1];
    const int chn = ch + 1 < G.nch ? ch + 1 : 0;
    return (y[ch * 16] >> 1) | ((y[chn * 16] & 1u) << (chunk_bits(G, ch) - 1));
  }
  if (t > 0) return y[ch * 16 + t - 1];
  const uint32_t carry = ch > 0 ? (y[(ch - 1) * 16 + 15] >> 31)
                                : ((y[(G.nch - 1) * 16 + 15] >> (chunk_bits(G, G.nch - 1) - 1)) & 1u);
  return ((y[ch * 16 + 15] << 1) | carry) & chunk_mask(G, ch);
}

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
};

// draw sources of the producer
constexpr int kSrcXoshiro = 0;  // persistent per-piece reference streams
constexpr int kSrcExt = 1;      // host-supplied u23 draws
constexpr int kSrcPhilox = 2;   // counter-based Philox4x32-10

// reference bit t of a uint16 word is gated by draw k = 4(t%4) + t/4 (the
// mapping is its own inverse, engine.py:326-330)
__device__ __forceinline__ int t_of_k(int k) { return 4 * (k & 3) + (k >> 2); }

__device__ __forceinline__ size_t plane_off(const Geo& G, int np, int X, int p, int s, int lr) {
  return ((((size_t)X * np + p) * G.n_sim + s) * G.rows + lr) * G.Wp;
}

// Persistent kernel: one 1024-thread CTA per SM shares one copy of the
// sweep-jump table in shared memory; warps claim 32 consecutive pieces at a
// time from a self-resetting counter (work[0] = next unit, work[1] = warps
// done), so SMs stay balanced whatever the piece count.  Each lane runs one
// piece: it generates the piece's draws (k-range x all w) and, spread through
// the generation loop, performs the 64 nibble lookups of its jump to the
// next sweep, so table reads overlap other warps' ALU work.
constexpr int kRngThreads = 1024;
#ifndef MSB_CHUNK_UNROLL
#define MSB_CHUNK_UNROLL 16
#endif
constexpr int kChunkUnroll = MSB_CHUNK_UNROLL;

// Work counters (caller-owned, zeroed once, left zeroed by every kernel):
//   work[0] next dynamic producer unit    work[1] consumer barrier arrivals
//   work[2] warps finished (last one resets all four)
__device__ __forceinline__ void finish_warp(unsigned* work, unsigned total_warps) {
  if ((threadIdx.x & 31) == 0) {
    __threadfence();
    if (atomicAdd(work + 2, 1u) == total_warps - 1) {
      atomicExch(work, 0u);
      atomicExch(work + 1, 0u);
      atomicExch(work + 2, 0u);
    }
  }
}

// One producer warp's share of a sweep's accept planes.  `role_warp` /
// `role_warps` number the producer warps of the grid; their first unit is
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
  for (;;) {
    if (u >= units) break;
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
          outk[ch * 16] = ~__brev(acc0);
          if (np > 1) outk[pstride + ch * 16] = ~__brev(acc1);
        }
      } else
      for (int ch = 0; ch < G.nch; ch++) {
        const int L = FULL ? 32 : chunk_bits(G, ch);
        uint32_t acc[NPMAX];
#pragma unroll
        for (int p = 0; p < NPMAX; p++) acc[p] = 0;
        if (SRC == kSrcPhilox) {
          const unsigned long long d0 = pd0 + (unsigned long long)k * G.words + 32 * ch;
          if ((d0 & 3) == 0 && (L & 3) == 0) {
            for (int i = 0; i < L; i += 4) {
              const unsigned long long c = (d0 + i) >> 2;
              uint32_t x0 = (uint32_t)c, x1 = (uint32_t)(c >> 32), x2 = ps0, x3 = ps1;
              philox10(x0, x1, x2, x3, a.seed_lo, a.seed_hi);
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
              philox10(x0, x1, x2, x3, a.seed_lo, a.seed_hi);
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
      if (XO) {
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
}

template <int NPMAX, int SRC, bool FULL>
__global__ void __launch_bounds__(kRngThreads, 1) k_rng_planes(const RngArgs a) {
  extern __shared__ uint4 jt[];  // nibble table of A^(4n), 32 KiB
  if (SRC == kSrcXoshiro) {
    for (int i = threadIdx.x; i < kJumpWords / 4; i += blockDim.x) jt[i] = a.jump[i];
    __syncthreads();
  }
  rng_produce<NPMAX, SRC, FULL>(a, jt, threadIdx.x >> 5, blockDim.x >> 5);
  finish_warp(a.work, gridDim.x * (blockDim.x >> 5));
}

// ---------------------------------------------------------------------------
// device: the flip pass (one colour)
// ---------------------------------------------------------------------------

struct FlipArgs {
  Geo G;
  uint32_t* spins;
  const uint32_t* planes;
  unsigned long long* flips;
  int X, np, cwarps;
  uint32_t inv;
  int fault;
  int8_t code_plane[16];
};

constexpr int kFlipSlots = 256;

__device__ __forceinline__ uint32_t flip_word(const FlipArgs& a, bool generic, uint32_t o, uint32_t n1, uint32_t n2,
                                              uint32_t y0, uint32_t n4, const uint32_t* pl, size_t pstride,
                                              uint32_t A4, uint32_t A8) {
  if (!generic) {
    const uint32_t ow = o ^ a.inv;
    const uint32_t x1 = n1 ^ ow, x2 = n2 ^ ow, x3 = y0 ^ ow;
    const uint32_t x4 = a.fault ? 0u : (n4 ^ ow);
    const uint32_t o12 = x1 | x2, a12 = x1 & x2, o34 = x3 | x4, a34 = x3 & x4;
    const uint32_t ge2 = a12 | a34 | (o12 & o34);  // >= 2 disagreeing neighbours
    const uint32_t any = o12 | o34;
    return ge2 | (any & ~ge2 & A4) | (~any & A8);
  }
  // neighbour up-count bit planes (bitkernels.py:63-79 restated)
  const uint32_t s1 = n1 ^ n2, c1 = n1 & n2, s2 = y0 ^ n4, c2 = y0 & n4;
  uint32_t ones = s1 ^ s2;
  const uint32_t twos = c1 ^ c2 ^ (s1 & s2), fours = c1 & c2;
  if (a.fault) ones = s1;
  uint32_t flip = 0;
  for (int code = 0; code < 16; code++) {
    const int pidx = a.code_plane[code];
    const int u = code & 7;
    if (pidx == -1 || u > 4) continue;
    const uint32_t msk = ((code & 8) ? o : ~o) & ((u & 1) ? ones : ~ones) & ((u & 2) ? twos : ~twos) &
                         ((u & 4) ? fours : ~fours);
    flip |= pidx == -2 ? msk : (msk & __ldg(pl + pidx * pstride));
  }
  return flip;
}

// One quad of 4 t-words (t0..t0+3 of chunk ch) of row (s, lr) in colour
// a.X.  Vertical neighbours are the other colour's rows c-1, c+1 (same
// word); horizontal ones the other colour's row c at sites i and i+-1
// (h_second).  COHERENT: other-colour words were written earlier in the same
// kernel by other SMs, so read them through L2 (ld.global.cg).
template <bool GENERIC, bool COHERENT>
__device__ __forceinline__ unsigned flip_quad_at(const FlipArgs& a, int s, int lr, unsigned qq, int X) {
  const Geo& G = a.G;
  const int c = G.row0 + lr, br = lr + G.ghost;
  const int ch = (int)(qq >> 2), t0 = 4 * (int)(qq & 3);
  const int w0 = ch * 16 + t0;
  int bu, bd;
  vert_rows(G, br, bu, bd);
  uint32_t* own = a.spins + row_off(G, s, X, br);
  const uint32_t* yc = a.spins + row_off(G, s, 1 - X, br);
  auto ld4 = [](const uint32_t* q) {
    return COHERENT ? __ldcg(reinterpret_cast<const uint4*>(q)) : __ldg(reinterpret_cast<const uint4*>(q));
  };
  auto ld1 = [](const uint32_t* q) { return COHERENT ? __ldcg(q) : __ldg(q); };
  const uint4 O = *reinterpret_cast<const uint4*>(own + w0);
  const uint4 Y = ld4(yc + w0);
  const uint4 U = ld4(a.spins + row_off(G, s, 1 - X, bu) + w0);
  const uint4 D = ld4(a.spins + row_off(G, s, 1 - X, bd) + w0);
  const size_t pstride = (size_t)G.n_sim * G.rows * G.Wp;
  const uint32_t* pl = a.planes + plane_off(G, a.np, X, 0, s, lr) + w0;
  uint4 P4 = make_uint4(0, 0, 0, 0), P8 = make_uint4(0, 0, 0, 0);
  if (!GENERIC) {
    P4 = __ldg(reinterpret_cast<const uint4*>(pl));
    P8 = __ldg(reinterpret_cast<const uint4*>(pl + pstride));
  }
  const int p = (c + X) & 1;
  const uint32_t y[4] = {Y.x, Y.y, Y.z, Y.w};
  const uint32_t o[4] = {O.x, O.y, O.z, O.w};
  const uint32_t u4[4] = {U.x, U.y, U.z, U.w};
  const uint32_t d4[4] = {D.x, D.y, D.z, D.w};
  const uint32_t a4[4] = {P4.x, P4.y, P4.z, P4.w};
  const uint32_t a8[4] = {P8.x, P8.y, P8.z, P8.w};
  // the neighbour word just outside the quad (t0+4 if p, t0-1 otherwise) or,
  // at t = 15 / t = 0, the shifted word of the next / previous w
  uint32_t edge;
  const int vb = chunk_bits(G, ch);
  if (p) {
    if (t0 + 4 < 16) {
      edge = ld1(yc + w0 + 4);
    } else {
      const int chn = ch + 1 < G.nch ? ch + 1 : 0;
      edge = (ld1(yc + ch * 16) >> 1) | ((ld1(yc + chn * 16) & 1u) << (vb - 1));
    }
  } else {
    if (t0 > 0) {
      edge = ld1(yc + w0 - 1);
    } else {
      const uint32_t carry = ch > 0 ? (ld1(yc + (ch - 1) * 16 + 15) >> 31)
                                    : ((ld1(yc + (G.nch - 1) * 16 + 15) >> (chunk_bits(G, G.nch - 1) - 1)) & 1u);
      edge = ((ld1(yc + ch * 16 + 15) << 1) | carry) & chunk_mask(G, ch);
    }
  }
  const uint32_t vm = chunk_mask(G, ch);
  uint32_t res[4];
  unsigned cnt = 0;
#pragma unroll
  for (int k = 0; k < 4; k++) {
    const uint32_t n4 = p ? (k < 3 ? y[k + 1] : edge) : (k > 0 ? y[k - 1] : edge);
    uint32_t f = flip_word(a, GENERIC, o[k], u4[k], d4[k], y[k], n4, pl + k, pstride, a4[k], a8[k]);
    f &= vm;
    res[k] = o[k] ^ f;
    cnt += __popc(f);
  }
  *reinterpret_cast<uint4*>(own + w0) = make_uint4(res[0], res[1], res[2], res[3]);
  return cnt;
}

template <bool GENERIC, bool COHERENT>
__device__ __forceinline__ unsigned flip_quad(const FlipArgs& a, unsigned i, int X) {
  const Geo& G = a.G;
  const unsigned quads = (unsigned)G.Wp >> 2;
  const unsigned gr = G.quads_div.div(i), qq = i - gr * quads;
  const int s = (int)G.rows_div.div(gr), lr = (int)(gr - (unsigned)s * G.rows);
  return flip_quad_at<GENERIC, COHERENT>(a, s, lr, qq, X);
}

// FERRO/ANTI flip of one whole 16-word chunk (t = 0..15 of chunk ch) of row
// (s, lr), colour X.  The other colour's same-row words stay in registers, so
// every t+-1 neighbour -- and, when the row is one chunk, the t = 0/15 wraps
// -- comes from registers; address math happens once per chunk.
template <bool COHERENT>
__device__ __forceinline__ unsigned flip_chunk_at(const FlipArgs& a, int s, int lr, int ch, int X) {
  const Geo& G = a.G;
  const int c = G.row0 + lr, br = lr + G.ghost;
  int bu, bd;
  vert_rows(G, br, bu, bd);
  const int w0 = ch * 16;
  uint32_t* own = a.spins + row_off(G, s, X, br) + w0;
  const uint32_t* ycr = a.spins + row_off(G, s, 1 - X, br);
  const uint32_t* yu = a.spins + row_off(G, s, 1 - X, bu) + w0;
  const uint32_t* yd = a.spins + row_off(G, s, 1 - X, bd) + w0;
  const size_t pstride = (size_t)G.n_sim * G.rows * G.Wp;
  const uint32_t* pl = a.planes + plane_off(G, a.np, X, 0, s, lr) + w0;
  auto ld4 = [](const uint32_t* q) {
    return COHERENT ? __ldcg(reinterpret_cast<const uint4*>(q)) : __ldg(reinterpret_cast<const uint4*>(q));
  };
  auto ld1 = [](const uint32_t* q) { return COHERENT ? __ldcg(q) : __ldg(q); };
  uint32_t y[16];
#pragma unroll
  for (int q = 0; q < 4; q++) {
    const uint4 v = ld4(ycr + w0 + 4 * q);
    y[4 * q] = v.x; y[4 * q + 1] = v.y; y[4 * q + 2] = v.z; y[4 * q + 3] = v.w;
  }
  const int p = (c + X) & 1;
  const int vb = chunk_bits(G, ch);
  const uint32_t vm = chunk_mask(G, ch);
  // the wrap word: p=1 -> t=15 needs bit 0 of the next chunk's t=0 word;
  // p=0 -> t=0 needs the top valid bit of the previous chunk's t=15 word
  uint32_t wrapn;
  if (p) {
    const int chn = ch + 1 < G.nch ? ch + 1 : 0;
    const uint32_t nx = chn == ch ? y[0] : ld1(ycr + chn * 16);
    wrapn = (y[0] >> 1) | ((nx & 1u) << (vb - 1));
  } else {
    uint32_t carry;
    if (ch > 0) carry = ld1(ycr + (ch - 1) * 16 + 15) >> 31;
    else carry = ((G.nch == 1 ? y[15] : ld1(ycr + (G.nch - 1) * 16 + 15)) >> (chunk_bits(G, G.nch - 1) - 1)) & 1u;
    wrapn = ((y[15] << 1) | carry) & vm;
  }
  unsigned cnt = 0;
#pragma unroll
  for (int q = 0; q < 4; q++) {
    const uint4 O = *reinterpret_cast<const uint4*>(own + 4 * q);
    const uint4 U = ld4(yu + 4 * q), D = ld4(yd + 4 * q);
    const uint4 P4 = __ldg(reinterpret_cast<const uint4*>(pl + 4 * q));
    const uint4 P8 = __ldg(reinterpret_cast<const uint4*>(pl + pstride + 4 * q));
    const uint32_t o[4] = {O.x, O.y, O.z, O.w}, u4[4] = {U.x, U.y, U.z, U.w}, d4[4] = {D.x, D.y, D.z, D.w};
    const uint32_t a4[4] = {P4.x, P4.y, P4.z, P4.w}, a8[4] = {P8.x, P8.y, P8.z, P8.w};
    uint32_t res[4];
#pragma unroll
    for (int k = 0; k < 4; k++) {
      const int t = 4 * q + k;
      const uint32_t n4 = p ? (t < 15 ? y[t + 1] : wrapn) : (t > 0 ? y[t - 1] : wrapn);
      const uint32_t f = flip_word(a, false, o[k], u4[k], d4[k], y[t], n4, nullptr, 0, a4[k], a8[k]) & vm;
      res[k] = o[k] ^ f;
      cnt += __popc(f);
    }
    *reinterpret_cast<uint4*>(own + 4 * q) = make_uint4(res[0], res[1], res[2], res[3]);
  }
  return cnt;
}

// A consumer warp's contiguous run of chunks [i0, i1) (lanes take
// consecutive chunks), walked with incremental (replica, row, chunk) state.
template <bool COHERENT>
__device__ __forceinline__ unsigned flip_run_chunks(const FlipArgs& a, unsigned i0, unsigned i1, int X) {
  const Geo& G = a.G;
  if (i0 >= i1) return 0;
  const unsigned nch = (unsigned)G.nch;
  unsigned gr = i0 / nch, ch = i0 - gr * nch;
  int s = (int)G.rows_div.div(gr), lr = (int)(gr - (unsigned)s * G.rows);
  const unsigned dr = 32u / nch, dc = 32u - dr * nch;
  unsigned cnt = 0;
  for (unsigned i = i0; i < i1; i += 32) {
    cnt += flip_chunk_at<COHERENT>(a, s, lr, (int)ch, X);
    ch += dc;
    lr += (int)dr;
    if (ch >= nch) {
      ch -= nch;
      lr++;
    }
    while (lr >= G.rows) {
      lr -= G.rows;
      s++;
    }
  }
  return cnt;
}

// A consumer warp's contiguous run of quads [i0, i1) of one colour, walked
// with incremental (replica, row, quad) bookkeeping: lanes take consecutive
// quads, each step advances all lanes by 32 quads (dr rows + dq quads).
template <bool COHERENT>
__device__ __forceinline__ unsigned flip_run(const FlipArgs& a, unsigned i0, unsigned i1, int X) {
  const Geo& G = a.G;
  const unsigned quads = (unsigned)G.Wp >> 2;
  if (i0 >= i1) return 0;
  unsigned gr = G.quads_div.div(i0), qq = i0 - gr * quads;
  int s = (int)G.rows_div.div(gr), lr = (int)(gr - (unsigned)s * G.rows);
  const unsigned dr = G.quads_div.div(32u), dq = 32u - dr * quads;
  unsigned cnt = 0;
  for (unsigned i = i0; i < i1; i += 32) {
    cnt += flip_quad_at<false, COHERENT>(a, s, lr, qq, X);
    qq += dq;
    lr += (int)dr;
    if (qq >= quads) {
      qq -= quads;
      lr++;
    }
    while (lr >= G.rows) {
      lr -= G.rows;
      s++;
    }
  }
  return cnt;
}

__device__ __forceinline__ void add_flips(unsigned long long* flips, unsigned cnt) {
  cnt = __reduce_add_sync(0xFFFFFFFFu, cnt);
  if ((threadIdx.x & 31) == 0 && cnt)
    atomicAdd(flips + ((blockIdx.x * 32 + (threadIdx.x >> 5)) % kFlipSlots), (unsigned long long)cnt);
}

template <bool GENERIC>
__global__ void __launch_bounds__(256) k_flip(const FlipArgs a) {
  const unsigned quads = (unsigned)a.G.Wp >> 2;
  const unsigned total = (unsigned)a.G.n_sim * (unsigned)a.G.rows * quads;
  const unsigned i = blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned cnt = i < total ? flip_quad<GENERIC, false>(a, i, a.X) : 0u;
  add_flips(a.flips, cnt);
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

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <int NPMAX, int SRC, bool FULL>
__global__ void __launch_bounds__(kRngThreads, 1) k_sweep_fused(const RngArgs ra, const FlipArgs fa) {
  const int kFlipWarps = fa.cwarps;
  const int kProducerWarps = (kRngThreads >> 5) - kFlipWarps;
  extern __shared__ uint4 jt[];
  if (SRC == kSrcXoshiro) {
    for (int i = threadIdx.x; i < kJumpWords / 4; i += blockDim.x) jt[i] = ra.jump[i];
    __syncthreads();
  }
  const int warp = threadIdx.x >> 5;
  const unsigned total_warps = gridDim.x * (blockDim.x >> 5);
  if (warp < kProducerWarps) {
    rng_produce<NPMAX, SRC, FULL>(ra, jt, warp, kProducerWarps);
  } else {
    const unsigned total = (unsigned)fa.G.n_sim * (unsigned)fa.G.rows * (unsigned)fa.G.nch;  // chunks
    const unsigned nc = gridDim.x * kFlipWarps;
    const unsigned cw = (warp - kProducerWarps) * gridDim.x + blockIdx.x;
    const unsigned per = ((total + nc - 1) / nc + 31) & ~31u;  // chunks per consumer warp
    const unsigned lo = min(total, cw * per), hi = min(total, lo + per);
    const unsigned i0 = lo + (threadIdx.x & 31);
    unsigned cnt = 0;
    for (int X = 0; X < 2; X++) {
      if (X == 0) {
        cnt += flip_run_chunks<false>(fa, i0, hi, 0);
      } else {
        cnt += flip_run_chunks<true>(fa, i0, hi, 1);
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
      }
    }
    add_flips(fa.flips, cnt);
  }
  finish_warp(ra.work, total_warps);
}

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

// Thread per (s, held row lr, word (ch, t)): both colours' word from the
// linear row, read as uint32 words (linear bit i -> bit i%32 of word i/32).
// Sites of word (ch, t): r = 32 w + 2 t + {0, 1}, w = 32 ch + b; the even r
// belongs to colour c&1, the odd one to (c+1)&1.
__global__ void k_from_linear(Geo G, const uint32_t* __restrict__ lin, uint32_t* spins) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long total = (long long)G.n_sim * G.rows * G.Wp;
  if (i >= total) return;
  const int wd = (int)(i % G.Wp);
  const long long gr = i / G.Wp;
  const int s = (int)(gr / G.rows), lr = (int)(gr % G.rows);
  const int c = G.row0 + lr, br = lr + G.ghost;
  const int ch = wd >> 4, t = wd & 15;
  const uint32_t* L = lin + ((size_t)s * G.rows + lr) * (G.n / 32) + 32 * ch;
  const int nb = chunk_bits(G, ch);
  uint32_t e = 0, od = 0;
  for (int b = 0; b < nb; b++) {
    const uint32_t v = L[b] >> (2 * t);
    e |= (v & 1u) << b;
    od |= ((v >> 1) & 1u) << b;
  }
  spins[row_off(G, s, c & 1, br) + wd] = e;
  spins[row_off(G, s, (c + 1) & 1, br) + wd] = od;
}

// Thread per linear uint32 word (s, lr, w): sites r = 32 w .. 32 w + 31.
__global__ void k_to_linear(Geo G, const uint32_t* __restrict__ spins, uint32_t* lin) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long total = (long long)G.n_sim * G.rows * G.words;
  if (i >= total) return;
  const int w = (int)(i % G.words);
  const long long gr = i / G.words;
  const int s = (int)(gr / G.rows), lr = (int)(gr % G.rows);
  const int c = G.row0 + lr, br = lr + G.ghost;
  const int ch = w >> 5, b = w & 31;
  const uint32_t* E = spins + row_off(G, s, c & 1, br) + ch * 16;
  const uint32_t* Od = spins + row_off(G, s, (c + 1) & 1, br) + ch * 16;
  uint32_t v = 0;
#pragma unroll
  for (int t = 0; t < 16; t++) v |= (((E[t] >> b) & 1u) << (2 * t)) | (((Od[t] >> b) & 1u) << (2 * t + 1));
  lin[i] = v;
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

__global__ void k_observe(Geo G, const uint32_t* __restrict__ spins, long long* ups, long long* unsat) {
  const long long gr = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long total = (long long)G.n_sim * G.rows;
  int s = -1;
  uint32_t u = 0, b = 0;
  if (gr < total) {
    s = (int)(gr / G.rows);
    const int lr = (int)(gr % G.rows);
    const int c = G.row0 + lr, br = lr + G.ghost;
    const int p = c & 1;  // red sites of row c sit at rows r with parity c&1
    int bu, bd;
    vert_rows(G, br, bu, bd);
    const uint32_t* red = spins + row_off(G, s, 0, br);
    const uint32_t* blu = spins + row_off(G, s, 1, br);
    const uint32_t* yu = spins + row_off(G, s, 1, bu);
    const uint32_t* yd = spins + row_off(G, s, 1, bd);
    for (int ch = 0; ch < G.nch; ch++) {
      const uint32_t vm = chunk_mask(G, ch);
      for (int t = 0; t < 16; t++) {
        const int wd = ch * 16 + t;
        const uint32_t o = red[wd], y0 = blu[wd];
        u += __popc(o) + __popc(y0);
        b += __popc((o ^ yu[wd]) & vm) + __popc((o ^ yd[wd]) & vm) + __popc((o ^ y0) & vm) +
             __popc((o ^ h_second(G, blu, ch, t, p)) & vm);
      }
    }
  }
  // segmented warp reduction by replica
  const unsigned lanes = __match_any_sync(0xFFFFFFFFu, s);
  const uint32_t su = __reduce_add_sync(lanes, u), sb = __reduce_add_sync(lanes, b);
  const int leader = __ffs(lanes) - 1;
  if (s >= 0 && (int)(threadIdx.x & 31) == leader) {
    atomicAdd(reinterpret_cast<unsigned long long*>(ups + s), (unsigned long long)su);
    atomicAdd(reinterpret_cast<unsigned long long*>(unsat + s), (unsigned long long)sb);
  }
}

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

// ---------------------------------------------------------------------------
// host helpers
// ---------------------------------------------------------------------------

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

inline unsigned blocks_for(long long n, int bt) { return (unsigned)((n + bt - 1) / bt); }

template <typename K>
int set_smem_attr(K kernel, std::once_flag& once, cudaError_t& err) {
  std::call_once(once, [&] {
    err = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  });
  if (err != cudaSuccess) return fail(MSB_ERR_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(err));
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
  if (p->rng != MSB_RNG_XOSHIRO && p->rng != MSB_RNG_PHILOX) return fail(MSB_ERR_ARG, "unknown rng");
  return MSB_OK;
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
}

void fill_flip_args(FlipArgs& a, const msb_geom* g, const msb_sweep_params* p, int colour, uint32_t* spins,
                    const uint32_t* planes, uint64_t* flips) {
  a.G = make_geo(g);
  a.spins = spins;
  a.planes = planes;
  a.flips = reinterpret_cast<unsigned long long*>(flips);
  a.X = colour;
  a.np = p->n_planes;
  a.inv = p->mode == MSB_MODE_ANTI ? 0xFFFFFFFFu : 0u;
  a.fault = p->fault;
  std::memcpy(a.code_plane, p->code_plane, 16);
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
  const size_t smem = (ext || p->rng == MSB_RNG_PHILOX) ? 0 : (size_t)kJumpWords * 4;
#define MSB_LAUNCH_RNG(NP, SRC, FULL)                                         \
  do {                                                                        \
    static std::once_flag o;                                                  \
    static cudaError_t e;                                                     \
    if (int r = set_smem_attr(k_rng_planes<NP, SRC, FULL>, o, e)) return r;   \
    k_rng_planes<NP, SRC, FULL><<<grid, kRngThreads, smem, st>>>(a);          \
  } while (0)
  const int src = ext ? kSrcExt : (p->rng == MSB_RNG_PHILOX ? kSrcPhilox : kSrcXoshiro);
  const bool full = (a.G.words % 32) == 0;
  if (p->mode != MSB_MODE_GENERIC) {
    if (src == kSrcExt) MSB_LAUNCH_RNG(2, kSrcExt, false);
    else if (src == kSrcPhilox) MSB_LAUNCH_RNG(2, kSrcPhilox, false);
    else if (full) MSB_LAUNCH_RNG(2, kSrcXoshiro, true);
    else MSB_LAUNCH_RNG(2, kSrcXoshiro, false);
  } else {
    if (src == kSrcExt) MSB_LAUNCH_RNG(MSB_MAX_PLANES, kSrcExt, false);
    else if (src == kSrcPhilox) MSB_LAUNCH_RNG(MSB_MAX_PLANES, kSrcPhilox, false);
    else MSB_LAUNCH_RNG(MSB_MAX_PLANES, kSrcXoshiro, false);
  }
#undef MSB_LAUNCH_RNG
  CUDA_TRY(cudaGetLastError());
  return MSB_OK;
}

int flip(const msb_geom* g, const msb_sweep_params* p, int colour, uint32_t* spins, const uint32_t* planes,
         uint64_t* flips, cudaStream_t st) {
  const Geo G = make_geo(g);
  FlipArgs a;
  fill_flip_args(a, g, p, colour, spins, planes, flips);
  const long long total = (long long)g->n_sim * g->rows * (G.Wp / 4);
  if (total >= (1LL << 31)) return fail(MSB_ERR_UNSUPPORTED, "too many words for one flip launch");
  if (p->mode == MSB_MODE_GENERIC)
    k_flip<true><<<blocks_for(total, 256), 256, 0, st>>>(a);
  else
    k_flip<false><<<blocks_for(total, 256), 256, 0, st>>>(a);
  CUDA_TRY(cudaGetLastError());
  return MSB_OK;
}


// flips of the sweep whose planes are in `cur` + planes of the next sweep
// into `next`, one cooperative launch (FERRO/ANTI whole lattices).
int fused_sweep(const msb_geom* g, const msb_sweep_params* p, uint32_t* spins, uint32_t* states, const uint32_t* cur,
                uint32_t* next, uint64_t* flips, cudaStream_t st) {
  RngArgs ra;
  fill_rng_args(ra, g, p, -1, states, nullptr, next);
  FlipArgs fa;
  fill_flip_args(fa, g, p, 0, spins, cur, flips);
  {
    // split the CTA's 32 warps between plane producers and flip consumers in
    // proportion to the work: a flip quad costs ~1/16 of a piece's draws per
    // word, but is latency-bound, so weight it up
    static const int env_cw = [] { const char* e = getenv("MSB_FLIP_WARPS"); return e ? atoi(e) : 0; }();
    // 6 flip warps per CTA measured best for flip-heavy shapes (cfg3/cfg4);
    // fewer when that keeps every producer warp to one unit (cfg2)
    int cw = 6;
    // never add a producer round: keep ceil(units / (SMs * producers)) minimal
    const long long units = (2LL * g->n_sim * g->rows * p->kg + 31) / 32;
    const int sms_est = 148;
    auto rounds = [&](int c) { return (units + (long long)sms_est * (32 - c) - 1) / ((long long)sms_est * (32 - c)); };
    if (rounds(2) == 1)  // single-round problems: every producer warp counts
      while (cw > 2 && rounds(cw) > 1) cw--;
    fa.cwarps = env_cw > 0 ? std::min(28, env_cw) : cw;
  }
  int dev = 0, sms = 148;
  CUDA_TRY(cudaGetDevice(&dev));
  CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const bool philox = p->rng == MSB_RNG_PHILOX;
  const bool full = (fa.G.words % 32) == 0;
  static std::once_flag o, o2, o3;
  static cudaError_t e, e2, e3;
  if (int r = set_smem_attr(k_sweep_fused<2, kSrcXoshiro, false>, o, e)) return r;
  if (int r = set_smem_attr(k_sweep_fused<2, kSrcPhilox, false>, o2, e2)) return r;
  if (int r = set_smem_attr(k_sweep_fused<2, kSrcXoshiro, true>, o3, e3)) return r;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)sms);
  cfg.blockDim = dim3(kRngThreads);
  cfg.dynamicSmemBytes = philox ? 0 : (size_t)kJumpWords * 4;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (philox) CUDA_TRY(cudaLaunchKernelEx(&cfg, k_sweep_fused<2, kSrcPhilox, false>, ra, fa));
  else if (full) CUDA_TRY(cudaLaunchKernelEx(&cfg, k_sweep_fused<2, kSrcXoshiro, true>, ra, fa));
  else CUDA_TRY(cudaLaunchKernelEx(&cfg, k_sweep_fused<2, kSrcXoshiro, false>, ra, fa));
  return MSB_OK;
}
}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================

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

int msb_abi_version(void) { return 1; }

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
  const long long total = (long long)G.n_sim * G.rows * G.Wp;
  k_from_linear<<<blocks_for(total, 256), 256, 0, as_stream(stream)>>>(
      G, reinterpret_cast<const uint32_t*>(lin), spins);
  CUDA_TRY(cudaGetLastError());
  return MSB_OK;
}

int msb_to_linear(const msb_geom* g, const uint32_t* spins, uint64_t* lin, void* stream) {
  if (int r = check_geom(g)) return r;
  if (!lin || !spins) return fail(MSB_ERR_ARG, "null buffer");
  const Geo G = make_geo(g);
  const long long total = (long long)G.n_sim * G.rows * G.words;
  k_to_linear<<<blocks_for(total, 256), 256, 0, as_stream(stream)>>>(G, spins, reinterpret_cast<uint32_t*>(lin));
  CUDA_TRY(cudaGetLastError());
  return MSB_OK;
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

int msb_observe(const msb_geom* g, const uint32_t* spins, int64_t* ups, int64_t* unsat, void* stream) {
  if (int r = check_geom(g)) return r;
  if (!spins || !ups || !unsat) return fail(MSB_ERR_ARG, "null buffer");
  const Geo G = make_geo(g);
  const long long total = (long long)g->n_sim * g->rows;
  k_observe<<<blocks_for(total, 256), 256, 0, as_stream(stream)>>>(G, spins, reinterpret_cast<long long*>(ups),
                                                                    reinterpret_cast<long long*>(unsat));
  CUDA_TRY(cudaGetLastError());
  return MSB_OK;
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
                                                              p->rng == MSB_RNG_PHILOX, (uint32_t)p->seed,
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
