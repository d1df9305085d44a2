// Shared device code of libmsb200 (sm_100a): the reference RNG restated for
// the GPU, the colour-split row geometry and the host-side argument checks.
// Included by msb_sweep.cu (hot path), msb_state.cu (state/layout kernels)
// and msb_host.cu (host-only ABI).  See include/msb200.h for the ABI and
// DESIGN.md for the layout / roofline discussion.
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
#pragma once
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

namespace msbk {

constexpr uint64_t kGolden = 0x9E3779B97F4B7C15ULL;
constexpr int kJumpWords = 8192;  // one nibble table = 32 KiB
constexpr uint32_t kKeyAlways = 0xFFFFFFFFu;

// error reporting (msb_last_error), defined in msb_host.cu
int fail(int code, const std::string& why);
int check_geom(const msb_geom* g);
int check_params(const msb_sweep_params* p);

#define CUDA_TRY(expr)                                                                 \
  do {                                                                                 \
    cudaError_t e_ = (expr);                                                           \
    if (e_ != cudaSuccess) return fail(MSB_ERR_CUDA, std::string(#expr ": ") + cudaGetErrorString(e_)); \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

inline unsigned blocks_for(long long n, int bt) { return (unsigned)((n + bt - 1) / bt); }

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
  // The XOR network's statement and operand order is part of the tuning:
  // ptxas's register assignment (and bank conflicts at dispatch) follows it,
  // and permutations measured up to 7% apart; this one was fastest
  // (1.5% over the natural order, cfg2 window).
  const uint32_t nd0 = s.d0 ^ s.b0, nd1 = s.d1 ^ s.b1;
  const uint32_t na0 = xor3(s.d0, s.b0, s.a0), na1 = xor3(s.d1, s.b1, s.a1);
  const uint32_t nb0 = xor3(s.c0, s.a0, s.b0), nb1 = xor3(s.c1, s.a1, s.b1);
  const uint32_t nc0 = xor3(t0, s.a0, s.c0), nc1 = xor3(t1, s.a1, s.c1);
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

// Round keys of Philox4x32-10 for one master seed, computed on the host
// (philox_keys): round r uses (k[2r], k[2r+1]).  Kernels take them by value
// in their parameter block, so every XOR reads its key straight from the
// constant bank instead of re-deriving it per call.
struct PhiloxKeys {
  uint32_t k[20];
};

inline PhiloxKeys philox_keys(uint64_t seed) {
  PhiloxKeys K;
  uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  for (int r = 0; r < 10; r++, k0 += 0x9E3779B9u, k1 += 0xBB67AE85u) {
    K.k[2 * r] = k0;
    K.k[2 * r + 1] = k1;
  }
  return K;
}

constexpr uint32_t kPhiloxM0 = 0xD2511F53u, kPhiloxM1 = 0xCD9E8D57u;

__device__ __forceinline__ void philox_round(uint32_t& c0, uint32_t& c1, uint32_t& c2, uint32_t& c3, uint32_t k0,
                                             uint32_t k1) {
  // plain XORs (not the asm xor3): the key can stay a constant-bank operand
  const uint64_t p0 = (uint64_t)c0 * kPhiloxM0, p1 = (uint64_t)c2 * kPhiloxM1;
  const uint32_t n0 = (uint32_t)(p1 >> 32) ^ k0 ^ c1, n2 = (uint32_t)(p0 >> 32) ^ k1 ^ c3;
  c1 = (uint32_t)p1;
  c3 = (uint32_t)p0;
  c0 = n0;
  c2 = n2;
}

// Bit b of the 32-bit key as an all-lanes mask, recomputed at its point of
// use (volatile: hoisted out of the group loop, the 46 masks spill).
__device__ __forceinline__ uint32_t key_mask(uint32_t key, int b) {
  uint32_t m;
  asm volatile("{.reg .b32 t;\n\tshl.b32 t, %1, %2;\n\tshr.s32 %0, t, 31;}" : "=r"(m) : "r"(key), "r"(b));
  return m;
}

// philox10 with host-computed round keys.
__device__ __forceinline__ void philox10k(uint32_t& c0, uint32_t& c1, uint32_t& c2, uint32_t& c3,
                                          const PhiloxKeys& K) {
#pragma unroll
  for (int r = 0; r < 10; r++) philox_round(c0, c1, c2, c3, K.k[2 * r], K.k[2 * r + 1]);
}

// Bit-plane Philox stream (paper_2404_16990_b200.rng.PhiloxBitStreams):
// group g of stream S = draws 32g .. 32g+31; Philox block j (0..5) with
// counter (g lo, (g hi << 3) | j, S lo, S hi | 2^31) gives planes 4j .. 4j+3;
// bit i of plane b is bit 22-b of draw 32g+i.  pbits_group resolves the 32
// comparisons u23 < K_p most significant plane first and stops generating
// planes once every comparison is decided (~7-8 planes instead of 23 bits
// per draw).  key[p] = K_p << 9 (kKeyAlways when K_p = 2^23, 0 when K_p = 0);
// acc[p] bit i = [draw 32g+i < K_p].  A comparison still open after plane 22
// is u == K: rejected.
//
// The six blocks of a group differ only in the low bits of counter word 1,
// so the first three rounds are largely shared: round 1 entirely (block j
// only XORs j into its output word 0), round 2's word-2 product and round
// 3's word-0 product.  A block then costs 16 IMAD.WIDE + 17 LOP3.
constexpr uint32_t kPbitsDomain = 0x80000000u;

struct PbitsLane {  // per stream: its id words and the stream-constant round-1 product
  uint32_t s0, s1d, h1, l1;  // s1d = S hi | domain; (h1, l1) = S lo * M1
};

__device__ __forceinline__ PbitsLane pbits_lane(uint32_t s0, uint32_t s1) {
  PbitsLane L;
  L.s0 = s0;
  L.s1d = s1 | kPbitsDomain;
  const uint64_t p = (uint64_t)s0 * kPhiloxM1;
  L.h1 = (uint32_t)(p >> 32);
  L.l1 = (uint32_t)p;
  return L;
}

// The group-shared part of rounds 1-3 of a group's blocks.
struct PbitsPrefix {
  uint32_t base, r1c3, r2c1, q2h, q2l;
};

__device__ __forceinline__ PbitsPrefix pbits_prefix(unsigned long long g, const PbitsLane& L, const PhiloxKeys& K) {
  PbitsPrefix f;
  // round 1 (keys 0, 1): c0 = base ^ j, c1 = l1, c2 = r1c2, c3 = r1c3
  const uint64_t q0 = (uint64_t)(uint32_t)g * kPhiloxM0;
  f.base = L.h1 ^ K.k[0] ^ ((uint32_t)(g >> 32) << 3);
  const uint32_t r1c2 = (uint32_t)(q0 >> 32) ^ K.k[1] ^ L.s1d;
  f.r1c3 = (uint32_t)q0;
  // round 2, shared half: c0' = hi(r1c2 M1) ^ l1 ^ k2, c1' = lo(r1c2 M1)
  const uint64_t q1 = (uint64_t)r1c2 * kPhiloxM1;
  const uint32_t r2c0 = (uint32_t)(q1 >> 32) ^ K.k[2] ^ L.l1;
  f.r2c1 = (uint32_t)q1;
  // round 3, shared product: r2c0 M0
  const uint64_t q2 = (uint64_t)r2c0 * kPhiloxM0;
  f.q2h = (uint32_t)(q2 >> 32);
  f.q2l = (uint32_t)q2;
  return f;
}

// Block j of a group: planes 4j .. 4j+3.
__device__ __forceinline__ void pbits_block(const PbitsPrefix& f, int j, const PhiloxKeys& K, uint32_t (&xs)[4]) {
  // round 2, block half
  const uint64_t pj = (uint64_t)(f.base ^ (uint32_t)j) * kPhiloxM0;
  const uint32_t r2c2 = (uint32_t)(pj >> 32) ^ K.k[3] ^ f.r1c3, r2c3 = (uint32_t)pj;
  // round 3
  const uint64_t p3 = (uint64_t)r2c2 * kPhiloxM1;
  uint32_t x0 = (uint32_t)(p3 >> 32) ^ K.k[4] ^ f.r2c1, x1 = (uint32_t)p3;
  uint32_t x2 = f.q2h ^ K.k[5] ^ r2c3, x3 = f.q2l;
#pragma unroll
  for (int r = 3; r < 10; r++) philox_round(x0, x1, x2, x3, K.k[2 * r], K.k[2 * r + 1]);
  xs[0] = x0; xs[1] = x1; xs[2] = x2; xs[3] = x3;
}

template <int NPMAX>
__device__ __forceinline__ void pbits_group(unsigned long long g, const PbitsLane& L, const PhiloxKeys& K,
                                            const uint32_t (&key)[NPMAX], int np, uint32_t (&acc)[NPMAX]) {
  uint32_t und[NPMAX], any = 0;
#pragma unroll
  for (int p = 0; p < NPMAX; p++) {
    const bool on = p < np && key[p] != 0xFFFFFFFFu && key[p] != 0u;  // K = 2^23 / K = 0: decided
    und[p] = on ? 0xFFFFFFFFu : 0u;
    acc[p] = (p < np && key[p] == 0xFFFFFFFFu) ? 0xFFFFFFFFu : 0u;
    any |= und[p];
  }
  if (!any) return;
  const PbitsPrefix f = pbits_prefix(g, L, K);
#pragma unroll
  for (int j = 0; j < 6; j++) {
    if (j > 0 && !any) break;
    uint32_t xs[4];
    pbits_block(f, j, K, xs);
    any = 0;
#pragma unroll
    for (int p = 0; p < NPMAX; p++) {
#pragma unroll
      for (int e = 0; e < 4; e++) {
        const int b = 4 * j + e;
        if (b < 23) {
          const uint32_t km = key_mask(key[p], b);  // bit 22-b of K, all lanes
          acc[p] |= und[p] & ~xs[e] & km;           // u bit 0, K bit 1: u < K
          und[p] &= ~(xs[e] ^ km);                  // still equal
        }
      }
      any |= und[p];
    }
  }
}

// Flip-time form: only the sites in `und` need a draw; a site in c4 is
// tested against key4 (Delta E = 4|J|), any other against key8 (8|J|).
// Draws 32g + o + i for bit i (o = 0, or 16 for 16-draw rows).  Returns the
// accepted sites among und.  The block loop stays rolled (one copy of the
// ten rounds): it runs inside the flip walk, next to its neighbour words.
// TABLE: the warp shares one pair of keys, and kt holds their bit masks per
// plane, block j at kt[2j] (key4's four planes) and kt[2j+1] (key8's), read
// as shared-memory broadcasts; otherwise every lane shifts its own keys.
template <bool TABLE>
__device__ __forceinline__ uint32_t pbits_accept_sel(unsigned long long g, int o, const PbitsLane& L,
                                                     const PhiloxKeys& K, uint32_t und, uint32_t c4, uint32_t key4,
                                                     uint32_t key8, const uint4* kt) {
  uint32_t acc = 0;
  if (key4 == kKeyAlways) { acc |= und & c4; und &= ~c4; }
  else if (key4 == 0u) und &= ~c4;
  if (key8 == kKeyAlways) { acc |= und & ~c4; und &= c4; }
  else if (key8 == 0u) und &= c4;
  if (!und) return acc;
  const PbitsPrefix f = pbits_prefix(g, L, K);
  // kk4 / kk8: the keys shifted so that the current plane's K bit is bit 31
  uint32_t kk4 = key4, kk8 = key8;
#pragma unroll 1
  for (int j = 0; j < 6 && und; j++) {
    uint32_t xs[4];
    pbits_block(f, j, K, xs);
    uint32_t m4[4], m8[4];
    if (TABLE) {
      const uint4 a = kt[2 * j], b = kt[2 * j + 1];
      m4[0] = a.x; m4[1] = a.y; m4[2] = a.z; m4[3] = a.w;
      m8[0] = b.x; m8[1] = b.y; m8[2] = b.z; m8[3] = b.w;
    }
#pragma unroll
    for (int e = 0; e < 4; e++) {
      const uint32_t x = xs[e] >> o;
      uint32_t km;
      if (TABLE) {
        km = (c4 & m4[e]) | (~c4 & m8[e]);
      } else {
        km = (c4 & (uint32_t)((int32_t)kk4 >> 31)) | (~c4 & (uint32_t)((int32_t)kk8 >> 31));
        kk4 <<= 1;
        kk8 <<= 1;
      }
      const uint32_t live = (j < 5 || e < 3) ? und : 0u;  // plane 23 does not exist
      acc |= live & ~x & km;
      und &= ~(live & (x ^ km));
    }
  }
  return acc;
}

// Accept bits of draws [d0, d0 + L) (1 <= L <= 32) of one stream: bit i =
// draw d0 + i.  Straddles at most two groups.
template <int NPMAX>
__device__ __forceinline__ void pbits_chunk(unsigned long long d0, int L, const PbitsLane& S, const PhiloxKeys& K,
                                            const uint32_t (&key)[NPMAX], int np, uint32_t (&acc)[NPMAX]) {
  const int o = (int)(d0 & 31);
  pbits_group<NPMAX>(d0 >> 5, S, K, key, np, acc);
  if (o) {
#pragma unroll
    for (int p = 0; p < NPMAX; p++) acc[p] >>= o;
    if (o + L > 32) {
      uint32_t hi[NPMAX];
      pbits_group<NPMAX>((d0 >> 5) + 1, S, K, key, np, hi);
#pragma unroll
      for (int p = 0; p < NPMAX; p++) acc[p] |= hi[p] << (32 - o);
    }
  }
  const uint32_t mask = L >= 32 ? 0xFFFFFFFFu : ((1u << L) - 1u);
#pragma unroll
  for (int p = 0; p < NPMAX; p++) acc[p] &= mask;
}

// u23 of draw d (debug / record path): all 23 planes of its group.
__device__ __forceinline__ uint32_t pbits_draw(unsigned long long d, uint32_t s0, uint32_t s1, uint32_t k0,
                                               uint32_t k1) {
  const unsigned long long g = d >> 5;
  const int i = (int)(d & 31);
  uint32_t u = 0;
  for (int j = 0; j < 6; j++) {
    uint32_t x0 = (uint32_t)g, x1 = ((uint32_t)(g >> 32) << 3) | (uint32_t)j, x2 = s0, x3 = s1 | kPbitsDomain;
    philox10(x0, x1, x2, x3, k0, k1);
    const uint32_t xs[4] = {x0, x1, x2, x3};
    for (int e = 0; e < 4; e++) {
      const int b = 4 * j + e;
      if (b < 23) u |= ((xs[e] >> i) & 1u) << (22 - b);
    }
  }
  return u;
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

// Inverse of row_stream: the row of colour X that quarter q of cell gamma's
// stream gates.  Forward quarters (0, 3) gate rows 2(gamma-1) + {0, 1},
// backward quarters (1, 2) rows m-1-2(gamma-1) - {0, 1}.
__device__ __host__ __forceinline__ int seg_row(int m, int gamma, int X, int q) {
  const int g2 = 2 * (gamma - 1);
  switch (q) {
    case 0: return g2 + X;
    case 3: return g2 + 1 - X;
    case 1: return m - 1 - g2 - X;
    default: return m - 1 - g2 - (1 - X);
  }
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

__host__ inline Geo make_geo(const msb_geom* g) {
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
// device: layout conversion helpers (msb_state.cu)
// ---------------------------------------------------------------------------

// 32 x 32 bit transpose across a warp: lane i holds row i (bit j = A[i][j]);
// afterwards lane j holds column j (bit i = A[i][j]).  Five butterfly stages
// swap the off-diagonal blocks of size s = 16, 8, 4, 2, 1 (masks m = low s
// bits of every 2s-bit block).  A lane with bit s clear keeps x & m and takes
// (y << s) & ~m, one with it set keeps x & ~m and takes (y >> s) & m, where y
// is the partner's word: both are a rotation of y (by s, or by 32 - s) whose
// wrapped bits land in the discarded positions, so a stage is SHFL + one
// funnel rotate + one LOP3 select.
__device__ __forceinline__ uint32_t warp_transpose32(uint32_t x) {
  const int lane = threadIdx.x & 31;
  uint32_t m = 0x0000FFFFu;
#pragma unroll
  for (int s = 16; s > 0; s >>= 1, m ^= m << s) {
    const uint32_t y = __shfl_xor_sync(0xFFFFFFFFu, x, s);
    const bool up = (lane & s) != 0;
    const uint32_t keep = up ? ~m : m;
    const uint32_t r = __funnelshift_l(y, y, up ? 32 - s : s);
    x = (x & keep) | (r & ~keep);
  }
  return x;
}

// (replica, held row, chunk) of flat chunk index wg, 32-bit math
__device__ __forceinline__ void chunk_coords(const Geo& G, unsigned wg, int& s, int& lr, int& ch) {
  const unsigned gr = G.nch == 1 ? wg : wg / (unsigned)G.nch;
  ch = (int)(wg - gr * (unsigned)G.nch);
  const unsigned sq = G.rows_div.div(gr);
  s = (int)sq;
  lr = (int)(gr - sq * (unsigned)G.rows);
}

// Linear <-> colour-split for one chunk is a whole-warp 32 x 32 bit transpose:
// the chunk's 32 linear words (1024 sites; lane b holds sites 32b..32b+31,
// bit k = site 32b + k) and its 2 x 16 colour-split words (bit b of word
// (X, t) = site 32b + 2t + p, p = (c+X)&1) are transposes of each other, and
// lane 2t + p holds word t of parity p (k_from_linear / k_export).

}  // namespace msbk
