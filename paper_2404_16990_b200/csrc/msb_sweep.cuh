// Device pieces shared by the per-sweep path (msb_sweep.cu) and the
// lookahead-window path (msb_window.cu): producer constants and work
// counters, the flip pass (FERRO/ANTI chunk flips, generic quads), the grid
// barrier primitive and small host helpers.
#pragma once
#include "msb_common.cuh"

#include <type_traits>

namespace msbk {
namespace {

// draw sources of the producer
constexpr int kSrcXoshiro = 0;  // persistent per-piece reference streams
constexpr int kSrcExt = 1;      // host-supplied u23 draws
constexpr int kSrcPhilox = 2;   // counter-based Philox4x32-10
constexpr int kSrcPbits = 3;    // counter-based Philox4x32-10, bit-plane form (lazy comparisons)

// reference bit t of a uint16 word is gated by draw k = 4(t%4) + t/4 (the
// mapping is its own inverse, engine.py:326-330)
__device__ __forceinline__ int t_of_k(int k) { return 4 * (k & 3) + (k >> 2); }

// n = 512 window planes (FlipArgs::pk16): the planes of k (even) and k + 1,
// t and t + 4 (t = t_of_k(k) in {0..3, 8..11}), share one plane word, and the
// four pairs of each t-half are words 0..3 and 4..7 of the plane row: one
// whole 32-byte sector per plane row, written in full by its piece (a sector
// left half written, words {0..3, 8..11}, was evicted dirty with a byte mask
// and read back by the ECC read-modify-write: 3 GB of DRAM reads per cfg3
// launch).
__device__ __forceinline__ int pk16_word(int k) {
  const int t = t_of_k(k);
  return t - ((t & 8) >> 1);
}

__device__ __forceinline__ size_t plane_off(const Geo& G, int np, int X, int p, int s, int lr) {
  return ((((size_t)X * np + p) * G.n_sim + s) * G.rows + lr) * G.Wp;
}

// Development trace (build with -DMSB_TRACE, tools/trace_producer.py): per
// warp, globaltimer / clock64 stamps at kernel entry, after the table load,
// and at the end of its work, plus SM id and the units it processed.
#ifdef MSB_TRACE
constexpr int kTraceWarps = 148 * 32;
__device__ unsigned long long g_trace[kTraceWarps * 8];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void trace_put(int slot, unsigned long long v) {
  const int w = blockIdx.x * 32 + (threadIdx.x >> 5);
  if ((threadIdx.x & 31) == 0 && w < kTraceWarps) g_trace[w * 8 + slot] = v;
}
#define MSB_TRACE_PUT(slot, v) trace_put(slot, v)
#else
#define MSB_TRACE_PUT(slot, v) ((void)0)
#endif

// Persistent kernel: one 1024-thread CTA per SM shares one copy of the
// sweep-jump table in shared memory; warps claim 32 consecutive pieces at a
// time from a self-resetting counter (work[0] = next unit, work[1] = warps
// done), so SMs stay balanced whatever the piece count.  Each lane runs one
// piece: it generates the piece's draws (k-range x all w) and, spread through
// the generation loop, performs the 64 nibble lookups of its jump to the
// next sweep, so table reads overlap other warps' ALU work.
constexpr int kRngThreads = 1024;
#ifndef MSB_CHUNK_UNROLL
#define MSB_CHUNK_UNROLL 4  // measured: 4 beats 8, 16 (-1.4%), 2 and 32 (spills)
#endif
constexpr int kChunkUnroll = MSB_CHUNK_UNROLL;
// The window producer's 32-draw chunks (n/32 % 32 == 0): unrolled 8 since
// the jump moved after the draws (cfg2 0.966 -> 0.970 T; 16: 0.967)
#ifndef MSB_CHUNK_UNROLL32
#define MSB_CHUNK_UNROLL32 8
#endif
constexpr int kChunkUnroll32 = MSB_CHUNK_UNROLL32;

// Work counters (caller-owned, zeroed once, left zeroed by every kernel):
//   work[0] next dynamic producer unit    work[1] consumer barrier arrivals
//   work[2] warps finished (last one resets all four)
__device__ __forceinline__ void finish_warp(unsigned* work, unsigned total_warps) {
  if ((threadIdx.x & 31) == 0) {
    __threadfence();
    if (atomicAdd(work + 2, 1u) == total_warps - 1) {
      atomicExch(work, 0u);
      atomicExch(work + 1, 0u);
      atomicExch(work + 3, 0u);
      atomicExch(work + 2, 0u);
    }
  }
}

// One producer warp's share of a sweep's accept planes.  `role_warp` /
// `role_warps` number the producer warps of the grid; their first unit is

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
  // slab halo push (fused slab windows, msb_halo): the first / last owned
  // row is also stored into the ghost row of the slab above / below, whose
  // spin buffers (peer memory over NVLink, or this slab itself) have up_R /
  // down_R rows per colour.  Null: no push.
  uint32_t* up_spins;
  uint32_t* down_spins;
  int up_R, down_R;
  // band walk (flip_band_run): rows of QPR <= 32 quads (QPR | 32); a warp
  // group covers band_gb bands of band_h rows, lanes = (band, quad).  0: off.
  int band_h, band_gb;
  int band_sq, band_nseg;  // quads per row segment (divides 32), segments per row
  unsigned band_groups;    // groups per colour phase (all replicas)
  // n = 512 window planes (pk16, pk16_word): plane word t - (t & 8) / 2 of t
  // in {0..3, 8..11} also holds plane t + 4 in its high half (the 32 draws of
  // k and k + 1 are one producer run), so a quad of t0 reads plane words
  // (t0 & 8) / 2 .. + 3, the high halves for t0 = 4, 12
  int pk16;
  // n = 512 packed spin rows inside a window launch (pks, flip_band_run
  // PKS): word j of a row holds the sites of t = tl(j) (low half) and
  // tl(j) + 4 (high half), tl(j) = j (j < 4) or j + 4, of w = bit -- the
  // pairing of the pk16 plane words, so plane word j gates word j without
  // shifts.  The row keeps its 16-word pitch; words 0..7 are used.
  int pks;
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
template <bool GENERIC, bool COHERENT, bool PUSH = false>
__device__ __forceinline__ unsigned flip_quad_at(const FlipArgs& a, int s, int lr, unsigned qq, int X) {
  const Geo& G = a.G;
  const int c = G.row0 + lr, br = lr + G.ghost;
  const int ch = (int)(qq >> 2), t0 = 4 * (int)(qq & 3);
  const int w0 = ch * 16 + t0;
  int bu, bd;
  vert_rows(G, br, bu, bd);
  // 32-bit word offsets (buffers < 2^32 words, checked by check_flip_extent):
  // the 64-bit offset chains were a third of the quad's instructions
  const unsigned R = (unsigned)G.R, Wp = (unsigned)G.Wp;
  const unsigned oth = (unsigned)s * 2u + (unsigned)(1 - X);
  uint32_t* own = a.spins + (((unsigned)s * 2u + (unsigned)X) * R + (unsigned)br) * Wp;
  const uint32_t* yc = a.spins + (oth * R + (unsigned)br) * Wp;
  auto ld4 = [](const uint32_t* q) {
    return COHERENT ? __ldcg(reinterpret_cast<const uint4*>(q)) : __ldg(reinterpret_cast<const uint4*>(q));
  };
  auto ld1 = [](const uint32_t* q) { return COHERENT ? __ldcg(q) : __ldg(q); };
  const uint4 O = *reinterpret_cast<const uint4*>(own + w0);
  const uint4 Y = ld4(yc + w0);
  const uint4 U = ld4(a.spins + ((oth * R + (unsigned)bu) * Wp + (unsigned)w0));
  const uint4 D = ld4(a.spins + ((oth * R + (unsigned)bd) * Wp + (unsigned)w0));
  const unsigned pstride = (unsigned)G.n_sim * (unsigned)G.rows * Wp;
  const uint32_t* pl =
      a.planes + ((((unsigned)X * (unsigned)a.np) * (unsigned)G.n_sim + (unsigned)s) * (unsigned)G.rows +
                  (unsigned)lr) * Wp + (unsigned)w0;
  uint4 P4 = make_uint4(0, 0, 0, 0), P8 = make_uint4(0, 0, 0, 0);
  if (!GENERIC) {
    const int sh = a.pk16 ? (t0 & 4) * 4 : 0;
    const uint32_t* pq = pl - (a.pk16 ? t0 - ((t0 & 8) >> 1) : 0);
    P4 = __ldg(reinterpret_cast<const uint4*>(pq));
    P8 = __ldg(reinterpret_cast<const uint4*>(pq + pstride));
    if (sh) {
      P4.x >>= 16; P4.y >>= 16; P4.z >>= 16; P4.w >>= 16;
      P8.x >>= 16; P8.y >>= 16; P8.z >>= 16; P8.w >>= 16;
    }
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
  const uint4 out = make_uint4(res[0], res[1], res[2], res[3]);
  *reinterpret_cast<uint4*>(own + w0) = out;
  if (PUSH) {
    if (lr == 0)  // our first row is the ghost below of the slab above
      *reinterpret_cast<uint4*>(a.up_spins + (((size_t)s * 2 + X) * a.up_R + a.up_R - 1) * G.Wp + w0) = out;
    if (lr == G.rows - 1)  // our last row is the ghost above of the slab below
      *reinterpret_cast<uint4*>(a.down_spins + ((size_t)s * 2 + X) * a.down_R * G.Wp + w0) = out;
  }
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

// A consumer warp's contiguous run of quads [i0, i1) of one colour, walked
// with incremental (replica, row, quad) bookkeeping: lanes take consecutive
// quads, each step advances all lanes by 32 quads (dr rows + dq quads).
// FERRO/ANTI flip of one colour over band groups [g0, g1) (one warp): each
// lane walks band_h consecutive rows of one quad column.  The other colour's
// rows above and at the current row stay in registers (U, Y), so a step loads
// the row below (D), the own quad (O) and the two plane quads; the horizontal
// neighbour word at the quad edge comes from the lane holding it (shuffle),
// including the one-bit chunk wraps of the interleaved layout.  A row is
// band_nseg segments of band_sq quads (band_sq | 32): lanes = (band, quad of
// the segment); when a row has several segments, the lanes at a segment's
// edges read their outer neighbour word from the row instead (one load).
//
// DIRECT (bit-plane Philox stream, PbitsDirect): no accept planes.  Each
// word's Metropolis tests are decided right here from the neighbour classes:
// sites with >= 2 disagreeing neighbours flip, the others compare their draw
// against the Delta E = 4|J| or 8|J| key, and only those comparisons pull
// bit planes (pbits_accept_sel).  DIRECT = 32: 32-draw rows (n/32 % 32 ==
// 0); 16: n = 512, a word is the low or high half of a group.
struct PbitsDirect {
  const uint32_t* thr9;    // [2][n_sim] keys (FERRO/ANTI)
  PhiloxKeys pk;
  unsigned long long blk;  // stream block of this colour phase (2 per sweep)
};

// L2 prefetch of the accept-plane rows (both planes) of band group g,
// colour X, issued by one lane per band (single-segment rows): the plane
// rows were written a window earlier and live in HBM.
__device__ __forceinline__ void band_prefetch(const FlipArgs& a, unsigned g, int X) {
  const Geo& G = a.G;
  const int lane = threadIdx.x & 31, sq = a.band_sq, bi = lane / sq, q = lane - bi * sq;
  if (q != 0) return;
  const int H = a.band_h, gb = a.band_gb;
  const unsigned Wp = (unsigned)G.Wp, pstride = (unsigned)G.n_sim * (unsigned)G.rows * Wp;
  const unsigned groups_per_sim = (unsigned)G.rows / (unsigned)(gb * H);
  const unsigned s = g / groups_per_sim;
  const int lr0 = (int)(g - s * groups_per_sim) * gb * H + bi * H;
  const uint32_t* pr =
      a.planes + ((((unsigned)X * (unsigned)a.np) * (unsigned)G.n_sim + s) * (unsigned)G.rows + (unsigned)lr0) * Wp;
  const unsigned bytes = (unsigned)H * Wp * 4u;
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(pr), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(pr + pstride), "r"(bytes) : "memory");
}

// The warps' key-mask tables of the direct walk (pbits_accept_sel<true>):
// ONE static shared array per kernel however many walk instantiations it
// inlines (a __shared__ inside the template would be one per instantiation).
__device__ __forceinline__ uint4 (*direct_key_tables())[12] {
  __shared__ uint4 kmt[32][12];
  return kmt;
}

// Per-group hooks of a band run: pre(g) before group g's flips, post(g)
// after them (phase ordering by band-group flags; NoHooks: none).
struct NoHooks {
  __device__ __forceinline__ void pre(unsigned) const {}
  __device__ __forceinline__ void post(unsigned) const {}
};

// PF: prefetch the plane rows of the run's groups one group ahead (callers
// that walk one group at a time prefetch themselves, band_prefetch).
template <bool COHERENT, bool PUSH = false, bool SEG = false, int DIRECT = 0, bool PF = true, class HK = NoHooks,
          bool PK16 = false, bool PKS = false>
__device__ __forceinline__ unsigned flip_band_run(const FlipArgs& a, unsigned g0, unsigned g1, int X,
                                                  const PbitsDirect* dp = nullptr, const HK& hk = HK{}) {
  const Geo& G = a.G;
  const int lane = threadIdx.x & 31;
  const int sq = a.band_sq, nseg = SEG ? a.band_nseg : 1;  // quads per segment, segments per row (SEG: > 1)
  const int H = a.band_h, gb = a.band_gb;        // rows per band, bands per warp (32 / sq)
  const int bi = lane / sq, q = lane - bi * sq, base = bi * sq;
  const int lastbits = chunk_bits(G, G.nch - 1);
  const unsigned Wp = (unsigned)G.Wp;
  const unsigned colour_words = (unsigned)G.R * Wp;  // one colour of one replica
  const unsigned pstride = (unsigned)G.n_sim * (unsigned)G.rows * Wp;
  const unsigned groups_per_sim = (unsigned)G.rows / (unsigned)(gb * H);
  // shuffle sources (fixed per lane): next quad, this chunk's first and last
  // quads, previous quad (the previous chunk's last / the row's last quad)
  const int s_next = base + (q + 1) % sq, s_first = base + (q & ~3), s_last = base + (q | 3),
            s_prev = base + (q + sq - 1) % sq;
  const bool chunk_last = (q & 3) == 3, chunk_first = (q & 3) == 0;
  const bool seg_last = SEG && q == sq - 1, seg_first = SEG && q == 0;
  auto ld4 = [](const uint32_t* p) {
    return COHERENT ? __ldcg(reinterpret_cast<const uint4*>(p)) : __ldg(reinterpret_cast<const uint4*>(p));
  };
  auto ld1 = [](const uint32_t* p) { return COHERENT ? __ldcg(p) : __ldg(p); };
  unsigned cnt = 0;
  // The accept planes were written a window earlier and live in HBM: one
  // lane per band bulk-prefetches the band's plane rows (both planes, H
  // contiguous rows) into L2 one group ahead, so the walk's plane loads hit
  // L2 instead of serialising an HBM round trip per row.
  auto prefetch_band = [&](unsigned g) {
    const unsigned s = g / groups_per_sim;
    const int lr0 = (int)(g - s * groups_per_sim) * gb * H + bi * H;
    const uint32_t* pr =
        a.planes + ((((unsigned)X * (unsigned)a.np) * (unsigned)G.n_sim + s) * (unsigned)G.rows + (unsigned)lr0) * Wp;
    const unsigned bytes = (unsigned)H * Wp * 4u;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(pr), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(pr + pstride), "r"(bytes) : "memory");
  };
  if (PF && !DIRECT && !SEG && q == 0 && g0 < g1) prefetch_band(g0);
  for (unsigned g = g0; g < g1; g++) {
    if (PF && !DIRECT && !SEG && q == 0 && g + 1 < g1) prefetch_band(g + 1);
    hk.pre(g);
    const unsigned gr = SEG ? g / (unsigned)nseg : g;
    const int seg = (int)(g - gr * (unsigned)nseg);
    const unsigned s = gr / groups_per_sim;
    const int lr0 = (int)(gr - s * groups_per_sim) * gb * H + bi * H;  // this lane's band
    const int qg = seg * sq + q;  // quad of the row
    const int ch = qg >> 2, w0 = qg * 4;
    const int vb = chunk_bits(G, ch);
    const uint32_t vm = PKS ? 0xFFFFFFFFu : chunk_mask(G, ch);
    // a segment-edge lane's outer neighbour word, relative to its quad
    const int off_next = (w0 + 4 == (int)Wp ? 0 : w0 + 4) - w0, off_prev = (w0 == 0 ? (int)Wp - 1 : w0 - 1) - w0;
    const uint32_t* ybase = a.spins + (s * 2u + (unsigned)(1 - X)) * colour_words + w0;
    const int br0 = lr0 + G.ghost;
    int bu, bd;
    vert_rows(G, br0, bu, bd);
    uint4 U = ld4(ybase + (unsigned)bu * Wp), Y = ld4(ybase + (unsigned)br0 * Wp);
    // incremental row pointers: the other colour's current row, the own row,
    // the plane rows; the row below wraps only past a whole lattice's last row
    const uint32_t* yrow = ybase + (unsigned)br0 * Wp;
    uint32_t* orow = a.spins + (s * 2u + (unsigned)X) * colour_words + (unsigned)br0 * Wp + w0;
    // PK16 (n = 512 window planes, a.pk16): a quad of t0 reads plane words (t0 & 8) / 2 .., the high halves for t0 = 4, 12
    const bool phi = !PKS && PK16 && a.pk16 && (w0 & 4);
    const uint32_t* prow =
        DIRECT ? nullptr
               : a.planes + ((((unsigned)X * (unsigned)a.np) * (unsigned)G.n_sim + s) * (unsigned)G.rows + (unsigned)lr0) * Wp +
                     (PKS ? w0 : PK16 && a.pk16 ? (w0 & 8) >> 1 : w0);
    uint32_t key4 = 0, key8 = 0;
    bool kuni = false;  // DIRECT: the warp's lanes share one pair of keys (bands of one replica)
    uint4* kt = nullptr;
    if (DIRECT) {
      uint4(*kmt)[12] = direct_key_tables();  // per warp: 6 blocks x (key4, key8) x 4 plane masks
      key4 = dp->thr9[s];
      key8 = dp->thr9[G.n_sim + s];
      kuni = __all_sync(0xFFFFFFFFu, key4 == __shfl_sync(0xFFFFFFFFu, key4, 0) &&
                                         key8 == __shfl_sync(0xFFFFFFFFu, key8, 0));
      kt = kmt[threadIdx.x >> 5];
      if (kuni) {
        __syncwarp();  // the previous group's reads of the table are done
        if (lane < 24) {
          uint32_t* t = reinterpret_cast<uint32_t*>(kt);
          t[(lane >> 2) * 8 + (lane & 3)] = key_mask(key4, lane);
          t[(lane >> 2) * 8 + 4 + (lane & 3)] = key_mask(key8, lane);
        }
        __syncwarp();
      }
    }
    // one row; the parity P of its red sites is a compile-time constant: bands
    // are even-aligned with even H, so rows alternate P, !P from the band's
    // first row and the loop below steps two rows at a time
    auto step = [&](auto PC, int h) {
      constexpr int P = decltype(PC)::value;
      const int lr = lr0 + h, br = br0 + h;
      const uint32_t* drow = br + 1 < G.R ? yrow + Wp : ybase;
      const uint4 D = ld4(drow);
      const uint4 O = *reinterpret_cast<const uint4*>(orow);
      uint4 P4 = make_uint4(0, 0, 0, 0), P8 = P4;
      if (!DIRECT) {
        P4 = __ldg(reinterpret_cast<const uint4*>(prow));
        P8 = __ldg(reinterpret_cast<const uint4*>(prow + pstride));
        if (PK16 && phi) {
          P4.x >>= 16; P4.y >>= 16; P4.z >>= 16; P4.w >>= 16;
          P8.x >>= 16; P8.y >>= 16; P8.z >>= 16; P8.w >>= 16;
        }
      }
      uint32_t edge;
      if (PKS) {
        // packed rows (two lanes, words 0-3 and 4-7).  t + 1: word 3 ->
        // (t 4 = word 0 high, t 8 = word 4 low); word 7 -> (t 12 = word 4
        // high, t 16 = t 0 of w + 1: word 0 low rotated by one bit).  t - 1:
        // word 0 -> (t -1 = t 15 of w - 1: word 7 high rotated, t 3 = word 3
        // low); word 4 -> (t 7 = word 3 high, t 11 = word 7 low)
        if (P) {
          const uint32_t xa = __shfl_sync(0xFFFFFFFFu, Y.x, s_next);
          const uint32_t other = q == 0 ? xa : (((xa & 0xFFFFu) >> 1) | ((xa & 1u) << 15));
          edge = (Y.x >> 16) | (other << 16);
        } else {
          const uint32_t h = __shfl_sync(0xFFFFFFFFu, Y.w, s_prev) >> 16;
          const uint32_t other = q == 0 ? (((h << 1) | (h >> 15)) & 0xFFFFu) : h;
          edge = other | (Y.w << 16);
        }
      } else if (P) {  // word t0+4, or the chunk wrap: (first word >> 1) | (next chunk's bit 0 << vb-1)
        uint32_t xa = __shfl_sync(0xFFFFFFFFu, Y.x, s_next);
        const uint32_t xb = __shfl_sync(0xFFFFFFFFu, Y.x, s_first);
        if (SEG && seg_last) xa = ld1(yrow + off_next);
        edge = chunk_last ? ((xb >> 1) | ((xa & 1u) << (vb - 1))) : xa;
      } else {  // word t0-1, or the chunk wrap: ((last word << 1) | carry) & mask
        uint32_t wa = __shfl_sync(0xFFFFFFFFu, Y.w, s_prev);
        const uint32_t wb = __shfl_sync(0xFFFFFFFFu, Y.w, s_last);
        if (SEG && seg_first) wa = ld1(yrow + off_prev);
        const uint32_t carry = ch > 0 ? (wa >> 31) : ((wa >> (lastbits - 1)) & 1u);
        edge = chunk_first ? (((wb << 1) | carry) & vm) : wa;
      }
      const uint32_t y[4] = {Y.x, Y.y, Y.z, Y.w};
      const uint32_t o[4] = {O.x, O.y, O.z, O.w};
      const uint32_t u4[4] = {U.x, U.y, U.z, U.w};
      const uint32_t d4[4] = {D.x, D.y, D.z, D.w};
      const uint32_t a4[4] = {P4.x, P4.y, P4.z, P4.w};
      const uint32_t a8[4] = {P8.x, P8.y, P8.z, P8.w};
      uint32_t res[4];
      if (DIRECT) {
        // the row's stream and the first draw of this quad's chunk in the phase
        const RowStream rs = row_stream(G.m, G.row0 + lr, X);
        const unsigned long long sid =
            ((unsigned long long)G.sim_offset + s) * (unsigned long long)(G.m / 4) + (unsigned long long)(rs.gamma - 1);
        const PbitsLane L = pbits_lane((uint32_t)sid, (uint32_t)(sid >> 32));
        const unsigned long long nn = (unsigned long long)G.n;
        // word t0 + k of the chunk holds draw index k(t) = 4 k + t0 / 4 of the row's quarter
        unsigned long long d = dp->blk * 2 * nn + (unsigned long long)rs.q * (nn / 2) + 32ull * ch +
                               (unsigned long long)(PKS ? w0 >> 1 : (w0 & 15) >> 2) * (unsigned)G.words;
        const unsigned long long dstep = 4ull * (unsigned)G.words;
        // neighbour classes of the 4 words (static indices), then the draws
        // word by word in a rolled loop over rotating registers
        uint32_t gw[4], cw[4];
#pragma unroll
        for (int k = 0; k < 4; k++) {
          const uint32_t n4 = P ? (k < 3 ? y[k + 1] : edge) : (k > 0 ? y[k - 1] : edge);
          const uint32_t ow = o[k] ^ a.inv;
          const uint32_t x1 = u4[k] ^ ow, x2 = d4[k] ^ ow, x3 = y[k] ^ ow;
          const uint32_t x4 = a.fault ? 0u : (n4 ^ ow);
          const uint32_t o12 = x1 | x2, a12 = x1 & x2, o34 = x3 | x4, a34 = x3 & x4;
          gw[k] = a12 | a34 | (o12 & o34);  // >= 2 disagreeing neighbours: Delta E <= 0
          cw[k] = (o12 | o34) & ~gw[k];    // exactly one: Delta E = 4|J|
        }
        if (DIRECT == 16) {
          // n = 512: the 16 draws of word k (quad lane q, k = 4 kk + q) are
          // one half of a 32-draw group whose other half is word kk of lane
          // q ^ 1.  The lane pair resolves each group once: the even lane
          // groups kk = 0, 1, the odd lane kk = 2, 3, over both halves.
          const bool odd = q & 1;
          uint32_t fo[4];
#pragma unroll
          for (int h = 0; h < 2; h++) {
            const int own = odd ? 2 + h : h;  // static after unrolling both ways below
            const uint32_t u_own = ~(odd ? gw[2 + h] : gw[h]) & vm, c_own = odd ? cw[2 + h] : cw[h];
            const uint32_t u_snd = ~(odd ? gw[h] : gw[2 + h]) & vm, c_snd = odd ? cw[h] : cw[2 + h];
            const uint32_t u_pa = __shfl_xor_sync(0xFFFFFFFFu, u_snd, 1), c_pa = __shfl_xor_sync(0xFFFFFFFFu, c_snd, 1);
            const uint32_t und = odd ? (u_pa | (u_own << 16)) : (u_own | (u_pa << 16));
            const uint32_t c4 = odd ? (c_pa | (c_own << 16)) : (c_own | (c_pa << 16));
            const unsigned long long dg = d + (unsigned long long)own * dstep;
            const uint32_t acc = kuni ? pbits_accept_sel<true>(dg >> 5, 0, L, dp->pk, und, c4, key4, key8, kt)
                                      : pbits_accept_sel<false>(dg >> 5, 0, L, dp->pk, und, c4, key4, key8, kt);
            const uint32_t a_own = odd ? acc >> 16 : acc & 0xFFFFu, a_snd = odd ? acc & 0xFFFFu : acc >> 16;
            const uint32_t a_back = __shfl_xor_sync(0xFFFFFFFFu, a_snd, 1);  // the partner's result for our word
            if (odd) { fo[2 + h] = a_own; fo[h] = a_back; }
            else { fo[h] = a_own; fo[2 + h] = a_back; }
          }
#pragma unroll
          for (int k = 0; k < 4; k++) {
            const uint32_t f = (gw[k] & vm) | fo[k];
            cnt += __popc(f);
            res[k] = o[k] ^ f;
          }
        } else {
        uint32_t g0 = gw[0], g1 = gw[1], g2 = gw[2], g3 = gw[3], q0 = cw[0], q1 = cw[1], q2 = cw[2], q3 = cw[3];
        uint32_t f0 = 0, f1 = 0, f2 = 0, f3 = 0;
#pragma unroll 1
        for (int k = 0; k < 4; k++) {
          const int o16 = DIRECT == 16 ? (int)(d & 16) : 0;
          const uint32_t acc = kuni ? pbits_accept_sel<true>(d >> 5, o16, L, dp->pk, ~g0 & vm, q0, key4, key8, kt)
                                    : pbits_accept_sel<false>(d >> 5, o16, L, dp->pk, ~g0 & vm, q0, key4, key8, kt);
          const uint32_t f = (g0 & vm) | acc;
          cnt += __popc(f);
          g0 = g1; g1 = g2; g2 = g3; q0 = q1; q1 = q2; q2 = q3;
          f0 = f1; f1 = f2; f2 = f3; f3 = f;
          d += dstep;
        }
        res[0] = o[0] ^ f0;
        res[1] = o[1] ^ f1;
        res[2] = o[2] ^ f2;
        res[3] = o[3] ^ f3;
        }
      } else {
#pragma unroll
        for (int k = 0; k < 4; k++) {
          const uint32_t n4 = P ? (k < 3 ? y[k + 1] : edge) : (k > 0 ? y[k - 1] : edge);
          const uint32_t f = flip_word(a, false, o[k], u4[k], d4[k], y[k], n4, nullptr, 0, a4[k], a8[k]) & vm;
          res[k] = o[k] ^ f;
          cnt += __popc(f);
        }
      }
      const uint4 out = make_uint4(res[0], res[1], res[2], res[3]);
      *reinterpret_cast<uint4*>(orow) = out;
      if (PUSH) {
        if (lr == 0)
          *reinterpret_cast<uint4*>(a.up_spins + (((size_t)s * 2 + X) * a.up_R + a.up_R - 1) * Wp + w0) = out;
        if (lr == G.rows - 1)
          *reinterpret_cast<uint4*>(a.down_spins + ((size_t)s * 2 + X) * a.down_R * Wp + w0) = out;
      }
      U = Y;
      Y = D;
      yrow = drow;
      orow += Wp;
      if (!DIRECT) prow += Wp;
    };
    using P0 = std::integral_constant<int, 0>;
    using P1 = std::integral_constant<int, 1>;
    if ((G.row0 + lr0 + X) & 1) {  // warp-uniform
      for (int h = 0; h < H; h += 2) {
        step(P1(), h);
        step(P0(), h + 1);
      }
    } else {
      for (int h = 0; h < H; h += 2) {
        step(P0(), h);
        step(P1(), h + 1);
      }
    }
    hk.post(g);
  }
  return cnt;
}

// Direct sweeps, split form (bands of 2 rows, 32-draw words: whole lattices
// and slabs, rows of one or several segments; PKS: n = 512 packed rows; the
// launches of every such shape use it, MSB_DIRECT_SPLIT=0 builds the walk
// form instead).  flip_band_run<DIRECT>
// resolves each word's tests inside its walk: the block loop of a word runs
// as long as the slowest lane of the warp needs planes (3.1 blocks per word
// slot against a lane mean of 1.9), next to the walk's live neighbour words.
// Here one band group's colour phase is three passes over a per-warp stash in
// shared memory (kSplitWords words per warp):
//   1. classify: each lane's 8 words (2 rows x 4) -> (>= 2 disagreeing
//      neighbours, exactly one) masks into the stash; no draws;
//   2. resolve: per word slot, Philox blocks 0 and 1 for every lane (8
//      planes: warp-uniform, nothing but the stash live); the ~9% of words
//      with tests still open are queued as (lane, slot);
//   3. tail: the queued words one per lane (blocks 2..5, rarely more than
//      one), accepted bits ORed into the owner's stash slot;
// then each lane XORs its 8 flip words into its rows.
constexpr int kSplitWords = 3 * 256 + 64;  // A (sure flips -> flips), B (Delta E = 4|J| sites), C (open tests), queue

//
// SEG: rows in several segments of band_sq quads (cfg4, cfg5): the group is
// (replica s, band l, segment seg), and the lanes at a segment's edges read
// their outer neighbour word from the row.  PUSH: slabs, whose first / last
// row also goes into the neighbour slabs' ghost rows.
template <bool PKS, bool SEG = false, bool PUSH = false>
__device__ __forceinline__ unsigned direct_group_split(const FlipArgs& a, unsigned s, unsigned l, unsigned seg, int X,
                                                       const PbitsDirect& dp, uint32_t* st, int& kt_s) {
  const Geo& G = a.G;
  const int lane = threadIdx.x & 31;
  const int sq = a.band_sq, gb = a.band_gb;
  const int lsq = __ffs(sq) - 1;
  const int bi = lane >> lsq, q = lane & (sq - 1), base = lane - q;
  const unsigned Wp = (unsigned)G.Wp, colour_words = (unsigned)G.R * Wp;
  const int lrg = (int)l * gb * 2;  // the group's first row (band l of replica s)
  const int lr0 = lrg + bi * 2;
  const int qg = SEG ? (int)seg * sq + q : q;  // quad of the row
  const int ch = qg >> 2, w0 = qg * 4;
  const int vb = chunk_bits(G, ch), lastbits = chunk_bits(G, G.nch - 1);
  const uint32_t vm = PKS ? 0xFFFFFFFFu : chunk_mask(G, ch);
  uint32_t* A = st + lane;        // [slot][lane]: sure flips -> flips
  uint32_t* B = st + 256 + lane;  // Delta E = 4|J| sites
  uint32_t* C = st + 512 + lane;  // open tests
  unsigned char* Q = reinterpret_cast<unsigned char*>(st + 768);
  // key masks of the group's replica (per warp, rebuilt when the replica changes)
  uint4(*kmt)[12] = direct_key_tables();
  const uint4* kt = kmt[threadIdx.x >> 5];
  const uint32_t key4 = dp.thr9[s], key8 = dp.thr9[G.n_sim + s];
  if (kt_s != (int)s) {
    __syncwarp();
    if (lane < 24) {
      uint32_t* t = reinterpret_cast<uint32_t*>(kmt[threadIdx.x >> 5]);
      t[(lane >> 2) * 8 + (lane & 3)] = key_mask(key4, lane);
      t[(lane >> 2) * 8 + 4 + (lane & 3)] = key_mask(key8, lane);
    }
    kt_s = (int)s;
  }
  // keys that need no draw (K = 2^23: always, K = 0: never), as masks
  const bool special = key4 == kKeyAlways || key4 == 0u || key8 == kKeyAlways || key8 == 0u;
  const uint32_t al4 = key4 == kKeyAlways ? ~0u : 0u, al8 = key8 == kKeyAlways ? ~0u : 0u;
  const uint32_t dc4 = (key4 == kKeyAlways || key4 == 0u) ? ~0u : 0u, dc8 = (key8 == kKeyAlways || key8 == 0u) ? ~0u : 0u;
  // --- 1. classify ---
  const int s_next = base + ((q + 1) & (sq - 1)), s_first = base + (q & ~3), s_last = base + (q | 3),
            s_prev = base + ((q + sq - 1) & (sq - 1));
  const bool chunk_last = (q & 3) == 3, chunk_first = (q & 3) == 0;
  const uint32_t* ybase = a.spins + (s * 2u + (unsigned)(1 - X)) * colour_words + w0;
  uint32_t* orow = a.spins + (s * 2u + (unsigned)X) * colour_words + (unsigned)(lr0 + G.ghost) * Wp + w0;
  uint32_t anyund = 0;
  {
    const int br0 = lr0 + G.ghost;
    int bu, bd;
    vert_rows(G, br0, bu, bd);
    auto ld4 = [](const uint32_t* p) { return __ldcg(reinterpret_cast<const uint4*>(p)); };
    const uint4 U = ld4(ybase + (unsigned)bu * Wp), Y0 = ld4(ybase + (unsigned)br0 * Wp),
                Y1 = ld4(ybase + (unsigned)(br0 + 1) * Wp),
                D1 = ld4(br0 + 2 < G.R ? ybase + (unsigned)(br0 + 2) * Wp : ybase);
    const uint4 O0 = *reinterpret_cast<const uint4*>(orow), O1 = *reinterpret_cast<const uint4*>(orow + Wp);
    // SEG: a segment-edge lane's outer neighbour word of each row (the word
    // after the segment for a row of parity 1, the word before it for 0)
    const bool p0 = ((G.row0 + lr0 + X) & 1) != 0;
    const bool seg_last = SEG && q == sq - 1, seg_first = SEG && q == 0;
    uint32_t e0 = 0, e1 = 0;
    if (SEG) {
      const int off_next = (w0 + 4 == (int)Wp ? 0 : w0 + 4) - w0, off_prev = (w0 == 0 ? (int)Wp - 1 : w0 - 1) - w0;
      const uint32_t* y0 = ybase + (unsigned)br0 * Wp;
      if (p0 ? seg_last : seg_first) e0 = __ldcg(y0 + (p0 ? off_next : off_prev));
      if (p0 ? seg_first : seg_last) e1 = __ldcg(y0 + Wp + (p0 ? off_prev : off_next));
    }
    auto classify = [&](auto PC, const uint4& Uq, const uint4& Yq, const uint4& Dq, const uint4& Oq, int slot0,
                        uint32_t eo) {
      constexpr int P = decltype(PC)::value;
      uint32_t edge;
      if (PKS) {
        if (P) {
          const uint32_t xa = __shfl_sync(0xFFFFFFFFu, Yq.x, s_next);
          const uint32_t other = q == 0 ? xa : (((xa & 0xFFFFu) >> 1) | ((xa & 1u) << 15));
          edge = (Yq.x >> 16) | (other << 16);
        } else {
          const uint32_t h = __shfl_sync(0xFFFFFFFFu, Yq.w, s_prev) >> 16;
          const uint32_t other = q == 0 ? (((h << 1) | (h >> 15)) & 0xFFFFu) : h;
          edge = other | (Yq.w << 16);
        }
      } else if (P) {
        uint32_t xa = __shfl_sync(0xFFFFFFFFu, Yq.x, s_next);
        const uint32_t xb = __shfl_sync(0xFFFFFFFFu, Yq.x, s_first);
        if (SEG && seg_last) xa = eo;
        edge = chunk_last ? ((xb >> 1) | ((xa & 1u) << (vb - 1))) : xa;
      } else {
        uint32_t wa = __shfl_sync(0xFFFFFFFFu, Yq.w, s_prev);
        const uint32_t wb = __shfl_sync(0xFFFFFFFFu, Yq.w, s_last);
        if (SEG && seg_first) wa = eo;
        const uint32_t carry = ch > 0 ? (wa >> 31) : ((wa >> (lastbits - 1)) & 1u);
        edge = chunk_first ? (((wb << 1) | carry) & vm) : wa;
      }
      const uint32_t y[4] = {Yq.x, Yq.y, Yq.z, Yq.w}, o[4] = {Oq.x, Oq.y, Oq.z, Oq.w};
      const uint32_t u4[4] = {Uq.x, Uq.y, Uq.z, Uq.w}, d4[4] = {Dq.x, Dq.y, Dq.z, Dq.w};
#pragma unroll
      for (int k = 0; k < 4; k++) {
        const uint32_t n4 = P ? (k < 3 ? y[k + 1] : edge) : (k > 0 ? y[k - 1] : edge);
        const uint32_t ow = o[k] ^ a.inv;
        const uint32_t x1 = u4[k] ^ ow, x2 = d4[k] ^ ow, x3 = y[k] ^ ow;
        const uint32_t x4 = a.fault ? 0u : (n4 ^ ow);
        const uint32_t o12 = x1 | x2, a12 = x1 & x2, o34 = x3 | x4, a34 = x3 & x4;
        const uint32_t ge2 = a12 | a34 | (o12 & o34);
        const uint32_t c4 = (o12 | o34) & ~ge2;
        uint32_t sure = ge2 & vm, und = ~ge2 & vm;
        if (special) {  // warp-uniform
          sure |= und & ((c4 & al4) | (~c4 & al8));
          und &= ~((c4 & dc4) | (~c4 & dc8));
        }
        A[(slot0 + k) * 32] = sure;
        B[(slot0 + k) * 32] = c4;
        C[(slot0 + k) * 32] = und;
        anyund |= und;
      }
    };
    using P0 = std::integral_constant<int, 0>;
    using P1 = std::integral_constant<int, 1>;
    if (p0) {  // warp-uniform
      classify(P1(), U, Y0, Y1, O0, 0, e0);
      classify(P0(), Y0, Y1, D1, O1, 4, e1);
    } else {
      classify(P0(), U, Y0, Y1, O0, 0, e0);
      classify(P1(), Y0, Y1, D1, O1, 4, e1);
    }
  }
  __syncwarp();  // the key table
  const unsigned long long nn = (unsigned long long)G.n;
  const unsigned long long dphase = dp.blk * 2 * nn;
  const unsigned dstep = 4u * (unsigned)G.words;
  const unsigned long long simbase = ((unsigned long long)G.sim_offset + s) * (unsigned long long)(G.m / 4);
  if (__any_sync(0xFFFFFFFFu, anyund != 0u)) {
    // --- 2. resolve: blocks 0 and 1 of every word slot (no control flow
    // inside a row, so the slots' Philox chains interleave) ---
    uint32_t om = 0;  // this lane's slots with tests still open
#pragma unroll 1
    for (int h = 0; h < 2; h++) {
      const RowStream rs = row_stream(G.m, G.row0 + lr0 + h, X);
      const unsigned long long sid = simbase + (unsigned long long)(rs.gamma - 1);
      const PbitsLane L = pbits_lane((uint32_t)sid, (uint32_t)(sid >> 32));
      const unsigned long long d0 =
          dphase + (unsigned long long)((unsigned)rs.q * (unsigned)(G.n / 2) + 32u * (unsigned)ch +
                                        (unsigned)(PKS ? w0 >> 1 : (w0 & 15) >> 2) * (unsigned)G.words);
      uint32_t* Ah = A + h * 128;
      uint32_t* Bh = B + h * 128;
      uint32_t* Ch = C + h * 128;
#pragma unroll
      for (int kk = 0; kk < 4; kk++) {
        const uint32_t c4 = Bh[kk * 32];
        uint32_t und = Ch[kk * 32], acc = 0;
        const PbitsPrefix f = pbits_prefix((d0 + (unsigned long long)kk * dstep) >> 5, L, dp.pk);
#pragma unroll
        for (int j = 0; j < 2; j++) {
          uint32_t xs[4];
          pbits_block(f, j, dp.pk, xs);
          const uint4 ma = kt[2 * j], mb = kt[2 * j + 1];
          const uint32_t m4[4] = {ma.x, ma.y, ma.z, ma.w}, m8[4] = {mb.x, mb.y, mb.z, mb.w};
#pragma unroll
          for (int e = 0; e < 4; e++) {
            const uint32_t km = (c4 & m4[e]) | (~c4 & m8[e]);
            acc |= und & ~xs[e] & km;
            und &= ~(xs[e] ^ km);
          }
        }
        Ah[kk * 32] |= acc;
        if (und) {
          Ch[kk * 32] = und;
          om |= 1u << (h * 4 + kk);
        }
      }
    }
    // --- 3. tail: the words with tests still open after 8 planes, queued
    // as (lane, slot) and finished one per lane ---
    const unsigned nopen = __popc(om);
    unsigned off = nopen;  // inclusive scan over the lanes
#pragma unroll
    for (int dlt = 1; dlt < 32; dlt <<= 1) {
      const unsigned t = __shfl_up_sync(0xFFFFFFFFu, off, dlt);
      if (lane >= dlt) off += t;
    }
    const unsigned qn = __shfl_sync(0xFFFFFFFFu, off, 31);
    if (qn) {
      off -= nopen;
      for (uint32_t m = om; m; m &= m - 1) Q[off++] = (unsigned char)(lane | ((__ffs(m) - 1) << 5));
      __syncwarp();
      for (unsigned i = lane; i < qn; i += 32) {
        const unsigned e = Q[i], sl = e & 31u, k = e >> 5;
        uint32_t und = st[512 + k * 32 + sl];
        const uint32_t c4 = st[256 + k * 32 + sl];
        const int q2 = (int)(sl & (unsigned)(sq - 1)) + (SEG ? (int)seg * sq : 0), w02 = q2 * 4;
        const int row = lrg + (int)(sl >> lsq) * 2 + (int)(k >> 2);
        const RowStream rs = row_stream(G.m, G.row0 + row, X);
        const unsigned long long sid = simbase + (unsigned long long)(rs.gamma - 1);
        const PbitsLane L = pbits_lane((uint32_t)sid, (uint32_t)(sid >> 32));
        const unsigned long long d =
            dphase + (unsigned long long)((unsigned)rs.q * (unsigned)(G.n / 2) + 32u * (unsigned)(q2 >> 2) +
                                          (unsigned)(PKS ? w02 >> 1 : (w02 & 15) >> 2) * (unsigned)G.words +
                                          (k & 3u) * dstep);
        const PbitsPrefix f = pbits_prefix(d >> 5, L, dp.pk);
        uint32_t acc = 0;
#pragma unroll 1
        for (int j = 2; j < 6 && und; j++) {
          uint32_t xs[4];
          pbits_block(f, j, dp.pk, xs);
          const uint4 ma = kt[2 * j], mb = kt[2 * j + 1];
          const uint32_t m4[4] = {ma.x, ma.y, ma.z, ma.w}, m8[4] = {mb.x, mb.y, mb.z, mb.w};
#pragma unroll
          for (int e2 = 0; e2 < 4; e2++) {
            const uint32_t km = (c4 & m4[e2]) | (~c4 & m8[e2]);
            const uint32_t live = (j < 5 || e2 < 3) ? und : 0u;  // plane 23 does not exist
            acc |= live & ~xs[e2] & km;
            und &= ~(live & (xs[e2] ^ km));
          }
        }
        if (acc) st[k * 32 + sl] |= acc;
      }
      __syncwarp();
    }
  }
  // --- flips into the rows ---
  unsigned cnt = 0;
#pragma unroll
  for (int h = 0; h < 2; h++) {
    const uint4 O = *reinterpret_cast<const uint4*>(orow + h * Wp);
    const uint32_t f0 = A[(h * 4 + 0) * 32], f1 = A[(h * 4 + 1) * 32], f2 = A[(h * 4 + 2) * 32],
                   f3 = A[(h * 4 + 3) * 32];
    cnt += __popc(f0) + __popc(f1) + __popc(f2) + __popc(f3);
    const uint4 out = make_uint4(O.x ^ f0, O.y ^ f1, O.z ^ f2, O.w ^ f3);
    *reinterpret_cast<uint4*>(orow + h * Wp) = out;
    if (PUSH) {
      if (lr0 + h == 0)  // our first row is the ghost below of the slab above
        *reinterpret_cast<uint4*>(a.up_spins + (((size_t)s * 2 + X) * a.up_R + a.up_R - 1) * Wp + w0) = out;
      if (lr0 + h == G.rows - 1)  // our last row is the ghost above of the slab below
        *reinterpret_cast<uint4*>(a.down_spins + ((size_t)s * 2 + X) * a.down_R * Wp + w0) = out;
    }
  }
  return cnt;
}

template <bool COHERENT, bool PUSH = false>
__device__ __forceinline__ unsigned flip_run(const FlipArgs& a, unsigned i0, unsigned i1, int X) {
  const Geo& G = a.G;
  const unsigned quads = (unsigned)G.Wp >> 2;
  if (i0 >= i1) return 0;
  unsigned gr = G.quads_div.div(i0), qq = i0 - gr * quads;
  int s = (int)G.rows_div.div(gr), lr = (int)(gr - (unsigned)s * G.rows);
  const unsigned dr = G.quads_div.div(32u), dq = 32u - dr * quads;
  unsigned cnt = 0;
  for (unsigned i = i0; i < i1; i += 32) {
    cnt += flip_quad_at<false, COHERENT, PUSH>(a, s, lr, qq, X);
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

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <typename K>
int set_smem_attr(K kernel, std::once_flag& once, cudaError_t& err) {
  std::call_once(once, [&] {
    cudaFuncAttributes fa = {};  // the 227 KiB per CTA include the kernel's static shared memory
    err = cudaFuncGetAttributes(&fa, kernel);
    if (err == cudaSuccess)
      err = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 227 * 1024 - (int)fa.sharedSizeBytes);
  });
  if (err != cudaSuccess) return fail(MSB_ERR_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(err));
  return MSB_OK;
}

inline void fill_flip_args(FlipArgs& a, const msb_geom* g, const msb_sweep_params* p, int colour, uint32_t* spins,
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
  a.up_spins = a.down_spins = nullptr;
  a.up_R = a.down_R = 0;
  // band walk geometry: lanes cover row segments of SQ quads (SQ | 32, the
  // largest power of two dividing the row's quads: a whole row when it has
  // at most 32), bands of H rows never cross a replica (H | rows / gb), H
  // even (uniform parity)
  a.band_h = a.band_gb = 0;
  a.band_sq = a.band_nseg = 0;
  a.band_groups = 0;
  a.pk16 = 0;
  a.pks = 0;
  const int qpr = a.G.Wp / 4;  // 4 * chunks: a multiple of 4
  if (p->mode != MSB_MODE_GENERIC) {
    int sq = 32;
    while (sq > 4 && qpr % sq) sq >>= 1;
    if (qpr < sq) sq = qpr;
    const int gb = 32 / sq, nseg = qpr / sq;
    for (int h = 16; h >= 2; h >>= 1)
      if (g->rows % (gb * h) == 0) {
        a.band_h = h;
        a.band_gb = gb;
        a.band_sq = sq;
        a.band_nseg = nseg;
        a.band_groups = (unsigned)((long long)g->n_sim * g->rows / (gb * h) * nseg);
        break;
      }
  }
}

// Flip warps per 32-warp CTA of a fused launch: 6 measured best for
// flip-heavy shapes (cfg3/cfg4); fewer when that keeps every producer warp
// to one unit on single-round problems (cfg2).  MSB_FLIP_WARPS overrides.
inline int flip_warps_for(long long units) {
  static const int env_cw = [] { const char* e = getenv("MSB_FLIP_WARPS"); return e ? atoi(e) : 0; }();
  if (env_cw > 0) return std::min(28, env_cw);
  int cw = 6;
  const int sms_est = 148;
  auto rounds = [&](int c) { return (units + (long long)sms_est * (32 - c) - 1) / ((long long)sms_est * (32 - c)); };
  if (rounds(2) == 1)
    while (cw > 2 && rounds(cw) > 1) cw--;
  return cw;
}


// One colour's flip pass as its own launch: a thread per 4-word quad.
template <bool GENERIC>
__global__ void __launch_bounds__(256) k_flip(const FlipArgs a) {
  const unsigned quads = (unsigned)a.G.Wp >> 2;
  const unsigned total = (unsigned)a.G.n_sim * (unsigned)a.G.rows * quads;
  const unsigned i = blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned cnt = i < total ? flip_quad<GENERIC, false>(a, i, a.X) : 0u;
  add_flips(a.flips, cnt);
}

// The flip path indexes spins and planes with 32-bit word offsets.
inline int check_flip_extent(const msb_geom* g, int n_planes) {
  const Geo G = make_geo(g);
  const long long spin_words = (long long)G.n_sim * 2 * G.R * G.Wp;
  const long long plane_words = 2LL * std::max(n_planes, 1) * G.n_sim * G.rows * G.Wp;
  if (spin_words >= (1LL << 32) || plane_words >= (1LL << 32))
    return fail(MSB_ERR_UNSUPPORTED, "spin or plane buffer of 2^32 words or more: split the replicas");
  return MSB_OK;
}

// Launch k_flip for colour `colour` of planes `planes`.
inline int flip(const msb_geom* g, const msb_sweep_params* p, int colour, uint32_t* spins, const uint32_t* planes,
         uint64_t* flips, cudaStream_t st) {
  if (int r = check_flip_extent(g, p->n_planes)) return r;
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

}  // namespace
}  // namespace msbk
