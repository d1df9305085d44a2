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
#include "msb_sweep.cuh"
#include "msb_io.cuh"

namespace msbk {
namespace {

struct WinArgs {
  Geo G;
  uint32_t* states;        // [8][npieces] piece start states (xoshiro)
  const uint32_t* thr9;    // [2][n_sim] keys (FERRO/ANTI)
  const uint4* jump;       // nibble table of A^(S*4n)
  uint32_t* planes;        // window buffer being produced
  unsigned* work;
  long long npieces;       // S * P * streams
  size_t slot_words;       // plane words of one sweep (both colours, both planes)
  int S, P, pshift, kg, kr, nseg, streams, kit;
  FastDiv streams_div, cells_div, sims_div;
  uint32_t seed_lo, seed_hi;    // Philox key
  unsigned long long block0;    // stream block of slot 0's first phase
  PhiloxKeys pk;                // Philox round keys
  unsigned* gflags;             // direct sweeps: per band group, phases completed (monotonic), or null
  unsigned gphase0;             // gflags value every group holds at launch start
};

// Direct sweeps with band-group flags instead of grid barriers: a group's
// phase i reads the other colour's rows of its own group and of the groups
// just above and below (same replica, periodic), and overwrites rows those
// groups read in phase i-1.  So it waits for both neighbours to have
// completed phase i-1, and publishes its own completion; slow groups delay
// only their neighbours instead of the whole grid.
__device__ __forceinline__ void group_wait(const unsigned* flags, unsigned g, unsigned gps, unsigned need) {
  if ((threadIdx.x & 31) == 0) {
    const unsigned s0 = g - g % gps, l = g - s0;
    const unsigned up = s0 + (l == 0 ? gps - 1 : l - 1), dn = s0 + (l + 1 == gps ? 0 : l + 1);
    while (ld_acquire(flags + up) < need || ld_acquire(flags + dn) < need) __nanosleep(32);
  }
  __syncwarp();
}

__device__ __forceinline__ void group_done(unsigned* flags, unsigned g, unsigned v) {
  __syncwarp();
  if ((threadIdx.x & 31) == 0) {
    __threadfence();
    atomicExch(flags + g, v);
  }
}

// One 32-bit word of the jump: 8 nibble lookups (paired 3-input XORs) from the
// piece's start state, consumed 4 bits at a time (jw0 is the current word).
__device__ __forceinline__ void jump_word(const uint4* __restrict__ jt, int& nib, uint32_t (&jw)[8],
                                          uint32_t (&r)[8]) {
  const char* e = reinterpret_cast<const char*>(jt) + nib * 512;
  const uint32_t w = jw[0];
#pragma unroll
  for (int j = 0; j < 8; j += 2) {
    // entry (position nib+j, value v) lives at byte (nib+j)*512 + v*32
    const uint32_t oa = j == 0 ? ((w << 5) & 0x1E0u) : ((w >> (4 * j - 5)) & 0x1E0u);
    const uint32_t ob = j == 0 ? ((w << 1) & 0x1E0u) : ((w >> (4 * j - 1)) & 0x1E0u);
    const uint4* ea = reinterpret_cast<const uint4*>(e + j * 512 + oa);
    const uint4* eb = reinterpret_cast<const uint4*>(e + (j + 1) * 512 + ob);
    const uint4 la = ea[0], ha = ea[1], lb = eb[0], hb = eb[1];
    r[0] = xor3(r[0], la.x, lb.x); r[1] = xor3(r[1], la.y, lb.y);
    r[2] = xor3(r[2], la.z, lb.z); r[3] = xor3(r[3], la.w, lb.w);
    r[4] = xor3(r[4], ha.x, hb.x); r[5] = xor3(r[5], ha.y, hb.y);
    r[6] = xor3(r[6], ha.z, hb.z); r[7] = xor3(r[7], ha.w, hb.w);
  }
  nib += 8;
#pragma unroll
  for (int i = 0; i < 7; i++) jw[i] = jw[i + 1];
}

// Draws of one k of one quarter-segment (all w, in chunks of 32) reduced to
// the two accept planes.  out points at word t(k) of the row's first plane.
// Philox: draw d of stream id (st.a1:st.a0) is word d&3 of block (d>>2, id);
// pd is the stream draw index of this k's first draw.
template <int SRC, int CB>
__device__ __forceinline__ void win_segment_k(const WinArgs& a, XState& st, const PbitsLane& pl, uint32_t* outk,
                                              uint32_t key0, uint32_t key1, size_t pstride, unsigned long long pd) {
  const Geo& G = a.G;
  if (SRC == kSrcPbits) {  // accept bits straight from the bit planes (bit i = draw i)
    const uint32_t key[2] = {key0, key1};
    for (int ch = 0; ch < G.nch; ch++) {
      uint32_t acc[2];
      if (CB == 32) pbits_group<2>((pd >> 5) + ch, pl, a.pk, key, 2, acc);
      else pbits_chunk<2>(pd + 32ull * ch, CB ? CB : chunk_bits(G, ch), pl, a.pk, key, 2, acc);
      outk[ch * 16] = acc[0];
      outk[pstride + ch * 16] = acc[1];
    }
    return;
  }
  for (int ch = 0; ch < G.nch; ch++) {
    const int L = CB ? CB : chunk_bits(G, ch);  // CB: compile-time chunk width (32, 16) or 0
    uint32_t acc0 = 0, acc1 = 0;
    if (SRC == kSrcXoshiro) {
      if (L == 32) {
#pragma unroll kChunkUnroll
        for (int i = 0; i < 32; i++) {
          const uint32_t h9 = xstep(st) << 9;
          acc_reject(acc0, h9, key0);
          acc_reject(acc1, h9, key1);
        }
      } else if (CB == 16) {  // n = 512: one 16-draw chunk per k
#pragma unroll
        for (int i = 0; i < 16; i++) {
          const uint32_t h9 = xstep(st) << 9;
          acc_reject(acc0, h9, key0);
          acc_reject(acc1, h9, key1);
        }
      } else {
        for (int i = 0; i < L; i++) {
          const uint32_t h9 = xstep(st) << 9;
          acc_reject(acc0, h9, key0);
          acc_reject(acc1, h9, key1);
        }
      }
    } else {
      const unsigned long long d0 = pd + 32ull * ch;
      if ((d0 & 3) == 0 && (L & 3) == 0) {
#pragma unroll 1  // one block in flight per thread measured best (register pressure)
        for (int i = 0; i < L; i += 4) {
          const unsigned long long c = (d0 + i) >> 2;
          uint32_t x0 = (uint32_t)c, x1 = (uint32_t)(c >> 32), x2 = st.a0, x3 = st.a1;
          philox10k(x0, x1, x2, x3, a.pk);
          const uint32_t xs[4] = {x0, x1, x2, x3};
#pragma unroll
          for (int q = 0; q < 4; q++) {
            const uint32_t h9 = xs[q] << 9;
            acc_reject(acc0, h9, key0);
            acc_reject(acc1, h9, key1);
          }
        }
      } else {
        for (int i = 0; i < L; i++) {
          const unsigned long long d = d0 + i, c = d >> 2;
          uint32_t x0 = (uint32_t)c, x1 = (uint32_t)(c >> 32), x2 = st.a0, x3 = st.a1;
          philox10k(x0, x1, x2, x3, a.pk);
          const int e = (int)(d & 3);
          const uint32_t h9 = (e == 0 ? x0 : e == 1 ? x1 : e == 2 ? x2 : x3) << 9;
          acc_reject(acc0, h9, key0);
          acc_reject(acc1, h9, key1);
        }
      }
    }
    // acc holds REJECT bits, newest draw in bit 0: reverse and invert
    if (CB == 32) {
      outk[ch * 16] = ~__brev(acc0);
      outk[pstride + ch * 16] = ~__brev(acc1);
    } else {
      outk[ch * 16] = (~__brev(acc0)) >> (32 - L);
      outk[pstride + ch * 16] = (~__brev(acc1)) >> (32 - L);
    }
  }
}

// Piece numbering.
//  P < 8 (whole lattices; a piece = 8/P whole quarter-segments of a stream):
//    gi = (j * P + p) * streams + stream -- a warp's lanes share (j, p), the
//    same segments, across 32 consecutive streams.
//  P >= 8 (a piece = 16/kg k-values of ONE quarter-segment, i.e. one row of
//  one colour; kg = P/8):  gi = (((j * n_sim + s) * 2 + X) * rows + lr) * kg
//    + kgi over the HELD rows lr -- so a slab generates exactly its own rows,
//    the kg parts of a row sit in adjacent lanes and a warp's plane stores
//    land in 32/kg adjacent rows.
struct WinPiece {
  int j, s, gamma, seg, k0, lr;  // lr: plane row (held-row index); seg = 4 X + q
};

__device__ __forceinline__ WinPiece win_piece(const WinArgs& a, unsigned gi) {
  const Geo& G = a.G;
  WinPiece w;
  if (a.P < 8) {
    const unsigned jp = a.streams_div.div(gi);
    const int sti = (int)(gi - jp * (unsigned)a.streams);
    w.j = (int)(jp >> a.pshift);
    w.seg = (int)(jp & (unsigned)(a.P - 1)) * a.nseg;
    w.k0 = 0;
    w.s = (int)a.cells_div.div((unsigned)sti);
    w.gamma = sti - w.s * (G.m / 4) + 1;
    w.lr = -1;  // per segment (seg_row)
  } else {
    const int kgs = a.pshift - 3;
    const unsigned t = gi >> kgs;
    const unsigned q1 = G.rows_div.div(t);
    w.lr = (int)(t - q1 * (unsigned)G.rows);
    const int X = (int)(q1 & 1u);
    const unsigned q2 = q1 >> 1;
    const unsigned jj = a.sims_div.div(q2);
    w.j = (int)jj;
    w.s = (int)(q2 - jj * (unsigned)G.n_sim);
    const RowStream rs = row_stream(G.m, G.row0 + w.lr, X);
    w.gamma = rs.gamma;
    w.seg = 4 * X + rs.q;
    w.k0 = (int)(gi & (unsigned)(a.kg - 1)) * a.kr;
  }
  return w;
}

// One producer warp's share of a window (pieces numbered as win_piece).
template <int SRC, int CB>
__device__ __forceinline__ void win_produce(const WinArgs& a, const uint4* __restrict__ jt, int role_warp,
                                            int role_warps) {
  constexpr bool XO = SRC == kSrcXoshiro;
  const Geo& G = a.G;
  const int lane = threadIdx.x & 31;
  const long long units = (a.npieces + 31) / 32;
  const size_t pstride = (size_t)G.n_sim * G.rows * G.Wp;
  const long long nwarps = (long long)role_warps * gridDim.x;
  const int cells = G.m / 4;
  const unsigned long long n = (unsigned long long)G.n;
  long long u = (long long)role_warp * gridDim.x + blockIdx.x;
  for (;;) {
    if (u >= units) break;
    const long long gi = u * 32 + lane;
    if (gi < a.npieces) {
      const WinPiece w = win_piece(a, (unsigned)gi);
      const uint32_t key0 = a.thr9[w.s], key1 = a.thr9[G.n_sim + w.s];
      uint32_t* slot = a.planes + (size_t)w.j * a.slot_words;
      XState st;
      PbitsLane pl = {0, 0, 0, 0};
      uint32_t jw[8] = {0, 0, 0, 0, 0, 0, 0, 0}, r[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      int nib = 0, jacc = 0;
      if (XO) {
        load_state(st, a.states, a.npieces, gi);
        jw[0] = st.a0; jw[1] = st.a1; jw[2] = st.b0; jw[3] = st.b1;
        jw[4] = st.c0; jw[5] = st.c1; jw[6] = st.d0; jw[7] = st.d1;
      } else {  // Philox: the stream id rides in st.a0 / st.a1
        const unsigned long long sid =
            ((unsigned long long)G.sim_offset + (unsigned long long)w.s) * cells + w.gamma - 1;
        st.a0 = (uint32_t)sid;
        st.a1 = (uint32_t)(sid >> 32);
        if (SRC == kSrcPbits) pl = pbits_lane(st.a0, st.a1);
      }
      for (int sg = 0; sg < a.nseg; sg++) {
        const int seg = w.seg + sg, X = seg >> 2, q = seg & 3;
        const int lr = w.lr >= 0 ? w.lr : seg_row(G.m, w.gamma, X, q);
        uint32_t* out = slot + plane_off(G, 2, X, 0, w.s, lr);
        const unsigned long long pseg = (a.block0 + 2ull * w.j + X) * 2 * n + (unsigned long long)q * (n / 2);
        if (SRC == kSrcPbits && CB == 16 && !(a.kr & 1)) {
          // n = 512: one bit-plane group is the 16 draws of k (even) and of
          // k + 1 -- resolve it once for both rows of plane words
          const uint32_t key[2] = {key0, key1};
          for (int kk = 0; kk < a.kr; kk += 2) {
            const int k = w.k0 + kk;
            uint32_t acc[2];
            pbits_group<2>((pseg + (unsigned long long)k * 16) >> 5, pl, a.pk, key, 2, acc);
            out[t_of_k(k)] = acc[0] & 0xFFFFu;
            out[pstride + t_of_k(k)] = acc[1] & 0xFFFFu;
            out[t_of_k(k + 1)] = acc[0] >> 16;
            out[pstride + t_of_k(k + 1)] = acc[1] >> 16;
          }
          continue;
        }
        for (int kk = 0; kk < a.kr; kk++) {
          const int k = w.k0 + kk;
          win_segment_k<SRC, CB>(a, st, pl, out + t_of_k(k), key0, key1, pstride,
                                   pseg + (unsigned long long)k * G.words);
          if (XO) {  // the 8 jump words, spread evenly over the piece's kit k-iterations
            jacc += 8;
            while (jacc >= a.kit) {
              jacc -= a.kit;
              jump_word(jt, nib, jw, r);
            }
          }
        }
      }
      if (XO) {
        XState nx;
        nx.a0 = r[0]; nx.a1 = r[1]; nx.b0 = r[2]; nx.b1 = r[3];
        nx.c0 = r[4]; nx.c1 = r[5]; nx.d0 = r[6]; nx.d1 = r[7];
        store_state(nx, a.states, a.npieces, gi);  // same piece, next window
      }
    }
    long long nu = 0;
    if (lane == 0) nu = nwarps + (long long)atomicAdd(a.work, 1u);
    u = __shfl_sync(0xFFFFFFFFu, nu, 0);
  }
}

// Grid barrier among the consumer warps: a named CTA barrier (id 1, the
// consumer warps only), one arrival per CTA on the counter, the CTA leader
// spins until all CTAs arrived, a second named barrier releases the CTA.
__device__ __forceinline__ void consumer_barrier(unsigned* ctr, unsigned target, int nthreads, bool leader) {
  asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
  if (leader) {
    __threadfence();
    atomicAdd(ctr, 1u);
    while (ld_acquire(ctr) < target) __nanosleep(64);
    __threadfence();
  }
  asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}

__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

struct HaloArgs {
  unsigned *up_flags, *down_flags, *my_flags;
  unsigned long long phase0;
  int on;
};

// Slab-window phase gate (msb_halo).  Ends local phase i (i = -1: launch
// start) and opens phase i+1 when `open`.  All consumer warps of this GPU
// arrive (work[1]); the GPU leader (first consumer thread of CTA 0) then
// signals both neighbours that global phase phase0+i is complete, waits
// until both neighbours completed phase0+i as well (their halo pushes into
// our ghost rows have landed, and they no longer read the ghost rows we are
// about to overwrite), and publishes the release in work[3].
__device__ __forceinline__ void halo_gate(const HaloArgs& h, unsigned* work, int i, bool open, int nthreads,
                                          bool cta_leader, bool gpu_leader) {
  asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
  if (i >= 0 && cta_leader) {
    __threadfence();
    atomicAdd(work + 1, 1u);
  }
  if (gpu_leader) {
    if (i >= 0) {
      while (ld_acquire(work + 1) < gridDim.x * (unsigned)(i + 1)) __nanosleep(64);
      __threadfence_system();
      atomicAdd_system(h.up_flags + 1, 1u);    // we are the lower neighbour of the slab above
      atomicAdd_system(h.down_flags + 0, 1u);  // and the upper neighbour of the slab below
    }
    if (open) {
      const unsigned need = (unsigned)(h.phase0 + (unsigned long long)(i + 1));
      while (ld_acquire_sys(h.my_flags + 0) < need || ld_acquire_sys(h.my_flags + 1) < need) __nanosleep(64);
      __threadfence_system();
      atomicExch(work + 3, (unsigned)(i + 2));
    }
  }
  if (open && cta_leader) {
    while (ld_acquire(work + 3) < (unsigned)(i + 2)) __nanosleep(64);
    __threadfence();
  }
  asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}

// Host I/O of a flip launch (msb_window_io): chunk groups of kIoCpw chunks.
struct WinIO {
  const uint32_t* lin_in;
  uint32_t* lin_out;
  long long *ups, *unsat;
  unsigned ngroups;  // groups of kIoCpw chunks
  int load16;        // rows * nch % 16 == 0: the prologue loads 16 chunks per batch
};

// Prologue share of warp w of nw (every warp of the grid): groups of CPW
// chunks.  With CPW = 16 a cfg2 lattice is fewer groups than warps, so each
// warp has at most one group, i.e. 16 loads in flight, and the conversion
// takes ~the latency of one load batch.
template <int CPW>
__device__ __forceinline__ void win_load(const Geo& G, uint32_t* spins, const WinIO& io, unsigned w, unsigned nw) {
  const unsigned ng = io.ngroups / (CPW / kIoCpw);
  for (unsigned q = w; q < ng; q += nw) from_linear_group<CPW>(G, io.lin_in, spins, q);
}

// Epilogue of one flip warp (cw of nc): export its contiguous range of chunk
// groups; observables summed per replica run, one atomic per run and warp.
template <bool LIN, bool OBS>
__device__ __forceinline__ void win_export(const Geo& G, const uint32_t* spins, const WinIO& io, unsigned cw,
                                           unsigned nc) {
  const unsigned per = (io.ngroups + nc - 1) / nc;
  const unsigned lo = min(io.ngroups, cw * per), hi = min(io.ngroups, lo + per);
  int cs = -1;
  uint32_t u = 0, b = 0;
  auto flush = [&]() {
    if (!OBS || cs < 0) return;
    const uint32_t tu = __reduce_add_sync(0xFFFFFFFFu, u), tb = __reduce_add_sync(0xFFFFFFFFu, b);
    if ((threadIdx.x & 31) == 0) {
      atomicAdd(reinterpret_cast<unsigned long long*>(io.ups + cs), (unsigned long long)tu);
      atomicAdd(reinterpret_cast<unsigned long long*>(io.unsat + cs), (unsigned long long)tb);
    }
  };
  for (unsigned q = lo; q < hi; q++) {
    uint32_t du = 0, db = 0;
    const int s = export_group<kIoCpw, LIN, OBS, true>(G, spins, io.lin_out, q, du, db);
    if (OBS && s != cs) {
      flush();
      cs = s;
      u = b = 0;
    }
    u += du;
    b += db;
  }
  flush();
}

// Window launch: warps [0, pwarps) fill the next window (pwarps = 0: no
// production); the other warps flip slots [first, first + count) of `cur`
// (red, barrier, blue, barrier, ...).  With a halo (slabs) every phase is
// gated by halo_gate and all neighbour reads go through L2.  Host I/O (io,
// whole lattices): every warp of the grid first converts io.lin_in into the
// spins (16-chunk groups: a few us; each CTA then arrives on work[1] and only
// the flip warps wait for all arrivals, the producers go on), and after the
// last phase the flip warps export io.lin_out / the observables in their
// slack behind the producers.  (The flip warps alone took ~190 us to
// convert beside 28 producer warps per SM, and became the critical path.)
// Threads per direct launch (tuning define).  1024 measured best at cfg2
// (1.99 T) against 768 (1.54 T) and 512 (1.68 T): with fewer warps the
// band groups no longer spread one per warp, which costs more than the
// 64-register cap's spills.
#ifndef MSB_DIRECT_THREADS
#define MSB_DIRECT_THREADS 1024
#endif
constexpr int kDirectThreads = MSB_DIRECT_THREADS;

template <int SRC, int CB, bool HALO, int DIRECT = 0, int NT = 0>
__global__ void __launch_bounds__(NT ? NT : (DIRECT ? kDirectThreads : kRngThreads), 1) k_win(const WinArgs wa, const FlipArgs fa0, const HaloArgs ha,
                                                        const WinIO io, const uint32_t* cur, int first, int count,
                                                        int pwarps) {
  extern __shared__ uint4 jt[];
#ifdef MSB_TRACE
  MSB_TRACE_PUT(0, gtimer());
#endif
  if (SRC == kSrcXoshiro && pwarps > 0) {
    for (int i = threadIdx.x; i < kJumpWords / 4; i += blockDim.x) jt[i] = wa.jump[i];
    __syncthreads();
  }
  const int warp = threadIdx.x >> 5;
  const unsigned total_warps = gridDim.x * (blockDim.x >> 5);
#ifdef MSB_TRACE
  MSB_TRACE_PUT(1, gtimer());
  MSB_TRACE_PUT(3, warp < pwarps ? 0ull : (1ull << 63));
#endif
  const bool pro = !HALO && io.lin_in != nullptr;
#ifdef MSB_TRACE
  MSB_TRACE_PUT(5, 0ull);
#endif
  if (pro) {
    // each warp converts its share and reports it; the CTA's last warp posts
    // the CTA's arrival, so a producer waits for nothing but its own share
    __shared__ unsigned pro_done;
    if (threadIdx.x == 0) pro_done = 0;
    __syncthreads();
    const unsigned w = (unsigned)warp * gridDim.x + blockIdx.x, nw = gridDim.x * (blockDim.x >> 5);
    if (io.load16) win_load<16>(fa0.G, fa0.spins, io, w, nw);
    else win_load<kIoCpw>(fa0.G, fa0.spins, io, w, nw);
    __syncwarp();
    if ((threadIdx.x & 31) == 0) {
      __threadfence();
      if (atomicAdd(&pro_done, 1u) == (blockDim.x >> 5) - 1) {
        __threadfence();
        atomicAdd(wa.work + 1, 1u);
      }
    }
#ifdef MSB_TRACE
    MSB_TRACE_PUT(5, gtimer());  // prologue done (this CTA)
#endif
  }
  if (!DIRECT && warp < pwarps) {
    win_produce<SRC, CB>(wa, jt, warp, pwarps);
  } else if (count > 0) {
    const int nwc = (int)(blockDim.x >> 5) - pwarps;
    const unsigned nc = gridDim.x * nwc;
    const unsigned cw = (warp - pwarps) * gridDim.x + blockIdx.x;
    // band walk: contiguous band groups per warp; else quads, lanes interleaved
    const bool band = fa0.band_h > 0;
    const unsigned total = band ? fa0.band_groups
                                : (unsigned)fa0.G.n_sim * (unsigned)fa0.G.rows * ((unsigned)fa0.G.Wp >> 2);
    const unsigned per = band ? (total + nc - 1) / nc : (((total + nc - 1) / nc + 31) & ~31u);
    const unsigned lo = min(total, cw * per), hi = min(total, lo + per);
    const unsigned i0 = lo + (threadIdx.x & 31);
    FlipArgs fa = fa0;
    unsigned cnt = 0;
    const bool leader = threadIdx.x == pwarps * 32;
    const bool gpu_leader = leader && blockIdx.x == 0;
    if (HALO) halo_gate(ha, wa.work, -1, true, nwc * 32, leader, gpu_leader);
    const unsigned base = pro ? gridDim.x : 0u;  // the prologue's arrivals on work[1]
    const bool epi = !HALO && (io.lin_out != nullptr || io.ups != nullptr);
    if (!HALO && io.ups != nullptr && blockIdx.x == 0)  // written, not added (ordered by the barriers below)
      for (int j = threadIdx.x - pwarps * 32; j < fa0.G.n_sim; j += nwc * 32) io.ups[j] = io.unsat[j] = 0;
    if (pro) {
      if (leader) {
        while (ld_acquire(wa.work + 1) < base) __nanosleep(64);
        __threadfence();
      }
      asm volatile("bar.sync 1, %0;" ::"r"(nwc * 32) : "memory");
    }
    const bool gflag_path = DIRECT && !HALO && wa.gflags && band && fa.band_nseg == 1;
    bool push_warp = true;  // HALO: this warp's bands include a slab's first or last row
    if (HALO && band) {
      const unsigned gps = (unsigned)fa0.G.rows / (unsigned)(fa0.band_gb * fa0.band_h), nseg = (unsigned)fa0.band_nseg;
      push_warp = false;
      for (unsigned g = lo; g < hi; g++) {
        const unsigned l = (g / nseg) % gps;
        push_warp |= l == 0 || l + 1 == gps;
      }
    }
    if (gflag_path) {
      // band groups in phase order, neighbour flags instead of grid barriers
      const unsigned gps = (unsigned)fa0.G.rows / (unsigned)(fa0.band_gb * fa0.band_h);
      for (int i = 0; i < 2 * count; i++) {
        const int X = i & 1;
        PbitsDirect dp;
        dp.thr9 = wa.thr9;
        dp.pk = wa.pk;
        dp.blk = wa.block0 + 2ull * (unsigned)(first + (i >> 1)) + (unsigned)X;
        for (unsigned g = lo; g < hi; g++) {
          if (i > 0) group_wait(wa.gflags, g, gps, wa.gphase0 + (unsigned)i);
          if (i == 0 && !pro) cnt += flip_band_run<false, false, false, DIRECT>(fa, g, g + 1, X, &dp);
          else cnt += flip_band_run<true, false, false, DIRECT>(fa, g, g + 1, X, &dp);
          group_done(wa.gflags, g, wa.gphase0 + (unsigned)i + 1u);
        }
      }
    } else
    for (int i = 0; i < 2 * count; i++) {
      const int X = i & 1;
      PbitsDirect dp;
      if (DIRECT) {  // inline bit-plane draws: the phase's stream block instead of a plane slot
        dp.thr9 = wa.thr9;
        dp.pk = wa.pk;
        dp.blk = wa.block0 + 2ull * (unsigned)(first + (i >> 1)) + (unsigned)X;
      } else {
        fa.planes = cur + (size_t)(first + (i >> 1)) * wa.slot_words;
      }
      if (band) {
        if (fa.band_nseg > 1) {  // wide rows (cfg4, cfg5): segment-edge words from memory
          if (HALO) cnt += flip_band_run<true, true, true, DIRECT>(fa, lo, hi, X, &dp);
          else if (i == 0 && !pro) cnt += flip_band_run<false, false, true, DIRECT>(fa, lo, hi, X, &dp);
          else cnt += flip_band_run<true, false, true, DIRECT>(fa, lo, hi, X, &dp);
        } else {
          if (HALO) cnt += flip_band_run<true, true, false, DIRECT>(fa, lo, hi, X, &dp);
          else if (i == 0 && !pro) cnt += flip_band_run<false, false, false, DIRECT>(fa, lo, hi, X, &dp);
          else cnt += flip_band_run<true, false, false, DIRECT>(fa, lo, hi, X, &dp);
        }
      } else if (!DIRECT) {
        if (HALO) cnt += flip_run<true, true>(fa, i0, hi, X);
        else if (i == 0 && !pro) cnt += flip_run<false>(fa, i0, hi, X);
        else cnt += flip_run<true>(fa, i0, hi, X);
      }
      const bool more = i + 1 < 2 * count;
      if (HALO) {
        // the halo pushes (peer stores) before the neighbours are told; only
        // warps holding a slab's first or last row push
        if (push_warp) __threadfence_system();
        halo_gate(ha, wa.work, i, more, nwc * 32, leader, gpu_leader);
      } else if (more) {
#ifdef MSB_TRACE
        if (i == 0) MSB_TRACE_PUT(6, gtimer());  // first phase done (before its barrier)
#endif
        consumer_barrier(wa.work + 1, base + gridDim.x * (unsigned)(i + 1), nwc * 32, leader);
      }
    }
    add_flips(fa.flips, cnt);
#ifdef MSB_TRACE
    MSB_TRACE_PUT(7, gtimer());  // flips done (before the epilogue)
#endif
    if (epi) {  // every flip of the launch is done before any export read
      // (the flag path has no per-phase grid barriers: this is its first)
      consumer_barrier(wa.work + 1, base + gridDim.x * (gflag_path ? 1u : (unsigned)(2 * count)), nwc * 32, leader);
      if (io.lin_out && io.ups) win_export<true, true>(fa0.G, fa0.spins, io, cw, nc);
      else if (io.lin_out) win_export<true, false>(fa0.G, fa0.spins, io, cw, nc);
      else win_export<false, true>(fa0.G, fa0.spins, io, cw, nc);
    }
  }
#ifdef MSB_TRACE
  MSB_TRACE_PUT(2, gtimer());
#endif
  finish_warp(wa.work, total_warps);
}

// Halo wait: until both neighbours completed `need` phases (their pushes
// into our ghost rows landed), e.g. before the observables of a slab.
__global__ void k_halo_wait(const unsigned* my_flags, unsigned need) {
  if (threadIdx.x == 0) {
    while (ld_acquire_sys(my_flags + 0) < need || ld_acquire_sys(my_flags + 1) < need) __nanosleep(128);
    __threadfence_system();
  }
}

// Piece start states of a window whose slot 0 starts at stream block
// `block0`: piece (j, segment = 4 X + q, k0, stream) starts at draw
// (block0 + 2j) 2n + seg n/2 + k0 n/32 of its stream.
__global__ void k_win_init(const WinArgs a, uint64_t seed, const uint4* __restrict__ pow) {
  const long long gi = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gi >= a.npieces) return;
  const WinPiece w = win_piece(a, (unsigned)gi);
  const Geo& G = a.G;
  const uint64_t n = (uint64_t)G.n, cells = (uint64_t)(G.m / 4);
  const uint64_t sid = ((uint64_t)G.sim_offset + (uint64_t)w.s) * cells + (uint64_t)(w.gamma - 1);
  const uint64_t D = (a.block0 + 2ull * w.j) * 2 * n + (uint64_t)w.seg * (n / 2) + (uint64_t)w.k0 * (n / 32);
  store_state(jump_by(stream_state(seed, sid), D, pow), a.states, a.npieces, gi);
}

int make_win_io(const msb_geom* g, const msb_window_io* io, int count, const msb_halo* halo, WinIO& wio) {
  wio = WinIO{};
  if (io && (io->lin_in || io->lin_out || io->ups || io->unsat)) {
    if (count == 0 || halo || g->ghost) return fail(MSB_ERR_ARG, "msb_window_io needs a flip launch of a whole lattice");
    if ((io->ups == nullptr) != (io->unsat == nullptr)) return fail(MSB_ERR_ARG, "ups and unsat go together");
    const Geo G = make_geo(g);
    const long long chunks = (long long)g->n_sim * g->rows * G.nch;
    if (((long long)g->rows * G.nch) % kIoCpw) return fail(MSB_ERR_UNSUPPORTED, "msb_window_io needs rows * chunks % 4 == 0");
    if (32LL * chunks >= (1LL << 31)) return fail(MSB_ERR_UNSUPPORTED, "too many chunks for msb_window_io");
    wio.lin_in = reinterpret_cast<const uint32_t*>(io->lin_in);
    wio.lin_out = reinterpret_cast<uint32_t*>(io->lin_out);
    wio.ups = reinterpret_cast<long long*>(io->ups);
    wio.unsat = reinterpret_cast<long long*>(io->unsat);
    wio.ngroups = (unsigned)(chunks / kIoCpw);
    wio.load16 = ((long long)g->rows * G.nch) % 16 == 0;
  }
  return MSB_OK;
}

int check_halo(const msb_geom* g, const msb_halo* halo, int count) {
  if (count > 0 && g->ghost && !halo) return fail(MSB_ERR_ARG, "slab windows flip with an msb_halo (in-kernel exchange)");
  if (halo && !g->ghost) return fail(MSB_ERR_ARG, "msb_halo needs a slab geometry (ghost = 1)");
  if (halo && (!halo->up_spins || !halo->down_spins || !halo->up_flags || !halo->down_flags || !halo->my_flags ||
               halo->up_R < 4 || halo->down_R < 4))
    return fail(MSB_ERR_ARG, "incomplete msb_halo");
  return MSB_OK;
}

void set_halo(const msb_halo* halo, int count, FlipArgs& fa, HaloArgs& ha) {
  ha = HaloArgs{};
  if (halo && count > 0) {
    fa.up_spins = halo->up_spins;
    fa.down_spins = halo->down_spins;
    fa.up_R = halo->up_R;
    fa.down_R = halo->down_R;
    ha.up_flags = halo->up_flags;
    ha.down_flags = halo->down_flags;
    ha.my_flags = halo->my_flags;
    ha.phase0 = halo->phase0;
    ha.on = 1;
  }
}

// Direct (bit-plane Philox) flips walk bands of 2 rows: all 32 warps of
// every SM flip, so the phase needs as many lane groups as possible.
bool direct_band(FlipArgs& fa, const msb_geom* g) {
  if (fa.band_h <= 0) return false;
  const int gb = fa.band_gb;
  if (g->rows % (gb * 2)) return false;
  fa.band_h = 2;
  fa.band_groups = (unsigned)((long long)g->n_sim * g->rows / (gb * 2) * fa.band_nseg);
  return true;
}

int check_window(const msb_geom* g, int S, int P, long long* npieces) {
  if (int r = check_geom(g)) return r;
  if (S < 1 || S > 64) return fail(MSB_ERR_ARG, "window length S must be in [1, 64]");
  if (P < 1 || P > 128 || (P & (P - 1))) return fail(MSB_ERR_ARG, "parts per stream-sweep P must be a power of two <= 128");
  if (g->ghost && P < 8) return fail(MSB_ERR_ARG, "slab windows need P >= 8 (one row per piece)");
  // P >= 8: S * n_sim * 2 colours * held rows * P/8 parts; P < 8: S * P * streams
  const long long np = P >= 8 ? (long long)S * g->n_sim * 2 * g->rows * (P / 8)
                              : (long long)S * P * g->n_sim * (g->m / 4);
  if (np >= (1LL << 31)) return fail(MSB_ERR_UNSUPPORTED, "too many window pieces");
  *npieces = np;
  return MSB_OK;
}

size_t slot_words(const msb_geom* g) {
  const Geo G = make_geo(g);
  return 2ull * 2 * (size_t)g->n_sim * g->rows * G.Wp;
}

void fill_win_args(WinArgs& w, const msb_geom* g, const msb_sweep_params* p, int S, int P, long long np,
                   uint32_t* states, uint32_t* planes) {
  w.G = make_geo(g);
  w.states = states;
  w.thr9 = p->thr9;
  w.jump = reinterpret_cast<const uint4*>(p->jump);
  w.planes = planes;
  w.work = p->work;
  w.npieces = np;
  w.slot_words = slot_words(g);
  w.S = S;
  w.P = P;
  w.pshift = 0;
  while ((1 << w.pshift) < P) w.pshift++;
  w.kg = P > 8 ? P / 8 : 1;
  w.kr = 16 / w.kg;
  w.nseg = P <= 8 ? 8 / P : 1;
  w.kit = w.nseg * w.kr;
  w.streams = g->n_sim * (g->m / 4);
  w.streams_div.init((uint32_t)w.streams);
  w.cells_div.init((uint32_t)(g->m / 4));
  w.sims_div.init((uint32_t)g->n_sim);
  w.seed_lo = (uint32_t)p->seed;
  w.seed_hi = (uint32_t)(p->seed >> 32);
  w.block0 = p->block;
  w.pk = philox_keys(p->seed);
}

}  // namespace
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
  // S = 8 sweeps unless two window buffers would exceed 8 GiB of planes
  const long long slot_bytes = 4LL * (long long)slot_words(g);
  int s = 8;
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

int msb_window_sweep(const msb_geom* g, const msb_sweep_params* p, int32_t S, int32_t P, uint32_t* spins,
                     uint32_t* states, const uint32_t* cur, int32_t first, int32_t count, uint32_t* next,
                     uint64_t* flips, const msb_halo* halo, const msb_window_io* io, void* stream) {
  long long np = 0;
  if (int r = check_window(g, S, P, &np)) return r;
  if (int r = check_params(p)) return r;
  if (p->mode == MSB_MODE_GENERIC) return fail(MSB_ERR_UNSUPPORTED, "lookahead windows need FERRO/ANTI tables");
  if (first < 0 || count < 0 || first + count > S) return fail(MSB_ERR_ARG, "slots [first, first+count) outside the window");
  if (count > 0 && (!spins || !cur || !flips)) return fail(MSB_ERR_ARG, "null buffer");
  if (int r = check_halo(g, halo, count)) return r;
  if (count > 0)
    if (int r = check_flip_extent(g, 2)) return r;
  WinIO wio = {};
  if (int r = make_win_io(g, io, count, halo, wio)) return r;
  if (!next && count == 0) {
    if (halo) {
      k_halo_wait<<<1, 32, 0, as_stream(stream)>>>(halo->my_flags, (unsigned)halo->phase0);
      CUDA_TRY(cudaGetLastError());
    }
    return MSB_OK;
  }
  if (next && p->rng == MSB_RNG_XOSHIRO && (!states || !p->jump)) return fail(MSB_ERR_ARG, "null RNG state or jump table");
  const bool produce = next != nullptr;
  WinArgs wa;
  fill_win_args(wa, g, p, S, P, np, states, next);
  FlipArgs fa;
  fill_flip_args(fa, g, p, 0, spins, cur, flips);
  HaloArgs ha;
  set_halo(halo, count, fa, ha);
  // Warp split of the 32-warp CTAs.  A unit (32 pieces) is a whole window's
  // share of a stream, so an extra producer round costs a full unit: when the
  // units fit one round, give producers exactly that round and the rest of
  // the CTA to the flips; otherwise 8 flip warps (flip-heavy shapes gain,
  // others are insensitive).  Producers are capped so the plane rows being
  // written stay L2-resident (see msb_window_parts).  MSB_FLIP_WARPS /
  // MSB_PRODUCER_WARPS override (tuning).
  static const int env_pw = [] { const char* e = getenv("MSB_PRODUCER_WARPS"); return e ? atoi(e) : 0; }();
  static const int env_cw = [] { const char* e = getenv("MSB_FLIP_WARPS"); return e ? atoi(e) : 0; }();
  int dev = 0, sms = 148;
  CUDA_TRY(cudaGetDevice(&dev));
  CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const long long units = (np + 31) / 32;
  // bytes of plane rows a producer warp has open: 2 rows (planes) per row
  // being written, 32 / max(1, P/8) rows per warp (win_piece numbering)
  const long long live_per_warp = 32LL * 2 * 4 * fa.G.Wp / std::max(1, P / 8);
  const int cap = (int)std::max(4LL, std::min(32LL, (100LL << 20) / ((long long)sms * live_per_warp)));
  int pwarps = 0;
  if (produce) {
    if (count == 0) {
      pwarps = cap;
    } else {
      const long long one_round = (units + sms - 1) / sms;  // producer warps per CTA for a single round
      int cw = one_round <= 30 ? (int)(32 - one_round) : 8;
      if (env_cw > 0) cw = std::min(28, env_cw);
      pwarps = std::min(cap, 32 - cw);
    }
    if (env_pw > 0) pwarps = std::min(32, env_pw);
  }
  const bool philox = p->rng == MSB_RNG_PHILOX, pbits = p->rng == MSB_RNG_PHILOX_BITS;
  // compile-time chunk width: every chunk 32 draws (n/32 % 32 == 0), a
  // single 16-draw chunk (n = 512), or generic
  const int cb = (wa.G.words % 32) == 0 ? 32 : (wa.G.words == 16 ? 16 : 0);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)sms);
  cfg.blockDim = dim3(kRngThreads);
  cfg.dynamicSmemBytes = (philox || pbits || pwarps == 0) ? 0 : (size_t)kJumpWords * 4;
  cfg.stream = as_stream(stream);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = count > 0 ? 1 : 0;  // grid barriers only among consumers
#define MSB_LAUNCH_WIN(SRC, CB, HALO)                                                            \
  do {                                                                                           \
    static std::once_flag o_;                                                                    \
    static cudaError_t e_;                                                                       \
    if (int r = set_smem_attr(k_win<SRC, CB, HALO>, o_, e_)) return r;                          \
    CUDA_TRY(cudaLaunchKernelEx(&cfg, k_win<SRC, CB, HALO>, wa, fa, ha, wio, cur, first, count, pwarps)); \
  } while (0)
#define MSB_LAUNCH_WIN_CB(SRC, HALO)                  \
  do {                                                \
    if (cb == 32) MSB_LAUNCH_WIN(SRC, 32, HALO);      \
    else if (cb == 16) MSB_LAUNCH_WIN(SRC, 16, HALO); \
    else MSB_LAUNCH_WIN(SRC, 0, HALO);                \
  } while (0)
  if (ha.on) {
    if (philox) MSB_LAUNCH_WIN_CB(kSrcPhilox, true);
    else if (pbits) MSB_LAUNCH_WIN_CB(kSrcPbits, true);
    else MSB_LAUNCH_WIN_CB(kSrcXoshiro, true);
  } else {
    if (philox) MSB_LAUNCH_WIN_CB(kSrcPhilox, false);
    else if (pbits) MSB_LAUNCH_WIN_CB(kSrcPbits, false);
    else MSB_LAUNCH_WIN_CB(kSrcXoshiro, false);
  }
#undef MSB_LAUNCH_WIN_CB
#undef MSB_LAUNCH_WIN
  return MSB_OK;
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

int64_t msb_direct_flag_words(const msb_geom* g, const msb_sweep_params* p) {
  if (!msb_direct_ok(g, p)) return -1;
  FlipArgs fa;
  fill_flip_args(fa, g, p, 0, nullptr, nullptr, nullptr);
  direct_band(fa, g);
  return fa.band_nseg == 1 ? (int64_t)fa.band_groups : 0;
}

int msb_direct_sweep(const msb_geom* g, const msb_sweep_params* p, uint32_t* spins, int32_t n_sweeps, uint64_t* flips,
                     uint32_t* group_flags, uint32_t flag_phase0, const msb_halo* halo, const msb_window_io* io,
                     void* stream) {
  if (int r = check_geom(g)) return r;
  if (int r = check_params(p)) return r;
  if (p->rng != MSB_RNG_PHILOX_BITS) return fail(MSB_ERR_ARG, "direct sweeps draw the bit-plane Philox stream");
  if (p->mode == MSB_MODE_GENERIC) return fail(MSB_ERR_UNSUPPORTED, "direct sweeps need FERRO/ANTI tables");
  if (n_sweeps < 0 || n_sweeps > (1 << 20)) return fail(MSB_ERR_ARG, "sweep count must be in [0, 2^20]");
  if (n_sweeps == 0) return MSB_OK;
  if (!spins || !flips) return fail(MSB_ERR_ARG, "null buffer");
  if (int r = check_halo(g, halo, n_sweeps)) return r;
  if (int r = check_flip_extent(g, 2)) return r;
  WinIO wio;
  if (int r = make_win_io(g, io, n_sweeps, halo, wio)) return r;
  const Geo G = make_geo(g);
  const int cb = (G.words % 32) == 0 ? 32 : (G.words == 16 ? 16 : 0);
  FlipArgs fa;
  fill_flip_args(fa, g, p, 0, spins, nullptr, flips);
  if (!cb || !direct_band(fa, g)) return fail(MSB_ERR_UNSUPPORTED, "direct sweeps need n/32 % 32 == 0 or n = 512 and band rows");
  HaloArgs ha;
  set_halo(halo, n_sweeps, fa, ha);
  WinArgs wa = {};
  wa.G = G;
  wa.thr9 = p->thr9;
  wa.work = p->work;
  wa.pk = philox_keys(p->seed);
  wa.block0 = p->block;
  wa.seed_lo = (uint32_t)p->seed;
  wa.seed_hi = (uint32_t)(p->seed >> 32);
  if (group_flags && !halo && fa.band_nseg == 1) {  // else grid barriers between phases
    wa.gflags = group_flags;
    wa.gphase0 = flag_phase0;
  }
  int dev = 0, sms = 148;
  CUDA_TRY(cudaGetDevice(&dev));
  CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)sms);
  cfg.blockDim = dim3(kDirectThreads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = as_stream(stream);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const uint32_t* cur = nullptr;
  const int first = 0, pwarps = 0;
#define MSB_LAUNCH_DIRECT(CB, HALO)                                                                  \
  do {                                                                                               \
    static std::once_flag o_;                                                                        \
    static cudaError_t e_;                                                                           \
    if (int r = set_smem_attr(k_win<kSrcPbits, CB, HALO, CB>, o_, e_)) return r;                    \
    CUDA_TRY(cudaLaunchKernelEx(&cfg, k_win<kSrcPbits, CB, HALO, CB>, wa, fa, ha, wio, cur, first, n_sweeps, pwarps)); \
  } while (0)
  // Band groups that fit one per warp in 28 warps per SM (cfg2: 4096 groups,
  // 148 x 28 = 4144 warps) run 896-thread CTAs: no warp idles, and ptxas gets
  // 72 registers instead of 64.
  const long long g28 = 28LL * sms, g24 = 24LL * sms;
  static const int env_nt = [] { const char* e = getenv("MSB_DIRECT_NT"); return e ? atoi(e) : -1; }();
  if (!ha.on && cb == 32 && env_nt != 0 && (long long)fa.band_groups <= g28 && (long long)fa.band_groups > g24) {
    cfg.blockDim = dim3(896);
    static std::once_flag o_;
    static cudaError_t e_;
    if (int r = set_smem_attr(k_win<kSrcPbits, 32, false, 32, 896>, o_, e_)) return r;
    CUDA_TRY(cudaLaunchKernelEx(&cfg, k_win<kSrcPbits, 32, false, 32, 896>, wa, fa, ha, wio, cur, first, n_sweeps,
                                pwarps));
    return MSB_OK;
  }
  // Many groups per warp (cfg3: 24128 groups, ~5 per warp): 768-thread CTAs
  // give ptxas 80 registers, and the extra groups per warp cost little
  // (measured 1.49 vs 1.45 T at cfg3).
  if (!ha.on && cb == 16 && env_nt != 0 && (long long)fa.band_groups >= 4LL * 32 * sms) {
    cfg.blockDim = dim3(768);
    static std::once_flag o_;
    static cudaError_t e_;
    if (int r = set_smem_attr(k_win<kSrcPbits, 16, false, 16, 768>, o_, e_)) return r;
    CUDA_TRY(cudaLaunchKernelEx(&cfg, k_win<kSrcPbits, 16, false, 16, 768>, wa, fa, ha, wio, cur, first, n_sweeps,
                                pwarps));
    return MSB_OK;
  }
  if (ha.on) {
    if (cb == 32) MSB_LAUNCH_DIRECT(32, true);
    else MSB_LAUNCH_DIRECT(16, true);
  } else {
    if (cb == 32) MSB_LAUNCH_DIRECT(32, false);
    else MSB_LAUNCH_DIRECT(16, false);
  }
#undef MSB_LAUNCH_DIRECT
  return MSB_OK;
}

}  // extern "C"
