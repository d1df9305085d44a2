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
#pragma once
#include "msb_sweep.cuh"
#include "msb_io.cuh"
#include "msb_window_api.h"

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
  unsigned* flags;              // msb_sweep_params.flags (header, halo slots, group flags) or null
  unsigned nslot;               // halo slots per direction: n_sim * row segments
};

// Flag buffer regions (include/msb200.h, msb_flag_words).
__device__ __forceinline__ unsigned* flags_above(const WinArgs& a) { return a.flags + 1; }
__device__ __forceinline__ unsigned* flags_below(const WinArgs& a) { return a.flags + 1 + a.nslot; }
__device__ __forceinline__ unsigned* flags_groups(const WinArgs& a) { return a.flags + 1 + 2 * a.nslot; }

__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Phases completed by earlier launches on this flag buffer (flags[0]; the
// launch's last warp advances it, finish_flags).
__device__ __forceinline__ unsigned flags_base(const WinArgs& a) {
  return a.flags ? ld_acquire(a.flags) : 0u;
}

// Direct sweeps with band-group flags instead of grid barriers: a group's
// phase i reads the other colour's rows of its own group and of the groups
// just above and below (same replica, periodic), and overwrites rows those
// groups read in phase i-1.  So it waits for both neighbours to have
// completed phase i-1, and publishes its own completion; slow groups delay
// only their neighbours instead of the whole grid.  (Whole lattices whose
// rows are one band segment; the general form is gf_wait / gf_done.)
#ifndef MSB_WAIT_MAX_NS
#define MSB_WAIT_MAX_NS 512
#endif
constexpr unsigned kWaitMaxNs = MSB_WAIT_MAX_NS;

__device__ __forceinline__ void group_wait(const unsigned* flags, unsigned g, unsigned gps, unsigned need) {
  if ((threadIdx.x & 31) == 0) {
    const unsigned s0 = g - g % gps, l = g - s0;
    const unsigned up = s0 + (l == 0 ? gps - 1 : l - 1), dn = s0 + (l + 1 == gps ? 0 : l + 1);
    // backing off: spinning lanes issue instructions the working warps of
    // the SM need (the polls were 7% of the cfg2 direct kernel's
    // instructions at a fixed 32 ns)
    unsigned ns = 32;
    while (ld_acquire(flags + up) < need || ld_acquire(flags + dn) < need) {
      __nanosleep(ns);
      ns = min(ns * 2, kWaitMaxNs);
    }
  }
  __syncwarp();
}

// group_wait for band l of its replica (no division).
__device__ __forceinline__ void group_wait_at(const unsigned* flags, unsigned g, unsigned l, unsigned gps, unsigned need) {
  if ((threadIdx.x & 31) == 0) {
    const unsigned up = l == 0 ? g + gps - 1 : g - 1, dn = l + 1 == gps ? g + 1 - gps : g + 1;
    unsigned ns = 32;
    while (ld_acquire(flags + up) < need || ld_acquire(flags + dn) < need) {
      __nanosleep(ns);
      ns = min(ns * 2, kWaitMaxNs);
    }
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

// The general band-group order (window consumers, wide rows in segments,
// row slabs).  Group g = (replica s, band l of gps, segment seg of nseg).
// Its phase i reads the other colour's rows of bands l-1, l, l+1 (same
// words) and the edge words of segments seg-1, seg+1 (same band), and
// overwrites rows those groups read in phase i-1: it waits for those four
// neighbours to have completed phase i-1 (periodic in l for a whole
// lattice, in seg always).  In a slab (HALO) band 0 reads the ghost row
// above instead of band gps-1: it waits for the slab above's last band of
// the same segment (the "from above" slot it writes into our flags), and
// after its phase tells the slab above (its "from below" slot); band gps-1
// likewise with the slab below.  So only the bands that hold a slab's first
// or last row ever wait on another GPU.
struct GroupOrder {
  unsigned* grp;           // group flags
  const unsigned* above;   // our "from above" slots
  const unsigned* below;   // our "from below" slots
  unsigned* up_below;      // the slab above's "from below" slots (HALO)
  unsigned* down_above;    // the slab below's "from above" slots (HALO)
  unsigned gps, nseg;
};

__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_relaxed_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(unsigned* p, unsigned v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_sys(unsigned* p, unsigned v) {
  asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Neighbours of band group g in the group order, and which of them another
// warp (or another slab: sys) owns.  [lo, hi) is the calling warp's range:
// a neighbour inside it was handled by this warp earlier in program order,
// so it needs neither a wait nor a published flag.
struct GroupNb {
  const unsigned *pu, *pd, *pl, *pr;
  bool ext_u, ext_d, ext_h, sys_u, sys_d;
  unsigned slot, l;
};

// (s, l, seg) = replica, band, segment of group g (g = (s gps + l) nseg + seg).
template <bool HALO>
__device__ __forceinline__ GroupNb group_nb_at(const GroupOrder& f, unsigned g, unsigned s, unsigned l, unsigned seg,
                                               unsigned lo, unsigned hi) {
  GroupNb n;
  n.l = l;
  n.slot = s * f.nseg + seg;
  n.sys_u = HALO && l == 0;
  n.sys_d = HALO && l + 1 == f.gps;
  const unsigned gu = l == 0 ? g + (f.gps - 1) * f.nseg : g - f.nseg;
  const unsigned gd = l + 1 == f.gps ? g - (f.gps - 1) * f.nseg : g + f.nseg;
  const unsigned gl = seg == 0 ? g + f.nseg - 1 : g - 1;
  const unsigned gr2 = seg + 1 == f.nseg ? g + 1 - f.nseg : g + 1;
  n.pu = n.sys_u ? f.above + n.slot : f.grp + gu;
  n.pd = n.sys_d ? f.below + n.slot : f.grp + gd;
  n.pl = f.grp + gl;
  n.pr = f.grp + gr2;
  auto out = [&](unsigned x) { return x < lo || x >= hi; };
  n.ext_u = n.sys_u || out(gu);
  n.ext_d = n.sys_d || out(gd);
  n.ext_h = f.nseg > 1 && (out(gl) || out(gr2));
  return n;
}

template <bool HALO>
__device__ __forceinline__ GroupNb group_nb(const GroupOrder& f, unsigned g, unsigned lo, unsigned hi) {
  const unsigned gr = g / f.nseg, seg = g - gr * f.nseg, s = gr / f.gps, l = gr - s * f.gps;
  return group_nb_at<HALO>(f, g, s, l, seg, lo, hi);
}

// Wait until the neighbours of a group that are owned elsewhere completed
// phase need-1 (acquire polls: one L2 round trip when the neighbour is
// already done, the common case; a relaxed poll followed by acquires
// measured two; backing off so spinning warps leave the issue slots to the
// working ones).  local = false (the first phase of a launch): the
// neighbours on this GPU finished the previous launch (stream order), only
// the slots written by the neighbour slabs count.
__device__ __forceinline__ void gf_wait_nb(const GroupNb& n, unsigned need, bool local) {
  if ((threadIdx.x & 31) == 0) {
    bool ok_u = !(n.ext_u && (local || n.sys_u)), ok_d = !(n.ext_d && (local || n.sys_d)), ok_h = !(n.ext_h && local);
    unsigned ns = 32;
    while (!(ok_u && ok_d && ok_h)) {
      if (!ok_u) ok_u = (n.sys_u ? ld_acquire_sys(n.pu) : ld_acquire(n.pu)) >= need;
      if (!ok_d) ok_d = (n.sys_d ? ld_acquire_sys(n.pd) : ld_acquire(n.pd)) >= need;
      if (!ok_h) ok_h = ld_acquire(n.pl) >= need && ld_acquire(n.pr) >= need;
      if (!(ok_u && ok_d && ok_h)) {
        __nanosleep(ns);
        ns = min(ns * 2, kWaitMaxNs);
      }
    }
  }
  __syncwarp();
}

// Publish group g's completion of a phase (value v) to whoever waits on it:
// neighbours owned by other warps (a release: one acq_rel fence, then a
// relaxed store), and for a slab's edge bands the neighbour slab (system
// scope: our halo pushes into its ghost rows are ordered before).  A group
// whose neighbours are all in this warp's range publishes nothing.
__device__ __forceinline__ void gf_done_nb(const GroupOrder& f, const GroupNb& n, unsigned g, unsigned v) {
  __syncwarp();
  if ((threadIdx.x & 31) == 0) {
    if (n.sys_u || n.sys_d) {
      asm volatile("fence.acq_rel.sys;" ::: "memory");
      if (n.sys_u) st_relaxed_sys(f.up_below + n.slot, v);
      if (n.sys_d) st_relaxed_sys(f.down_above + n.slot, v);
      st_relaxed(f.grp + g, v);
    } else if (n.ext_u || n.ext_d || n.ext_h) {
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
      st_relaxed(f.grp + g, v);
    }
  }
}

// flip_band_run hook of the group order: wait before a group (when `wait`:
// later phases, or the first phase of a slab's edge bands).  Completion is
// published per CTA after the phase (gf_publish_cta).
// PER_GROUP: publish each group right after it (gf_done) -- the direct
// walk, whose 32 warps per SM diverge too much to meet at a CTA barrier every
// phase (1.73 -> 1.27 T at cfg4 with gf_publish_cta); the window consumers
// publish per CTA instead.
template <bool HALO, bool PER_GROUP>
struct GfHooks {
  const GroupOrder* f;
  unsigned need, lo, hi;
  bool local, wait;
  // cursor of the walk (groups come in order lo, lo+1, ...): no divisions per group
  mutable unsigned g_next = ~0u, cs = 0, cl = 0, cseg = 0;
  mutable GroupNb nb;
  __device__ __forceinline__ void pre(unsigned g) const {
    if (g != g_next) {
      const unsigned gr = g / f->nseg;
      cseg = g - gr * f->nseg;
      cs = gr / f->gps;
      cl = gr - cs * f->gps;
    }
    nb = group_nb_at<HALO>(*f, g, cs, cl, cseg, lo, hi);
    if (wait) gf_wait_nb(nb, need, local);
  }
  __device__ __forceinline__ void post(unsigned g) const {
    if (PER_GROUP) gf_done_nb(*f, nb, g, need + 1u);
    g_next = g + 1;
    if (++cseg == f->nseg) {
      cseg = 0;
      if (++cl == f->gps) {
        cl = 0;
        cs++;
      }
    }
  }
};

// End of a phase of the group order, per CTA: the flip warps meet at a named
// barrier, then the CTA's leader issues ONE fence (system scope if one of the
// CTA's groups holds a slab edge row: its pushes into the neighbour's ghost
// rows) and publishes value v for every group of the CTA's warps that a
// warp elsewhere or a neighbour slab waits on.  A fence per group cost
// ~3% at cfg4 (the fence drains the warp's outstanding stores each time).
template <bool HALO>
__device__ __forceinline__ void gf_publish_cta(const GroupOrder& f, unsigned v, unsigned per, unsigned total, int nwc,
                                               unsigned vgrid, unsigned vb, bool leader) {
  asm volatile("bar.sync 1, %0;" ::"r"(nwc * 32) : "memory");
  if (!leader) return;
  bool sys = false;
  if (HALO) {
    for (int j = 0; j < nwc && !sys; j++) {
      const unsigned lo = min(total, ((unsigned)j * vgrid + vb) * per), hi = min(total, lo + per);
      for (unsigned g = lo; g < hi && !sys; g++) {
        const unsigned l = (g / f.nseg) % f.gps;
        sys = l == 0 || l + 1 == f.gps;
      }
    }
  }
  if (sys) asm volatile("fence.acq_rel.sys;" ::: "memory");
  else asm volatile("fence.acq_rel.gpu;" ::: "memory");
  for (int j = 0; j < nwc; j++) {
    const unsigned lo = min(total, ((unsigned)j * vgrid + vb) * per), hi = min(total, lo + per);
    for (unsigned g = lo; g < hi; g++) {
      const GroupNb n = group_nb<HALO>(f, g, lo, hi);
      if (n.sys_u) st_relaxed_sys(f.up_below + n.slot, v);
      if (n.sys_d) st_relaxed_sys(f.down_above + n.slot, v);
      if (n.ext_u || n.ext_d || n.ext_h) st_relaxed(f.grp + g, v);
    }
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
#pragma unroll kChunkUnroll32
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

// Where a window piece jumps its stream to the next window: after its draws
// (1) or spread through the draw loop (0, 8 nibble-table words at a time).
// Measured at 64-sweep windows: after the draws, cfg3 0.963 -> 0.977 T, cfg2
// 0.965 either way (at 8-sweep windows both measured within 1%).
#ifndef MSB_JUMP_END
#define MSB_JUMP_END 1
#endif
constexpr bool kJumpEnd = MSB_JUMP_END;

// One producer warp's share of a window (pieces numbered as win_piece).
template <int SRC, int CB>
__device__ __forceinline__ void win_produce(const WinArgs& a, const uint4* __restrict__ jt, int role_warp,
                                            int role_warps, unsigned vb, unsigned vgrid) {
  constexpr bool XO = SRC == kSrcXoshiro;
  const Geo& G = a.G;
  const int lane = threadIdx.x & 31;
  const long long units = (a.npieces + 31) / 32;
  const size_t pstride = (size_t)G.n_sim * G.rows * G.Wp;
  const long long nwarps = (long long)role_warps * vgrid;
  const int cells = G.m / 4;
  const unsigned long long n = (unsigned long long)G.n;
  long long u = (long long)role_warp * vgrid + vb;
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
        if (!kJumpEnd) {
          jw[0] = st.a0; jw[1] = st.a1; jw[2] = st.b0; jw[3] = st.b1;
          jw[4] = st.c0; jw[5] = st.c1; jw[6] = st.d0; jw[7] = st.d1;
        }
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
        if (XO && CB == 16 && !(a.kr & 1)) {
          // n = 512: the 16 draws of k (even) and the 16 of k + 1 are one
          // run of 32 consecutive draws of the stream: one 32-draw loop (as
          // for 32-draw rows) fills both plane words, halving the per-k
          // stores, addressing and jump bookkeeping
          for (int kk = 0; kk < a.kr; kk += 2) {
            const int k = w.k0 + kk;
            uint32_t acc0 = 0, acc1 = 0;
#pragma unroll kChunkUnroll
            for (int i = 0; i < 32; i++) {
              const uint32_t h9 = xstep(st) << 9;
              acc_reject(acc0, h9, key0);
              acc_reject(acc1, h9, key1);
            }
            // REJECT bits, newest draw in bit 0: reversed, bit i = draw i
            // packed planes (FlipArgs::pk16): t(k + 1) = t(k) + 4 rides in the high half
            out[pk16_word(k)] = ~__brev(acc0);
            out[pstride + pk16_word(k)] = ~__brev(acc1);
            if (!kJumpEnd) {
              jacc += 16;
              while (jacc >= a.kit) {
                jacc -= a.kit;
                jump_word(jt, nib, jw, r);
              }
            }
          }
          continue;
        }
        if (SRC == kSrcPbits && CB == 16 && !(a.kr & 1)) {
          // n = 512: one bit-plane group is the 16 draws of k (even) and of
          // k + 1 -- resolve it once for both rows of plane words
          const uint32_t key[2] = {key0, key1};
          for (int kk = 0; kk < a.kr; kk += 2) {
            const int k = w.k0 + kk;
            uint32_t acc[2];
            pbits_group<2>((pseg + (unsigned long long)k * 16) >> 5, pl, a.pk, key, 2, acc);
            out[pk16_word(k)] = acc[0];  // packed planes, as above
            out[pstride + pk16_word(k)] = acc[1];
          }
          continue;
        }
        for (int kk = 0; kk < a.kr; kk++) {
          const int k = w.k0 + kk;
          win_segment_k<SRC, CB>(a, st, pl, out + t_of_k(k), key0, key1, pstride,
                                   pseg + (unsigned long long)k * G.words);
          if (XO && !kJumpEnd) {  // the 8 jump words, spread evenly over the piece's kit k-iterations
            jacc += 8;
            while (jacc >= a.kit) {
              jacc -= a.kit;
              jump_word(jt, nib, jw, r);
            }
          }
        }
      }
      if (XO && kJumpEnd) {
        // the jump after the draws: the piece's start state is still in
        // memory, and the draw loop keeps no 16 jump registers live
        XState s0;
        load_state(s0, a.states, a.npieces, gi);
        store_state(jump_apply(s0, jt), a.states, a.npieces, gi);  // same piece, next window
      } else if (XO) {
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

struct HaloArgs {
  unsigned *up_below, *down_above;  // the neighbours' "from below" / "from above" slots
  int on;
};

// Slab phase gate, for slab rows without a band walk (msb_halo; the band
// walk orders phases per group instead, gf_wait / gf_done).  Ends local
// phase i (i = -1: launch start) and opens phase i+1 when `open`.  All
// consumer warps of this GPU's slab arrive (work[1]); its leader then tells
// both neighbours that phase base+i+1 is complete (every slot: the group
// form has one per segment and replica), waits until both neighbours have
// completed it too (their halo pushes into our ghost rows have landed, and
// they no longer read the ghost rows we are about to overwrite), and
// publishes the release in work[3].
__device__ __forceinline__ void halo_gate(const HaloArgs& h, const WinArgs& wa, unsigned base, int i, bool open,
                                          int nthreads, bool cta_leader, bool gpu_leader, unsigned vgrid) {
  unsigned* work = wa.work;
  asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
  if (i >= 0 && cta_leader) {
    __threadfence();
    atomicAdd(work + 1, 1u);
  }
  if (gpu_leader) {
    if (i >= 0) {
      while (ld_acquire(work + 1) < vgrid * (unsigned)(i + 1)) __nanosleep(64);
      __threadfence_system();
      const unsigned v = base + (unsigned)(i + 1);
      for (unsigned j = 0; j < wa.nslot; j++) {
        atomicExch_system(h.up_below + j, v);    // we are the slab below the one above
        atomicExch_system(h.down_above + j, v);  // and the slab above the one below
      }
    }
    if (open) {
      const unsigned need = base + (unsigned)(i + 1);
      for (unsigned j = 0; j < 2 * wa.nslot; j++)
        while (ld_acquire_sys(flags_above(wa) + j) < need) __nanosleep(64);
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

// n = 512 rows <-> packed rows in place (FlipArgs::pks), one row per thread
// (16 words in, 8 out, or back), rows [t, rows) step nt.
template <bool UNPACK>
__device__ __forceinline__ void pack_rows(uint32_t* spins, unsigned nrows, unsigned t, unsigned nt) {
  for (unsigned r = t; r < nrows; r += nt) {
    uint4* row = reinterpret_cast<uint4*>(spins + (size_t)r * 16);
    if (!UNPACK) {
      const uint4 a = __ldcg(row), b = __ldcg(row + 1), c = __ldcg(row + 2), d = __ldcg(row + 3);
      // word j: (t, t + 4), t = j (j < 4) or j + 4
      __stcg(row, make_uint4(a.x | (b.x << 16), a.y | (b.y << 16), a.z | (b.z << 16), a.w | (b.w << 16)));
      __stcg(row + 1, make_uint4(c.x | (d.x << 16), c.y | (d.y << 16), c.z | (d.z << 16), c.w | (d.w << 16)));
    } else {
      const uint4 lo = __ldcg(row), hi = __ldcg(row + 1);
      __stcg(row, make_uint4(lo.x & 0xFFFFu, lo.y & 0xFFFFu, lo.z & 0xFFFFu, lo.w & 0xFFFFu));
      __stcg(row + 1, make_uint4(lo.x >> 16, lo.y >> 16, lo.z >> 16, lo.w >> 16));
      __stcg(row + 2, make_uint4(hi.x & 0xFFFFu, hi.y & 0xFFFFu, hi.z & 0xFFFFu, hi.w & 0xFFFFu));
      __stcg(row + 3, make_uint4(hi.x >> 16, hi.y >> 16, hi.z >> 16, hi.w >> 16));
    }
  }
}

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
// (red, barrier, blue, barrier, ...).  Phase order: with flags, per band
// group (GF: gf_wait / gf_done, whole lattices and slabs; the direct path's
// single-segment whole lattices use group_wait / group_done); without,
// grid-wide consumer barriers, or for slabs without a band walk the
// GPU-wide halo_gate.  With a halo (slabs) all neighbour reads go through
// L2 and the edge rows are pushed into the neighbours' ghost rows.  Host
// I/O (io, whole lattices): every warp of the grid first converts
// io.lin_in into the spins (16-chunk groups: a few us; each CTA then
// arrives on work[1] and only the flip warps wait for all arrivals, the
// producers go on), and after the last phase the flip warps export
// io.lin_out / the observables in their slack behind the producers.  (The
// flip warps alone took ~190 us to convert beside 28 producer warps per SM,
// and became the critical path.)
// Threads per direct launch (tuning define).  1024 measured best at cfg2
// (1.99 T) against 768 (1.54 T) and 512 (1.68 T): with fewer warps the
// band groups no longer spread one per warp, which costs more than the
// 64-register cap's spills.
// Direct sweeps over 32-draw words in the split form (direct_group_split,
// msb_sweep.cuh): the group-flag path of single-segment whole lattices and the
// general group order (rows in segments, slabs, rings).  0: the walk form.
#ifndef MSB_DIRECT_SPLIT
#define MSB_DIRECT_SPLIT 1
#endif
constexpr bool kDirectSplit = MSB_DIRECT_SPLIT != 0;
#ifndef MSB_CTA_BLOCKS
#define MSB_CTA_BLOCKS 1
#endif
constexpr bool kCtaBlocks = MSB_CTA_BLOCKS != 0;
#ifndef MSB_CHUNK_MAP
#define MSB_CHUNK_MAP 4
#endif
constexpr unsigned kChunkMap = MSB_CHUNK_MAP;

#ifndef MSB_DIRECT_THREADS
#define MSB_DIRECT_THREADS 1024
#endif
constexpr int kDirectThreads = MSB_DIRECT_THREADS;

// Per-slab kernel arguments of a ring launch (msb_window_sweep_ring /
// msb_direct_sweep_ring), in device memory.
struct SlabCtx {
  WinArgs wa;
  FlipArgs fa;
  HaloArgs ha;
  const uint32_t* cur;
};

// The last warp of a launch (of a slab, in a ring launch) resets the work
// counters and advances the flag header by the launch's phases.
__device__ __forceinline__ void finish_launch(const WinArgs& wa, unsigned total_warps, unsigned phases) {
  if ((threadIdx.x & 31) == 0) {
    __threadfence();
    if (atomicAdd(wa.work + 2, 1u) == total_warps - 1) {
      if (wa.flags && phases) atomicAdd(wa.flags, phases);
      atomicExch(wa.work, 0u);
      atomicExch(wa.work + 1, 0u);
      atomicExch(wa.work + 3, 0u);
      atomicExch(wa.work + 2, 0u);
    }
  }
}

// vb / vgrid: this CTA's index among, and the number of, the CTAs working on
// its slab (the whole grid except in ring launches).
template <int SRC, int CB, bool HALO, int DIRECT, int GFX>
__device__ __forceinline__ void win_body(const WinArgs& wa, const FlipArgs& fa0, const HaloArgs& ha, const WinIO& io,
                                         const uint32_t* cur, int first, int count, int pwarps, unsigned vb,
                                         unsigned vgrid, uint4* jt) {
#ifdef MSB_TRACE
  MSB_TRACE_PUT(0, gtimer());
#endif
  if (SRC == kSrcXoshiro && pwarps > 0) {
    for (int i = threadIdx.x; i < kJumpWords / 4; i += blockDim.x) jt[i] = wa.jump[i];
    __syncthreads();
  }
  const int warp = threadIdx.x >> 5;
  const unsigned total_warps = vgrid * (blockDim.x >> 5);
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
    const unsigned w = (unsigned)warp * vgrid + vb, nw = vgrid * (blockDim.x >> 5);
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
    win_produce<SRC, CB>(wa, jt, warp, pwarps, vb, vgrid);
  } else if (count > 0) {
    const int nwc = (int)(blockDim.x >> 5) - pwarps;
    const unsigned nc = vgrid * nwc;
    const unsigned cw = (warp - pwarps) * vgrid + vb;
    // band walk: contiguous band groups per warp; else quads, lanes interleaved
    const bool band = fa0.band_h > 0;
    const unsigned total = band ? fa0.band_groups
                                : (unsigned)fa0.G.n_sim * (unsigned)fa0.G.rows * ((unsigned)fa0.G.Wp >> 2);
    const unsigned per = band ? (total + nc - 1) / nc : (((total + nc - 1) / nc + 31) & ~31u);
    unsigned lo = min(total, cw * per), hi = min(total, lo + per);
    // (also the flag path of single-segment lattices when a warp has several
    // groups and every CTA's block spans several replicas, so that the
    // blocks mix temperatures: cfg3 2.957 -> 2.984 T)
    const bool many_replicas = !GFX && per >= 2 && (unsigned)fa0.G.n_sim >= 4u * vgrid;
    if (kCtaBlocks && DIRECT && (GFX || many_replicas) && band && vgrid == gridDim.x) {
      // Direct flips in the general group order (rows in segments, one slab
      // per launch): a CTA's warps take one contiguous block of groups
      // (floor / ceil(total / CTAs) of them), so most neighbour groups live
      // on the same SM: a warp that waits there leaves its issue slots to
      // exactly the warps it waits for, and only the block's edge groups
      // depend on another SM's progress (cfg4 philox-bits 2.45 -> 2.64 T,
      // cfg5 unchanged).  Measured worse for the two-neighbour flag path of
      // single-segment lattices (cfg2 2.99 -> 2.85 T, one group per warp)
      // and for rings (cfg4 in 8 slabs 2.24 -> 2.18 T), which keep the
      // interleaved ranges.
      const unsigned c_lo = (unsigned)((unsigned long long)vb * total / vgrid);
      const unsigned c_hi = (unsigned)((unsigned long long)(vb + 1) * total / vgrid);
      const unsigned pw = (c_hi - c_lo + (unsigned)nwc - 1) / (unsigned)nwc;
      lo = min(c_hi, c_lo + (unsigned)(warp - pwarps) * pw);
      hi = min(c_hi, lo + pw);
    }
    if (kChunkMap && DIRECT && !GFX && band && per == 1 && nwc % kChunkMap == 0) {
      // One group per warp (cfg2): chunks of kChunkMap consecutive groups
      // per CTA, the chunks interleaved over the CTAs.  Half of the neighbour
      // pairs then share an SM (see the block mapping above) while every SM
      // still gets groups of every replica, i.e. of every temperature --
      // whole blocks gave an SM the groups of one replica and the SMs of the
      // hot replicas (more draws) became the launch's critical path.
      // Measured at cfg2: chunks of 2 3.017, 4 3.030, 7 3.006, 14 2.955 T
      // against 2.991 interleaved.
      const unsigned w = (unsigned)(warp - pwarps), idx = (w / kChunkMap) * vgrid + vb;
      lo = min(total, idx * kChunkMap + w % kChunkMap);
      hi = min(total, lo + 1);
    }
    const unsigned i0 = lo + (threadIdx.x & 31);
    FlipArgs fa = fa0;
    unsigned cnt = 0;
    const bool leader = threadIdx.x == pwarps * 32;
    const bool gpu_leader = leader && vb == 0;
    const unsigned fbase = flags_base(wa);  // phases completed by earlier flag launches
    const bool gf = GFX && band && wa.flags != nullptr;
    if (HALO && !gf) halo_gate(ha, wa, fbase, -1, true, nwc * 32, leader, gpu_leader, vgrid);
    const unsigned base = pro ? vgrid : 0u;  // the prologue's arrivals on work[1]
    const bool epi = !HALO && (io.lin_out != nullptr || io.ups != nullptr);
    if (!HALO && io.ups != nullptr && vb == 0)  // written, not added (ordered by the barriers below)
      for (int j = threadIdx.x - pwarps * 32; j < fa0.G.n_sim; j += nwc * 32) io.ups[j] = io.unsat[j] = 0;
    if (pro) {
      if (leader) {
        while (ld_acquire(wa.work + 1) < base) __nanosleep(64);
        __threadfence();
      }
      asm volatile("bar.sync 1, %0;" ::"r"(nwc * 32) : "memory");
    }
    const bool gflag_path = DIRECT && !GFX && !HALO && wa.flags && band && fa.band_nseg == 1;
    unsigned epi_bar = 1;  // the epilogue barrier's index among this launch's consumer barriers
    // n = 512 rows packed in place for the flips (FlipArgs::pks): thread
    // share of the rows
    const unsigned ct = cw * 32u + (threadIdx.x & 31), nct = nc * 32u;
    const unsigned nrows = (unsigned)fa0.G.n_sim * 2u * (unsigned)fa0.G.R;
    bool push_warp = true;  // HALO: this warp's bands include a slab's first or last row
    if (HALO && band && !gf) {
      const unsigned gps = (unsigned)fa0.G.rows / (unsigned)(fa0.band_gb * fa0.band_h), nseg = (unsigned)fa0.band_nseg;
      push_warp = false;
      for (unsigned g = lo; g < hi; g++) {
        const unsigned l = (g / nseg) % gps;
        push_warp |= l == 0 || l + 1 == gps;
      }
    }
    if (gflag_path) {
      // band groups in phase order, neighbour flags instead of grid barriers
      unsigned* gflags = flags_groups(wa);
      const unsigned gps = (unsigned)fa0.G.rows / (unsigned)(fa0.band_gb * fa0.band_h);
      // n = 512 on packed rows: a packed word (t, t + 4) is one whole 32-draw
      // group, so the 32-draw walk applies (DIRECT = 32 over CB = 16 rows)
      constexpr bool kPksD = CB == 16 && DIRECT == 32;
      const bool pksd = kPksD && fa0.pks;
      unsigned nb = 0;
      int kt_s = -1;  // replica whose key masks the warp's table holds (direct_group_split)
      unsigned gs = 0, gl = 0;  // replica and band of the current group (direct_group_split)
      if (pksd) {
        pack_rows<false>(fa0.spins, nrows, ct, nct);
        consumer_barrier(wa.work + 1, base + vgrid * ++nb, nwc * 32, leader);
      }
      for (int i = 0; i < 2 * count; i++) {
        const int X = i & 1;
        PbitsDirect dp;
        dp.thr9 = wa.thr9;
        dp.pk = wa.pk;
        dp.blk = wa.block0 + 2ull * (unsigned)(first + (i >> 1)) + (unsigned)X;
        if constexpr (kDirectSplit && DIRECT == 32) {
          // (replica, band) of the groups, stepped from the warp's first one.
          // (Taking the range's first and last group -- the ones whose
          // neighbours another warp owns -- after the interior ones, to give
          // the neighbour warps a phase of slack, measured no gain: cfg3
          // 2.949 against 2.954 T.)
          uint32_t* st = reinterpret_cast<uint32_t*>(jt) + (size_t)warp * kSplitWords;
          gs = lo / gps;
          gl = lo - gs * gps;
          for (unsigned g = lo; g < hi; g++) {
            if (i > 0) group_wait_at(gflags, g, gl, gps, fbase + (unsigned)i);
            if (kPksD && pksd) cnt += direct_group_split<kPksD>(fa, gs, gl, 0u, X, dp, st, kt_s);
            else cnt += direct_group_split<false>(fa, gs, gl, 0u, X, dp, st, kt_s);
            group_done(gflags, g, fbase + (unsigned)i + 1u);
            if (++gl == gps) {
              gl = 0;
              gs++;
            }
          }
        }
        for (unsigned g = lo; g < hi; g++) {
          if constexpr (kDirectSplit && DIRECT == 32) {
            break;
          } else {
            if (i > 0) group_wait(gflags, g, gps, fbase + (unsigned)i);
            if (kPksD && pksd) cnt += flip_band_run<true, false, false, DIRECT, true, NoHooks, false, kPksD>(fa, g, g + 1, X, &dp);
            else if (i == 0 && !pro) cnt += flip_band_run<false, false, false, DIRECT>(fa, g, g + 1, X, &dp);
            else cnt += flip_band_run<true, false, false, DIRECT>(fa, g, g + 1, X, &dp);
            group_done(gflags, g, fbase + (unsigned)i + 1u);
          }
        }
      }
      if (pksd) {
        consumer_barrier(wa.work + 1, base + vgrid * ++nb, nwc * 32, leader);
        pack_rows<true>(fa0.spins, nrows, ct, nct);
      }
      epi_bar = nb + 1;
    } else if (GFX && gf) {
      // general band-group order: whole lattices with rows in several
      // segments, and slabs, whose edge bands alone wait on the neighbours.
      // One walk instantiation (GFX == 2: segment walk, valid for any row;
      // 1: single-segment rows); always through L2 (neighbour groups may
      // already be a phase ahead).
      GroupOrder go;
      go.grp = flags_groups(wa);
      go.above = flags_above(wa);
      go.below = flags_below(wa);
      go.up_below = ha.up_below;
      go.down_above = ha.down_above;
      go.gps = (unsigned)fa0.G.rows / (unsigned)(fa0.band_gb * fa0.band_h);
      go.nseg = (unsigned)fa0.band_nseg;
      constexpr bool GSEG = GFX == 2;
      int kt_s = -1;  // replica whose key masks the warp's table holds (direct_group_split)
      for (int i = 0; i < 2 * count; i++) {
        const int X = i & 1;
        PbitsDirect dp;
        if (DIRECT) {
          dp.thr9 = wa.thr9;
          dp.pk = wa.pk;
          dp.blk = wa.block0 + 2ull * (unsigned)(first + (i >> 1)) + (unsigned)X;
        } else {
          fa.planes = cur + (size_t)(first + (i >> 1)) * wa.slot_words;
        }
        constexpr bool PG = DIRECT != 0;
        const GfHooks<HALO, PG> hk{&go, fbase + (unsigned)i, lo, hi, i > 0, HALO || i > 0};
        if constexpr (kDirectSplit && DIRECT == 32) {
          // the split form over the general group order (the hooks' cursor is the group's (s, l, seg))
          uint32_t* st = reinterpret_cast<uint32_t*>(jt) + (size_t)warp * kSplitWords;
          for (unsigned g = lo; g < hi; g++) {
            hk.pre(g);
            cnt += direct_group_split<false, GSEG, HALO>(fa, hk.cs, hk.cl, hk.cseg, X, dp, st, kt_s);
            hk.post(g);
          }
          continue;
        }
        cnt += flip_band_run<true, HALO, GSEG, DIRECT, true, GfHooks<HALO, PG>, CB == 16 && !DIRECT>(fa, lo, hi, X, &dp, hk);
        if (!PG) gf_publish_cta<HALO>(go, fbase + (unsigned)i + 1u, per, total, nwc, vgrid, vb, leader);
      }
    } else {
    // n = 512 window flips on packed rows (FlipArgs::pks): packed in place
    // by the consumer warps after the prologue, unpacked after the last phase
    constexpr bool kPks = CB == 16 && !DIRECT && !HALO && !GFX;
    const bool pks = kPks && band && fa0.pks;
    unsigned nbar = 0;  // consumer barriers of this launch after the prologue's
    if (pks) {
      pack_rows<false>(fa0.spins, nrows, ct, nct);
      consumer_barrier(wa.work + 1, base + vgrid * ++nbar, nwc * 32, leader);
    }
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
      if constexpr (!GFX) {  // (GFX kernels get flags from the host: a band walk is always gf)
        if (band) {
          constexpr bool PK = CB == 16 && !DIRECT;
          if (fa.band_nseg > 1) {  // wide rows (cfg4, cfg5): segment-edge words from memory
            if (HALO) cnt += flip_band_run<true, true, true, DIRECT>(fa, lo, hi, X, &dp);
            else if (i == 0 && !pro) cnt += flip_band_run<false, false, true, DIRECT>(fa, lo, hi, X, &dp);
            else cnt += flip_band_run<true, false, true, DIRECT>(fa, lo, hi, X, &dp);
          } else if (kPks && pks) {
            cnt += flip_band_run<true, false, false, DIRECT, true, NoHooks, PK, kPks>(fa, lo, hi, X, &dp);
          } else {
            if (HALO) cnt += flip_band_run<true, true, false, DIRECT, true, NoHooks, PK>(fa, lo, hi, X, &dp);
            else if (i == 0 && !pro) cnt += flip_band_run<false, false, false, DIRECT, true, NoHooks, PK>(fa, lo, hi, X, &dp);
            else cnt += flip_band_run<true, false, false, DIRECT, true, NoHooks, PK>(fa, lo, hi, X, &dp);
          }
        }
      }
      if (!band && !DIRECT) {
        if (HALO) cnt += flip_run<true, true>(fa, i0, hi, X);
        else if (i == 0 && !pro) cnt += flip_run<false>(fa, i0, hi, X);
        else cnt += flip_run<true>(fa, i0, hi, X);
      }
      const bool more = i + 1 < 2 * count;
      if (HALO) {
        // the halo pushes (peer stores) before the neighbours are told; only
        // warps holding a slab's first or last row push
        if (push_warp) __threadfence_system();
        halo_gate(ha, wa, fbase, i, more, nwc * 32, leader, gpu_leader, vgrid);
      } else if (more) {
#ifdef MSB_TRACE
        if (i == 0) MSB_TRACE_PUT(6, gtimer());  // first phase done (before its barrier)
#endif
        consumer_barrier(wa.work + 1, base + vgrid * ++nbar, nwc * 32, leader);
      }
    }
    if (pks) {
      consumer_barrier(wa.work + 1, base + vgrid * ++nbar, nwc * 32, leader);
      pack_rows<true>(fa0.spins, nrows, ct, nct);
    }
    if (epi) nbar++;  // the epilogue's barrier below
    epi_bar = nbar;
    }
    add_flips(fa.flips, cnt);
#ifdef MSB_TRACE
    MSB_TRACE_PUT(7, gtimer());  // flips done (before the epilogue)
#endif
    if (epi) {  // every flip of the launch is done before any export read
      // (the flag paths have no per-phase grid barriers: this is their first)
      consumer_barrier(wa.work + 1, base + vgrid * (gf ? 1u : epi_bar), nwc * 32, leader);
      if (io.lin_out && io.ups) win_export<true, true>(fa0.G, fa0.spins, io, cw, nc);
      else if (io.lin_out) win_export<true, false>(fa0.G, fa0.spins, io, cw, nc);
      else win_export<false, true>(fa0.G, fa0.spins, io, cw, nc);
    }
  }
#ifdef MSB_TRACE
  MSB_TRACE_PUT(2, gtimer());
#endif
  finish_launch(wa, total_warps, count > 0 ? 2u * (unsigned)count : 0u);
}

// RING: a ring launch over nv slabs (SlabCtx per slab in device memory);
// the grid's CTAs are split into nv contiguous equal parts, one per slab.
template <int SRC, int CB, bool HALO, int DIRECT = 0, int NT = 0, int GFX = 0, bool RING = false>
__global__ void __launch_bounds__(NT ? NT : (DIRECT ? kDirectThreads : kRngThreads), 1)
    k_win(const WinArgs wa, const FlipArgs fa0, const HaloArgs ha, const WinIO io, const uint32_t* cur, int first,
          int count, int pwarps, const SlabCtx* __restrict__ ring, int nv) {
  extern __shared__ uint4 jt[];
  if (RING) {
    const unsigned vg = gridDim.x / (unsigned)nv, v = blockIdx.x / vg;
    if (v >= (unsigned)nv) return;
    const SlabCtx& c = ring[v];
    win_body<SRC, CB, HALO, DIRECT, GFX>(c.wa, c.fa, c.ha, io, c.cur, first, count, pwarps, blockIdx.x - v * vg, vg,
                                         jt);
  } else {
    win_body<SRC, CB, HALO, DIRECT, GFX>(wa, fa0, ha, io, cur, first, count, pwarps, blockIdx.x, gridDim.x, jt);
  }
}

// Halo wait: until both neighbours completed the phases counted in our flag
// header (their pushes into our ghost rows landed), e.g. before the
// observables of a slab.  Every slot of both directions.
__global__ void k_halo_wait(const unsigned* flags, unsigned nslot) {
  const unsigned need = ld_acquire(flags);
  for (unsigned j = threadIdx.x; j < 2 * nslot; j += blockDim.x)
    while (ld_acquire_sys(flags + 1 + j) < need) __nanosleep(128);
  __threadfence_system();
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

// Halo slots per direction of a flag buffer: one per (replica, row segment).
inline int g_nslot(const FlipArgs& fa) { return fa.G.n_sim * std::max(1, fa.band_nseg); }

int check_halo(const msb_geom* g, const msb_sweep_params* p, const msb_halo* halo, int count) {
  if (count > 0 && g->ghost && !halo) return fail(MSB_ERR_ARG, "slab windows flip with an msb_halo (in-kernel exchange)");
  if (halo && !g->ghost) return fail(MSB_ERR_ARG, "msb_halo needs a slab geometry (ghost = 1)");
  if (halo && (!halo->up_spins || !halo->down_spins || !halo->up_flags || !halo->down_flags || halo->up_R < 4 ||
               halo->down_R < 4))
    return fail(MSB_ERR_ARG, "incomplete msb_halo");
  if (halo && !p->flags) return fail(MSB_ERR_ARG, "slab launches need msb_sweep_params.flags (msb_flag_words)");
  return MSB_OK;
}

void set_halo(const msb_halo* halo, int count, FlipArgs& fa, HaloArgs& ha) {
  ha = HaloArgs{};
  if (halo && count > 0) {
    fa.up_spins = halo->up_spins;
    fa.down_spins = halo->down_spins;
    fa.up_R = halo->up_R;
    fa.down_R = halo->down_R;
    // the neighbours' flag buffers: we write the slab above's "from below"
    // slots and the slab below's "from above" slots
    const unsigned nslot = (unsigned)g_nslot(fa);
    ha.up_below = reinterpret_cast<unsigned*>(halo->up_flags) + 1 + nslot;
    ha.down_above = reinterpret_cast<unsigned*>(halo->down_flags) + 1;
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
  w.flags = reinterpret_cast<unsigned*>(p->flags);
  w.nslot = 0;  // set with the flip geometry (g_nslot)
}

int sm_count(int* sms) {
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  CUDA_TRY(cudaDeviceGetAttribute(sms, cudaDevAttrMultiProcessorCount, dev));
  return MSB_OK;
}

template <int SRC, int CB, bool HALO, int DIRECT, int NT, int GFX, bool RING>
int launch_k_win(const cudaLaunchConfig_t& cfg, const WinArgs& wa, const FlipArgs& fa, const HaloArgs& ha,
                 const WinIO& wio, const uint32_t* cur, int first, int count, int pwarps, const SlabCtx* ring, int nv) {
  static std::once_flag o_;
  static cudaError_t e_;
  if (int r = set_smem_attr(k_win<SRC, CB, HALO, DIRECT, NT, GFX, RING>, o_, e_)) return r;
  CUDA_TRY(cudaLaunchKernelEx(&cfg, k_win<SRC, CB, HALO, DIRECT, NT, GFX, RING>, wa, fa, ha, wio, cur, first, count,
                              pwarps, ring, nv));
  return MSB_OK;
}

// Window instantiations of one stream kind: whole lattices with grid
// barriers or group flags, slabs (group flags; GPU-wide gate when there is
// no band walk), one slab or a ring of them per launch.
template <int SRC, bool HALO, int GFX, bool RING>
int launch_window_cb(int cb, const cudaLaunchConfig_t& cfg, const WinArgs& wa, const FlipArgs& fa, const HaloArgs& ha,
                     const WinIO& wio, const uint32_t* cur, int first, int count, int pwarps, const SlabCtx* ring,
                     int nv) {
  if (cb == 32) return launch_k_win<SRC, 32, HALO, 0, 0, GFX, RING>(cfg, wa, fa, ha, wio, cur, first, count, pwarps, ring, nv);
  if (cb == 16) return launch_k_win<SRC, 16, HALO, 0, 0, GFX, RING>(cfg, wa, fa, ha, wio, cur, first, count, pwarps, ring, nv);
  return launch_k_win<SRC, 0, HALO, 0, 0, GFX, RING>(cfg, wa, fa, ha, wio, cur, first, count, pwarps, ring, nv);
}

// Direct instantiations (bit-plane Philox, every warp flips).
template <bool HALO, int GFX, bool RING, int NT>
int launch_direct(int cb, const cudaLaunchConfig_t& cfg, const WinArgs& wa, const FlipArgs& fa, const HaloArgs& ha,
                  const WinIO& wio, int count, const SlabCtx* ring, int nv) {
  // NT = 896 is a 32-draw-row shape, NT = 768 an n = 512 one (direct_run_impl)
  if (cb == 32) {
    if constexpr (NT != 768) return launch_k_win<kSrcPbits, 32, HALO, 32, NT, GFX, RING>(cfg, wa, fa, ha, wio, nullptr, 0, count, 0, ring, nv);
  } else {
    if constexpr (NT != 896) return launch_k_win<kSrcPbits, 16, HALO, 16, NT, GFX, RING>(cfg, wa, fa, ha, wio, nullptr, 0, count, 0, ring, nv);
  }
  return fail(MSB_ERR_ARG, "direct launch shape");
}

// n = 512 direct sweeps on packed rows (FlipArgs::pks): the 32-draw walk
// over 16-site rows packed in place.
template <int NT>
int launch_direct_pks(const cudaLaunchConfig_t& cfg, const WinArgs& wa, const FlipArgs& fa, const HaloArgs& ha,
                      const WinIO& wio, int count) {
  return launch_k_win<kSrcPbits, 16, false, 32, NT, 0, false>(cfg, wa, fa, ha, wio, nullptr, 0, count, 0, nullptr, 0);
}

cudaLaunchConfig_t coop_config(unsigned grid, unsigned threads, size_t smem, void* stream, cudaLaunchAttribute* attr,
                               bool coop) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = as_stream(stream);
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = coop ? 1 : 0;
  return cfg;
}

// Producer warps per 32-warp CTA of a window launch with `units` warp-units
// of pieces over `ctas` CTAs.  A unit (32 pieces) is a whole window's share
// of a stream, so an extra producer round costs a full unit: when the units
// fit one round, give producers exactly that round and the rest of the CTA
// to the flips; otherwise 8 flip warps (flip-heavy shapes gain, others are
// insensitive).  Producers are capped so the plane rows being written stay
// L2-resident (see msb_window_parts).  MSB_FLIP_WARPS / MSB_PRODUCER_WARPS
// override (tuning).
int producer_warps(long long units, int ctas, int Wp, int P, bool produce, int count, bool whole = false,
                   int S = 8) {
  static const int env_pw = [] { const char* e = getenv("MSB_PRODUCER_WARPS"); return e ? atoi(e) : 0; }();
  static const int env_cw = [] { const char* e = getenv("MSB_FLIP_WARPS"); return e ? atoi(e) : 0; }();
  // bytes of plane rows a producer warp has open: 2 rows (planes) per row
  // being written, 32 / max(1, P/8) rows per warp (win_piece numbering)
  const long long live_per_warp = 32LL * 2 * 4 * Wp / std::max(1, P / 8);
  const int cap = (int)std::max(4LL, std::min(32LL, (100LL << 20) / ((long long)ctas * live_per_warp)));
  int pwarps = 0;
  if (produce) {
    if (count == 0) {
      pwarps = cap;
    } else {
      const long long one_round = (units + ctas - 1) / ctas;  // producer warps per CTA for a single round
      int cw = one_round <= 30 ? (int)(32 - one_round) : 8;
      if (one_round > 30 && whole) {
        // Several rounds (whole lattices): the producers are ALU-bound, so a
        // round of pw units per SM lasts ~pw unit-times and the window
        // ~pw * ceil(units / (ctas pw)); take the pw in [24, 28] that
        // minimises it.  Ties: 28 for long windows (the flip warps' per-launch
        // work, the n = 512 row packing, is amortised; cfg3 at S = 32: 4 flip
        // warps 0.963 T, 8: 0.951), 24 for short ones (S = 8: 8 flip warps
        // 0.936, 4: 0.904).
        long long best = -1;
        for (int pw = 24; pw <= 28; pw++) {
          const long long cost = (long long)pw * ((units + (long long)ctas * pw - 1) / ((long long)ctas * pw));
          if (best < 0 || cost < best || (cost == best && S >= 16)) {
            best = cost;
            cw = 32 - pw;
          }
        }
      }
      if (env_cw > 0) cw = std::min(28, env_cw);
      pwarps = std::min(cap, 32 - cw);
    }
    if (env_pw > 0) pwarps = std::min(32, env_pw);
  }
  return pwarps;
}

// Band height of a slab's window flips: the default (tallest) band, or
// MSB_BAND_H (tuning).  Measured at cfg4 (one slab, and a ring of 8 slabs of
// 1792 rows on 18 SMs each, where 16-row bands leave a third of the flip
// warps without a group): 16 rows 0.941 / 0.850 T, 8: 0.938 / 0.845, 4:
// 0.918 / 0.833, 2: 0.853 / 0.786 -- a band's setup and its group waits
// cost more than the idle flip warps.  The flag buffer is sized for 2-row
// bands (msb_flag_words).
void fit_band_h(FlipArgs& fa, const msb_geom* g) {
  if (fa.band_h <= 0) return;
  const int gb = fa.band_gb;
  static const int env_h = [] { const char* e = getenv("MSB_BAND_H"); return e ? atoi(e) : 0; }();
  if (env_h >= 2 && env_h <= fa.band_h && !(env_h & (env_h - 1)) && g->rows % (gb * env_h) == 0) {
    fa.band_h = env_h;
    fa.band_groups = (unsigned)((long long)g->n_sim * g->rows / (gb * env_h) * fa.band_nseg);
  }
}

// compile-time chunk width: every chunk 32 draws (n/32 % 32 == 0), a single
// 16-draw chunk (n = 512), or generic
int chunk_width(const Geo& G) { return (G.words % 32) == 0 ? 32 : (G.words == 16 ? 16 : 0); }

// One window slab/lattice launch's kernel arguments (checks included).
int plan_window(const msb_geom* g, const msb_sweep_params* p, int S, int P, uint32_t* spins, uint32_t* states,
                const uint32_t* cur, int first, int count, uint32_t* next, uint64_t* flips, const msb_halo* halo,
                const msb_window_io* io, WinArgs& wa, FlipArgs& fa, HaloArgs& ha, WinIO& wio, long long& np) {
  if (int r = check_window(g, S, P, &np)) return r;
  if (int r = check_params(p)) return r;
  if (p->mode == MSB_MODE_GENERIC) return fail(MSB_ERR_UNSUPPORTED, "lookahead windows need FERRO/ANTI tables");
  if (first < 0 || count < 0 || first + count > S) return fail(MSB_ERR_ARG, "slots [first, first+count) outside the window");
  if (count > 0 && (!spins || !cur || !flips)) return fail(MSB_ERR_ARG, "null buffer");
  if (int r = check_halo(g, p, halo, count)) return r;
  if (count > 0)
    if (int r = check_flip_extent(g, 2)) return r;
  if (int r = make_win_io(g, io, count, halo, wio)) return r;
  if (next && p->rng == MSB_RNG_XOSHIRO && (!states || !p->jump)) return fail(MSB_ERR_ARG, "null RNG state or jump table");
  fill_win_args(wa, g, p, S, P, np, states, next);
  fill_flip_args(fa, g, p, 0, spins, cur, flips);
  // the producer's packed n = 512 planes (one 32-draw run fills t(k) and t(k + 1) = t(k) + 4)
  fa.pk16 = chunk_width(wa.G) == 16 && wa.kr % 2 == 0 && p->rng != MSB_RNG_PHILOX;
  wa.nslot = (unsigned)g_nslot(fa);
  set_halo(halo, count, fa, ha);
  // n = 512 whole lattices: the window's flips run on packed rows (two
  // 16-site words per uint32, FlipArgs::pks), lanes = 2 quads per row.
  // MSB_PACK16=0: the 16-bit words as they are (tuning / comparison).
  static const int env_pk = [] { const char* e = getenv("MSB_PACK16"); return e ? atoi(e) : 1; }();
  if (env_pk && fa.pk16 && !ha.on && count > 0 && fa.band_h > 0 && wa.G.words == 16 && wa.G.nch == 1) {
    for (int h = 16; h >= 2; h >>= 1)
      if (g->rows % (16 * h) == 0) {
        fa.pks = 1;
        fa.band_sq = 2;
        fa.band_gb = 16;
        fa.band_nseg = 1;
        fa.band_h = h;
        fa.band_groups = (unsigned)((long long)g->n_sim * g->rows / (16 * h));
        break;
      }
  }
  return MSB_OK;
}

// One direct launch's kernel arguments (checks included).
int plan_direct(const msb_geom* g, const msb_sweep_params* p, uint32_t* spins, int n_sweeps, uint64_t* flips,
                const msb_halo* halo, const msb_window_io* io, WinArgs& wa, FlipArgs& fa, HaloArgs& ha, WinIO& wio,
                int& cb) {
  if (int r = check_geom(g)) return r;
  if (int r = check_params(p)) return r;
  if (p->rng != MSB_RNG_PHILOX_BITS) return fail(MSB_ERR_ARG, "direct sweeps draw the bit-plane Philox stream");
  if (p->mode == MSB_MODE_GENERIC) return fail(MSB_ERR_UNSUPPORTED, "direct sweeps need FERRO/ANTI tables");
  if (n_sweeps < 0 || n_sweeps > (1 << 20)) return fail(MSB_ERR_ARG, "sweep count must be in [0, 2^20]");
  if (n_sweeps > 0 && (!spins || !flips)) return fail(MSB_ERR_ARG, "null buffer");
  if (int r = check_halo(g, p, halo, n_sweeps)) return r;
  if (int r = check_flip_extent(g, 2)) return r;
  if (int r = make_win_io(g, io, n_sweeps, halo, wio)) return r;
  const Geo G = make_geo(g);
  cb = chunk_width(G) == 32 ? 32 : (G.words == 16 ? 16 : 0);
  fill_flip_args(fa, g, p, 0, spins, nullptr, flips);
  if (!cb || !direct_band(fa, g)) return fail(MSB_ERR_UNSUPPORTED, "direct sweeps need n/32 % 32 == 0 or n = 512 and band rows");
  set_halo(halo, n_sweeps, fa, ha);
  wa = WinArgs{};
  wa.G = G;
  wa.thr9 = p->thr9;
  wa.work = p->work;
  wa.pk = philox_keys(p->seed);
  wa.block0 = p->block;
  wa.seed_lo = (uint32_t)p->seed;
  wa.seed_hi = (uint32_t)(p->seed >> 32);
  wa.flags = reinterpret_cast<unsigned*>(p->flags);
  wa.nslot = (unsigned)g_nslot(fa);
  return MSB_OK;
}


// ---------------------------------------------------------------------------
// launch drivers, instantiated per stream kind in their own translation
// units (msb_win_xo.cu, msb_win_philox.cu, msb_win_pbits.cu, msb_direct.cu)
// ---------------------------------------------------------------------------

// One window launch (ring = false: slabs[0] alone, with io) or a ring launch.
template <int SRC>
int window_run(int nslabs, const msb_ring_slab* slabs, bool ring, int S, int P, int first, int count,
               const msb_window_io* io, void* ctx, void* stream) {
  int sms = 148;
  if (!ring) {
    const msb_ring_slab& r = slabs[0];
    WinArgs wa;
    FlipArgs fa;
    HaloArgs ha;
    WinIO wio;
    long long np = 0;
    if (int e = plan_window(r.g, r.p, S, P, r.spins, r.states, r.cur, first, count, r.next, r.flips, r.halo, io, wa,
                            fa, ha, wio, np))
      return e;
    if (int e = sm_count(&sms)) return e;
    const int pwarps = producer_warps((np + 31) / 32, sms, fa.G.Wp, P, r.next != nullptr, count, !ha.on, S);
    if (ha.on) fit_band_h(fa, r.g);
    const int cb = chunk_width(wa.G);
    const bool pj = SRC == kSrcXoshiro && pwarps > 0;
    cudaLaunchAttribute attr[1];
    const cudaLaunchConfig_t cfg = coop_config((unsigned)sms, kRngThreads, pj ? (size_t)kJumpWords * 4 : 0, stream,
                                               attr, count > 0);  // grid barriers only among consumers
    if (ha.on) return launch_window_cb<SRC, true, 2, false>(cb, cfg, wa, fa, ha, wio, r.cur, first, count, pwarps, nullptr, 0);
    return launch_window_cb<SRC, false, 0, false>(cb, cfg, wa, fa, ha, wio, r.cur, first, count, pwarps, nullptr, 0);
  }
  SlabCtx host[MSB_RING_MAX];
  long long units = 0;
  int cb = -1, mode = -1;
  bool next_all = true, next_any = false;
  for (int v = 0; v < nslabs; v++) {
    const msb_ring_slab& r = slabs[v];
    if (!r.g || !r.halo) return fail(MSB_ERR_ARG, "ring slabs need a geometry and an msb_halo");
    WinIO wio;
    long long np = 0;
    if (int e = plan_window(r.g, r.p, S, P, r.spins, r.states, r.cur, first, count, r.next, r.flips, r.halo, nullptr,
                            host[v].wa, host[v].fa, host[v].ha, wio, np))
      return e;
    host[v].cur = r.cur;
    units = std::max(units, (np + 31) / 32);
    const int c = chunk_width(host[v].wa.G);
    if (v > 0 && (c != cb || r.p->mode != mode))
      return fail(MSB_ERR_ARG, "ring slabs must share the stream kind, the row width and the table mode");
    cb = c;
    mode = r.p->mode;
    next_all &= r.next != nullptr;
    next_any |= r.next != nullptr;
  }
  if (next_any != next_all) return fail(MSB_ERR_ARG, "either every ring slab produces its next window or none");
  if (int e = sm_count(&sms)) return e;
  const int vg = sms / nslabs;
  if (vg < 1) return fail(MSB_ERR_UNSUPPORTED, "more slabs than SMs");
  const int pwarps = producer_warps(units, vg, host[0].fa.G.Wp, P, next_all, count);
  for (int v = 0; v < nslabs; v++) fit_band_h(host[v].fa, slabs[v].g);
  CUDA_TRY(cudaMemcpyAsync(ctx, host, sizeof(SlabCtx) * nslabs, cudaMemcpyHostToDevice, as_stream(stream)));
  const bool pj = SRC == kSrcXoshiro && pwarps > 0;
  cudaLaunchAttribute attr[1];
  const cudaLaunchConfig_t cfg =
      coop_config((unsigned)(vg * nslabs), kRngThreads, pj ? (size_t)kJumpWords * 4 : 0, stream, attr, true);
  return launch_window_cb<SRC, true, 2, true>(cb, cfg, host[0].wa, host[0].fa, host[0].ha, WinIO{}, nullptr, first,
                                                 count, pwarps, reinterpret_cast<const SlabCtx*>(ctx), nslabs);
}

// One direct launch (ring = false: slabs[0] alone, with io) or a ring launch.
template <int = 0>
int direct_run_impl(int nslabs, const msb_ring_slab* slabs, bool ring, int n_sweeps, const msb_window_io* io,
                           void* ctx, void* stream) {
  int sms = 148;
  if (!ring) {
    const msb_ring_slab& r = slabs[0];
    WinArgs wa;
    FlipArgs fa;
    HaloArgs ha;
    WinIO wio;
    int cb = 0;
    if (int e = plan_direct(r.g, r.p, r.spins, n_sweeps, r.flips, r.halo, io, wa, fa, ha, wio, cb)) return e;
    if (n_sweeps == 0) return MSB_OK;
    if (int e = sm_count(&sms)) return e;
    cudaLaunchAttribute attr[1];
    cudaLaunchConfig_t cfg = coop_config((unsigned)sms, kDirectThreads, 0, stream, attr, true);
    if (kDirectSplit) cfg.dynamicSmemBytes = (size_t)(kDirectThreads / 32) * kSplitWords * 4;  // the warps' stashes
    if (ha.on) return launch_direct<true, 2, false, 0>(cb, cfg, wa, fa, ha, wio, n_sweeps, nullptr, 0);
    // rows in several segments: the general group order (flags) or grid barriers
    if (fa.band_nseg > 1) {
      if (wa.flags) return launch_direct<false, 2, false, 0>(cb, cfg, wa, fa, ha, wio, n_sweeps, nullptr, 0);
      return launch_direct<false, 0, false, 0>(cb, cfg, wa, fa, ha, wio, n_sweeps, nullptr, 0);
    }
    // Band groups that fit one per warp in 28 warps per SM (cfg2: 4096
    // groups, 148 x 28 = 4144 warps) run 896-thread CTAs: no warp idles, and
    // ptxas gets 72 registers instead of 64.  Many groups per warp (cfg3:
    // 24128 groups, ~5 per warp): 768-thread CTAs give ptxas 80 registers,
    // and the extra groups per warp cost little (measured 1.49 vs 1.45 T).
    static const int env_nt = [] { const char* e = getenv("MSB_DIRECT_NT"); return e ? atoi(e) : -1; }();
    const long long g28 = 28LL * sms, g24 = 24LL * sms;
    // n = 512 with group flags: rows packed in place, two 16-draw words per
    // uint32, i.e. one whole 32-draw group per word (MSB_PACK16=0: off)
    static const int env_pk = [] { const char* e = getenv("MSB_PACK16"); return e ? atoi(e) : 1; }();
    if (cb == 16 && env_pk && wa.flags && fa.G.nch == 1 && r.g->rows % 32 == 0) {
      fa.pks = 1;
      fa.band_sq = 2;
      fa.band_gb = 16;
      fa.band_nseg = 1;
      fa.band_h = 2;
      fa.band_groups = (unsigned)((long long)r.g->n_sim * r.g->rows / 32);
      if (env_nt == 768) {
        cfg.blockDim = dim3(768);
        return launch_direct_pks<768>(cfg, wa, fa, ha, wio, n_sweeps);
      }
      if (env_nt != 0 && (long long)fa.band_groups <= g28 && (long long)fa.band_groups > g24) {
        cfg.blockDim = dim3(896);
        return launch_direct_pks<896>(cfg, wa, fa, ha, wio, n_sweeps);
      }
      return launch_direct_pks<0>(cfg, wa, fa, ha, wio, n_sweeps);
    }
    if (cb == 32 && env_nt != 0 && (long long)fa.band_groups <= g28 && (long long)fa.band_groups > g24) {
      cfg.blockDim = dim3(896);
      return launch_direct<false, 0, false, 896>(cb, cfg, wa, fa, ha, wio, n_sweeps, nullptr, 0);
    }
    if (cb == 16 && env_nt != 0 && (long long)fa.band_groups >= 4LL * 32 * sms) {
      cfg.blockDim = dim3(768);
      return launch_direct<false, 0, false, 768>(cb, cfg, wa, fa, ha, wio, n_sweeps, nullptr, 0);
    }
    return launch_direct<false, 0, false, 0>(cb, cfg, wa, fa, ha, wio, n_sweeps, nullptr, 0);
  }
  SlabCtx host[MSB_RING_MAX];
  int cb = -1;
  for (int v = 0; v < nslabs; v++) {
    const msb_ring_slab& r = slabs[v];
    if (!r.g || !r.halo) return fail(MSB_ERR_ARG, "ring slabs need a geometry and an msb_halo");
    WinIO wio;
    int c = 0;
    if (int e = plan_direct(r.g, r.p, r.spins, n_sweeps, r.flips, r.halo, nullptr, host[v].wa, host[v].fa, host[v].ha,
                            wio, c))
      return e;
    host[v].cur = nullptr;
    if (v > 0 && c != cb) return fail(MSB_ERR_ARG, "ring slabs must share the row width");
    cb = c;
  }
  if (n_sweeps == 0) return MSB_OK;
  if (int e = sm_count(&sms)) return e;
  const int vg = sms / nslabs;
  if (vg < 1) return fail(MSB_ERR_UNSUPPORTED, "more slabs than SMs");
  CUDA_TRY(cudaMemcpyAsync(ctx, host, sizeof(SlabCtx) * nslabs, cudaMemcpyHostToDevice, as_stream(stream)));
  cudaLaunchAttribute attr[1];
  cudaLaunchConfig_t cfg = coop_config((unsigned)(vg * nslabs), kDirectThreads, 0, stream, attr, true);
  if (kDirectSplit) cfg.dynamicSmemBytes = (size_t)(kDirectThreads / 32) * kSplitWords * 4;  // the warps' stashes
  return launch_direct<true, 2, true, 0>(cb, cfg, host[0].wa, host[0].fa, host[0].ha, WinIO{}, n_sweeps,
                                           reinterpret_cast<const SlabCtx*>(ctx), nslabs);
}

}  // namespace
}  // namespace msbk
