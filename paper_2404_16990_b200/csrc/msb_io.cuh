// libmsb200 device code: layout conversions and observables, one warp per
// group of CPW consecutive chunks (replica, row, chunk), shared by the
// standalone kernels (msb_state.cu: msb_from_linear / msb_export) and the
// window kernel's host-I/O prologue / epilogue (msb_window.cu, msb_window_io).
//
// A chunk is a whole-warp 32 x 32 bit transpose (warp_transpose32): its 32
// linear words (1024 sites; lane b holds sites 32b..32b+31) and its 2 x 16
// colour-split words (bit b of word (X, t) = site 32b + 2t + p, p = (c+X)&1)
// are transposes of each other, and lane 2t + p holds word t of parity p.  A
// group issues all its loads before the first transpose, so CPW 128-byte
// requests per warp are in flight (one per warp left the conversions at
// ~1.5 TB/s, latency-bound).  A group never spans two replicas: CPW divides
// rows * nch (msb_state.cu's conv_cpw; the window epilogue uses kIoCpw = 4,
// which divides every whole lattice's m).
#pragma once
#include "msb_common.cuh"

namespace msbk {

constexpr int kIoCpw = 4;

// Walks the consecutive chunks of one replica with 32-bit word offsets
// (every buffer a conversion touches is < 2^31 words, msb_state.cu's
// check_conv): lrow = linear row start, srow = colour-0 spin row start (the
// colour-1 row is cstride further), c = lattice row, ch = chunk of the row.
struct ChunkWalk {
  unsigned lrow, srow;
  int s, c, ch, br;
  __device__ __forceinline__ ChunkWalk(const Geo& G, unsigned q, int cpw) {
    int lr;
    chunk_coords(G, q * (unsigned)cpw, s, lr, ch);
    c = G.row0 + lr;
    br = lr + G.ghost;
    lrow = ((unsigned)s * (unsigned)G.rows + (unsigned)lr) * (unsigned)G.words;
    srow = ((unsigned)s * 2u * (unsigned)G.R + (unsigned)br) * (unsigned)G.Wp;
  }
  __device__ __forceinline__ void next(const Geo& G) {
    if (++ch == G.nch) {
      ch = 0;
      ++c;
      ++br;
      lrow += (unsigned)G.words;
      srow += (unsigned)G.Wp;
    }
  }
  // valid linear words of the current chunk (only a row's last chunk is partial)
  __device__ __forceinline__ int bits(const Geo& G) const { return chunk_bits(G, ch); }
};

// Linear -> colour-split for chunk group q (engine.py:285-300 layout).
template <int CPW>
__device__ __forceinline__ void from_linear_group(const Geo& G, const uint32_t* __restrict__ lin,
                                                  uint32_t* __restrict__ spins, unsigned q) {
  const int lane = threadIdx.x & 31, t = lane >> 1, p = lane & 1;
  const unsigned cstride = (unsigned)G.R * (unsigned)G.Wp;
  const ChunkWalk w0(G, q, CPW);
  uint32_t L[CPW];
  ChunkWalk w = w0;
#pragma unroll
  for (int j = 0; j < CPW; j++, w.next(G))
    L[j] = lane < w.bits(G) ? __ldcs(lin + (w.lrow + 32u * (unsigned)w.ch + (unsigned)lane)) : 0u;
  w = w0;
#pragma unroll
  for (int j = 0; j < CPW; j++, w.next(G))
    spins[w.srow + (((w.c + p) & 1) ? cstride : 0u) + 16u * (unsigned)w.ch + (unsigned)t] = warp_transpose32(L[j]);  // unsigned index
}

// Colour-split -> linear (LIN) and/or the observables (OBS; engine.py:372-386)
// of chunk group q, one pass; returns the group's replica.  The warp holds
// both colours' words of its chunk for the transpose, so the observables add
// only the blue rows above and below.  u gets the +1 spins of both colours,
// b the unsatisfied bonds of the red sites (4 neighbours each, every bond
// once); both are per-lane partial sums.  Red lane 2t+p0 (p0 = c&1) takes
// its blue word t from lane ^ 1; the row below's from that partner lane
// (which loads it while the red lane loads the row above); the second
// horizontal neighbour (h_second) from lane +-1, or at the chunk's edge word
// from lane 0 / 31 plus one bit of the adjacent chunk (a load).  COHERENT:
// the spins were written earlier in the same kernel by other SMs.
template <int CPW, bool LIN, bool OBS, bool COHERENT>
__device__ __forceinline__ int export_group(const Geo& G, const uint32_t* __restrict__ spins,
                                            uint32_t* __restrict__ lin, unsigned q, uint32_t& u, uint32_t& b) {
  const int lane = threadIdx.x & 31, t = lane >> 1, p = lane & 1;
  auto ld = [](const uint32_t* a) { return COHERENT ? __ldcg(a) : *a; };
  const unsigned Wp = (unsigned)G.Wp, cstride = (unsigned)G.R * Wp;
  const ChunkWalk w0(G, q, CPW);
  uint32_t W[CPW], V[CPW], E[CPW];
  ChunkWalk w = w0;
#pragma unroll
  for (int j = 0; j < CPW; j++, w.next(G)) {
    const unsigned wd = 16u * (unsigned)w.ch + (unsigned)t;
    W[j] = ld(spins + (w.srow + (((w.c + p) & 1) ? cstride : 0u) + wd));
    if (OBS) {
      const int p0 = w.c & 1;
      const bool red = p == p0;
      int bu, bd;
      vert_rows(G, w.br, bu, bd);
      const unsigned blu = w.srow + cstride;  // the blue row of c
      // blue word t of the row above (red lanes) / below (their blue partners)
      // (32-bit offset arithmetic first: the row delta may be negative)
      V[j] = ld(spins + (blu + (unsigned)((red ? bu : bd) - w.br) * Wp + wd));
      E[j] = 0u;  // the adjacent chunk's word that supplies the edge bit
      if (red && p0 && t == 15) E[j] = ld(spins + (blu + 16u * (unsigned)(w.ch + 1 < G.nch ? w.ch + 1 : 0)));
      if (red && !p0 && t == 0) E[j] = ld(spins + (blu + 16u * (unsigned)(w.ch > 0 ? w.ch - 1 : G.nch - 1) + 15u));
    }
  }
  w = w0;
#pragma unroll
  for (int j = 0; j < CPW; j++, w.next(G)) {
    if (LIN) {
      const uint32_t L = warp_transpose32(W[j]);
      if (lane < w.bits(G)) __stcs(lin + (w.lrow + 32u * (unsigned)w.ch + (unsigned)lane), L);
    }
    if (OBS) {
      const int p0 = w.c & 1;
      const int nb = w.bits(G);
      const uint32_t vm = nb >= 32 ? 0xFFFFFFFFu : ((1u << nb) - 1u);
      const uint32_t y0 = __shfl_xor_sync(0xFFFFFFFFu, W[j], 1);
      const uint32_t yd = __shfl_xor_sync(0xFFFFFFFFu, V[j], 1);
      const uint32_t yi = __shfl_sync(0xFFFFFFFFu, W[j], p0 ? (lane + 1) & 31 : (lane + 31) & 31);
      const uint32_t ye = __shfl_sync(0xFFFFFFFFu, W[j], p0 ? 0 : 31);
      uint32_t hs = yi;
      if (p0 && t == 15) hs = (ye >> 1) | ((E[j] & 1u) << (nb - 1));
      if (!p0 && t == 0) {
        const uint32_t carry = w.ch > 0 ? E[j] >> 31 : (E[j] >> (chunk_bits(G, G.nch - 1) - 1)) & 1u;
        hs = ((ye << 1) | carry) & vm;
      }
      u += __popc(W[j]);
      if (p == p0) {
        const uint32_t o = W[j];
        b += __popc((o ^ V[j]) & vm) + __popc((o ^ yd) & vm) + __popc((o ^ y0) & vm) + __popc((o ^ hs) & vm);
      }
    }
  }
  return w0.s;
}

}  // namespace msbk
