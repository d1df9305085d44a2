/*
 * msb200.h -- C ABI of libmsb200.so, the B200 (sm_100a) multispin Ising
 * hot path: bit-packed checkerboard Metropolis sweeps over many replicas and
 * row slabs of very large lattices.
 *
 * The reference (`multispin`, pure Python/numpy) has no FFI; its operator
 * seam is the `Engine` class and `run_simulations`
 * (pkg/src/multispin/__init__.py:26, engine.py:216-492).  Each entry point
 * below names the reference code it replaces.  The Python drop-in
 * (paper_2404_16990_b200.engine.Engine) binds these with ctypes; a
 * maintainer could bind them from the reference the same way
 * (INTEGRATION.md).
 *
 * Conventions
 *   - Every function returns int status: MSB_OK (0) or a negative MSB_ERR_*;
 *     msb_status_string() names it, msb_last_error() (thread-local) says why.
 *     No C++ exception crosses the ABI.
 *   - Device work is asynchronous on the caller's cudaStream_t (passed as
 *     void*; NULL = legacy default stream).  The caller owns every device
 *     buffer; the library keeps no mutable global state beyond lazily built
 *     read-only tables.
 *   - Spin layout ("colour split"): uint32 spins[n_sim][2][R][Wp], colour X
 *     (0 = red, (c+r) even; 1 = blue), R = rows + 2*ghost buffer rows, row
 *     pitch Wp words.  Bit b of word j of lattice row c, colour X, is the
 *     site r = 2(32j+b) + ((c+X)&1).  Padding bits are always 0.
 *   - Linear layout: uint64 lin[n_sim][rows*n/64], bit (i%64) of word i/64
 *     is site i = (c-row0)*n + r of the held rows (np.packbits(...,
 *     bitorder="little") of the reference's (m, n) lattice, engine.py:368-370).
 *   - Reference interop layout: uint16 state[n_sim][8][m/4+2][n/32+2]
 *     (engine.py:262, lattice.py:208-234), halos and moats included.
 */
#ifndef MSB200_H
#define MSB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MSB_OK 0
#define MSB_ERR_ARG -1         /* invalid argument (dims, sizes, null pointers) */
#define MSB_ERR_CUDA -2        /* a CUDA runtime call failed */
#define MSB_ERR_UNSUPPORTED -3 /* valid request outside what this build handles */

#define MSB_MODE_FERRO 0   /* table has the J>0 Metropolis structure: 2 planes */
#define MSB_MODE_ANTI 1    /* table has the J<0 structure: 2 planes, own spin inverted */
#define MSB_MODE_GENERIC 2 /* arbitrary per-code table (tests overwrite Engine._tables) */

#define MSB_MAX_PLANES 10

/* Flip-draw streams.  XOSHIRO: the reference's own per-(replica, cell)
 * xoshiro256++ streams (rng.py:150-220), persistent per-piece states + GF(2)
 * jump-ahead.  PHILOX: counter-based Philox4x32-10, draw d of stream S =
 * low 23 bits of word d&3 of Philox(counter = (d>>2, S), key = seed); the
 * same stream on the host is paper_2404_16990_b200.rng.PhiloxStreams, which
 * the reference Engine accepts through its duck-typed `streams` seam
 * (engine.py:259-261, 336).  PHILOX_BITS: counter-based, bit-plane form:
 * draw d = 32g + i of stream S is the u23 whose bit 22-b is bit i of plane
 * word b (b = 0..22) of group g; plane 4j+e is word e of Philox(counter =
 * (g lo, (g hi << 3) | j, S lo, S hi | 2^31), key = seed), j = 0..5.  The
 * device reads only the planes its comparisons need; the host stream is
 * paper_2404_16990_b200.rng.PhiloxBitStreams. */
#define MSB_RNG_XOSHIRO 0
#define MSB_RNG_PHILOX 1
#define MSB_RNG_PHILOX_BITS 2

typedef struct msb_geom {
  int32_t n_sim;      /* replicas in the buffer */
  int32_t m, n;       /* full lattice extents (LatticeDims, lattice.py:97-136) */
  int32_t row0;       /* first lattice row c held (row-slab mode); 0 otherwise */
  int32_t rows;       /* rows held (== m for a whole lattice) */
  int32_t ghost;      /* 1 = one ghost row above/below per colour (slab mode) */
  int64_t sim_offset; /* global replica index of replica 0 (engine.py:232-236) */
} msb_geom;

typedef struct msb_sweep_params {
  int32_t mode;                  /* MSB_MODE_* */
  int32_t n_planes;              /* distinct thresholds strictly inside (0, 2^23) */
  const uint32_t *thr9;          /* device [n_planes][n_sim]: reject iff (u23 << 9) >= key */
  int8_t code_plane[16];         /* GENERIC: plane per code 8*own+n_up; -1 never, -2 always */
  int32_t kg;                    /* stream pieces per target row: 1,2,4,8 or 16 */
  const uint32_t *jump;          /* device: 32 KiB nibble table of A^(4n) */
  int32_t fault;                 /* test-only adder corruption (cli.py:467-480 analogue) */
  int32_t block_rows;            /* reserved, 0 */
  uint32_t *work;                /* device: 4 uint32 scratch counters, zeroed once by the caller;
                                    every kernel leaves them zeroed (one engine/slab per counter
                                    set: kernels sharing one must be stream-ordered) */
  int32_t rng;                   /* MSB_RNG_XOSHIRO (reference streams), _PHILOX or _PHILOX_BITS */
  uint64_t seed;                 /* Philox key (the engine's master seed), both Philox streams */
  uint64_t block;                /* Philox: stream block (2 per sweep; red = even) of the first
                                    phase whose draws the call generates */
  uint32_t *flags;               /* device: msb_flag_words() uint32, zeroed once by the caller and
                                    owned by one engine / slab (nullable for whole lattices).
                                    Band-group phase flags of the window and direct launches:
                                    flags[0] counts the colour phases completed by earlier flag
                                    launches and is advanced by each launch itself, so callers
                                    never pass a phase count.  Null: grid-wide barriers. */
} msb_sweep_params;

/* Words of a msb_sweep_params.flags buffer for geometry g:
 *   [0]                 phases completed (advanced by every window / direct flip launch)
 *   [1, 1+S)            "from above": per (replica, row segment), phases the slab above has
 *                       completed on its last row (written by that slab, peer memory)
 *   [1+S, 1+2S)         "from below": the same for the slab below's first row
 *   [1+2S, ...)         one flag per band group of the flip walk (phases completed)
 * S = n_sim * row segments.  Whole lattices use [0] and the group flags; slabs all of it. */
int64_t msb_flag_words(const msb_geom *g);

/* ---- status -------------------------------------------------------------- */
const char *msb_status_string(int status);
const char *msb_last_error(void);
int msb_abi_version(void);

/* ---- geometry helpers ------------------------------------------------------ */
/* Validates dims exactly as LatticeDims.__post_init__ (lattice.py:104-112). */
int msb_check_geom(const msb_geom *g);
int64_t msb_spin_words(const msb_geom *g);      /* uint32 words of the spin buffer */
int32_t msb_row_pitch(const msb_geom *g);       /* Wp */
int64_t msb_pieces_per_phase(const msb_geom *g, int32_t kg);
int32_t msb_default_kg(const msb_geom *g);

/* ---- thresholds: replaces the float64 gather+compare of engine.py:321-331 --- */
/* tables: host float64 [n_sim][16] (Engine._tables, engine.py:257).  Decides
 * the flip mode and writes host thr9[MSB_MAX_PLANES][n_sim] keys such that
 * u23 * 2^-23 < table[s][code]  <=>  (u23 << 9) < key of the code's plane. */
int msb_plan_thresholds(const double *tables, int32_t n_sim, int32_t *mode, int32_t *n_planes,
                        int8_t code_plane[16], uint32_t *thr9_host);

/* ---- RNG stream (rng.py:53-220, engine.py:259-261) ----------------------- */
/* Host: 64 nibble tables of A^(2^b) (64 x 32 KiB) and of A^jump (32 KiB). */
int msb_rng_power_tables(uint32_t *host_out);
int msb_rng_jump_table(uint64_t jump, uint32_t *host_out);
/* Device: per-piece xoshiro states.  One stream "block" is the 2n draws a
 * stream spends on one colour phase (engine.py:336); sweep k uses blocks 2k
 * (red) and 2k+1 (blue).  colour = -1 positions red at `block` and blue at
 * `block`+1; colour = 0/1 positions only that colour at `block`.  Stream id
 * (sim_offset+s)*(m/4) + cell-1 (engine.py:259-261).
 * states: uint32[2][8][msb_pieces_per_phase(g, kg)]. */
int msb_rng_init(const msb_geom *g, uint64_t seed, int32_t kg, uint64_t block, int32_t colour,
                 const uint32_t *pow_tables, uint32_t *states, void *stream);

/* ---- initial states (engine.py:274-300) ---------------------------------- */
/* init="random": Xoshiro256pp(seed, 2^48 + sim_offset + s).bits(m*n).
 * scratch: uint64[n_sim][rows*n/64] (the linear layout; left holding it). */
int msb_init_random(const msb_geom *g, uint64_t seed, const uint32_t *pow_tables,
                    uint64_t *scratch, uint32_t *spins, void *stream);
/* init="all-up" (up=1) or all-down (up=0); also clears ghost rows/padding. */
int msb_init_const(const msb_geom *g, int32_t up, uint32_t *spins, void *stream);
/* from_lattices / unpack (engine.py:285-300, 368-370). */
int msb_from_linear(const msb_geom *g, const uint64_t *lin, uint32_t *spins, void *stream);
int msb_to_linear(const msb_geom *g, const uint32_t *spins, uint64_t *lin, void *stream);
/* Engine.state interop incl. halo/moat refresh (engine.py:123-143,
 * lattice.py:248-329).  Whole lattices only (row0 == 0, rows == m). */
int msb_to_ref16(const msb_geom *g, const uint32_t *spins, uint16_t *state, void *stream);
int msb_from_ref16(const msb_geom *g, const uint16_t *state, uint32_t *spins, void *stream);

/* ---- the hot path: Engine.flip_red / flip_blue / sweep (engine.py:314-360) - */
/* A sweep is split in two because the reference's draws never depend on the
 * spins (engine.py:336-341 draws a whole block before flipping):
 *   msb_rng_planes: every stream piece generates its draws and reduces each
 *     to n_planes accept bits (u23 < K_p), written as bit planes in the
 *     colour-split layout: planes[2][n_planes][n_sim][rows][Pp] uint32,
 *     msb_plane_words() words per buffer.  Advances the pieces by a sweep.
 *   msb_flip: one colour phase -- bit-sliced neighbour classes select the
 *     plane bit, flips by XOR, counts accepted flips into
 *     flips[MSB_FLIP_SLOTS] (device uint64; the total is their sum,
 *     engine.py:331-332).
 * ext_draws (nullable, one colour of a whole lattice): device uint32 u23
 * draws in the reference block order [n_sim][m/4][4][16][n/32] of the phase;
 * when given, the pieces' own streams are neither used nor advanced. */
#define MSB_FLIP_SLOTS 256
int64_t msb_plane_words(const msb_geom *g, int32_t n_planes);
int msb_rng_planes(const msb_geom *g, const msb_sweep_params *p, int32_t colour, uint32_t *states,
                   const uint32_t *ext_draws, uint32_t *planes, void *stream);
int msb_flip(const msb_geom *g, const msb_sweep_params *p, int32_t colour, uint32_t *spins,
             const uint32_t *planes, uint64_t *flips, void *stream);
/* One colour phase = msb_rng_planes(colour) + msb_flip(colour). */
int msb_phase(const msb_geom *g, const msb_sweep_params *p, int32_t phase, uint32_t *spins,
              uint32_t *states, const uint32_t *ext_draws, uint32_t *planes, uint64_t *flips,
              void *stream);
/* n_sweeps full sweeps (red then blue) of a whole lattice.  planes holds
 * two msb_plane_words() buffers.  FERRO/ANTI modes run one cooperative,
 * warp-specialised kernel per sweep: the flips of sweep k (from one buffer)
 * overlap the accept planes of sweep k+1 (into the other).  Lookahead flags:
 *   MSB_SWEEP_AHEAD_IN  buffer *cur_io already holds the first sweep's planes
 *                       (the piece states are then one sweep ahead);
 *   MSB_SWEEP_AHEAD_OUT leave the next sweep's planes generated, in buffer
 *                       *cur_io on return (states one sweep ahead);
 *   MSB_SWEEP_SERIAL    separate launches, no overlap. */
#define MSB_SWEEP_AHEAD_IN 1
#define MSB_SWEEP_AHEAD_OUT 2
#define MSB_SWEEP_SERIAL 4
int msb_sweep(const msb_geom *g, const msb_sweep_params *p, uint32_t *spins, uint32_t *states,
              uint32_t *planes, int32_t n_sweeps, int32_t flags, int32_t *cur_io, uint64_t *flips,
              void *stream);

/* ---- lookahead windows: S sweeps of accept planes per launch -------------- */
/* Steady-state path for FERRO/ANTI whole lattices (replaces the Engine.sweep
 * loop, engine.py:353-360 / 416-417, S sweeps at a time).  The draws of a
 * window (sweeps w..w+S-1, stream blocks B..B+2S-1) are produced by pieces
 * (slot j, part p, stream): the stream's draws of sweep w+j, split into P
 * contiguous parts (P = 1: the whole sweep, 4n draws).  Each piece runs its
 * stream contiguously and jumps S*4n ahead once; the jump table passed in
 * p->jump must be msb_rng_jump_table(S*4n).  A window buffer holds
 * msb_window_words() uint32 words: [S][2 colours][2 planes][n_sim][m][Wp].
 * msb_window_pieces: piece count (piece states are 8 uint32 each).
 * msb_default_window: S and P for a geometry (balanced SM load, bounded
 * plane memory, rows being written kept L2-resident); msb_window_parts: P
 * for a given S.
 * msb_window_init: piece states for a window whose slot 0 starts at stream
 * block `block` (xoshiro).
 * msb_window_sweep: flips slots [first, first+count) of window `cur` (red,
 * blue, red, ... separated by grid barriers) and, if next != NULL, produces
 * the following window into `next`, in ONE cooperative launch: producer
 * warps fill `next` while the remaining warps of every CTA flip (the two
 * touch disjoint buffers).  For Philox p->block is the block of the produced
 * window's slot 0.  count == 0 with next != NULL produces only. */
/* Row slabs (g->ghost = 1; P must be >= 8 so a piece stays within one row):
 * the producer generates exactly the slab's rows, and the flips exchange
 * halos IN the kernel.  Each flip of the first / last owned row is also
 * stored into the ghost row of the slab above / below (up_spins /
 * down_spins: their spin buffers, e.g. NVLink peer mappings from symmetric
 * memory; a single slab ring passes its own buffer).  Phases are ordered per
 * band group (p->flags required): an interior group of rows waits only for
 * its neighbour groups on the same GPU; a group holding the slab's first /
 * last row also waits for the matching row segment of the slab above /
 * below to finish the previous phase (its "from above" / "from below" slot,
 * written by that slab), and after its own phase publishes completion into
 * the neighbour's slot (system-scope release in peer memory: up_flags /
 * down_flags are the neighbours' flag buffers).  Interior rows therefore
 * never wait on another GPU, and a slab's edge rows overlap its interior.
 * When the rows admit no band walk, every phase ends in a GPU-wide gate
 * instead (the same slots, one per neighbour).  All slabs of a ring start
 * from zeroed flags with valid ghost rows.  A call with count == 0, next ==
 * NULL and a halo waits (on the stream) until both neighbours completed the
 * phases in flags[0], i.e. the ghost rows are current (before observables). */
typedef struct msb_halo {
  uint32_t *up_spins, *down_spins; /* spin buffers of the slabs above / below */
  int32_t up_R, down_R;            /* their rows per colour (rows + 2) */
  uint32_t *up_flags, *down_flags; /* their msb_sweep_params.flags buffers */
} msb_halo;
/* Host I/O fused into a flip launch (whole lattices: no halo, count > 0).
 * lin_in: every warp of the launch first converts this linear lattice into
 * `spins` (msb_from_linear; all its SMs share the 8 MiB of cfg2 in a few us),
 * then the flips start.  lin_out and/or ups + unsat: after the last flip
 * phase the flip warps export the lattice / the observables (msb_export)
 * inside their slack behind the producers; ups and unsat are WRITTEN (zeroed
 * in the launch), not added.  Any member may be NULL (ups and unsat go
 * together).  Chunk groups of 4 chunks: m * ceil(n/1024) % 4 == 0. */
typedef struct msb_window_io {
  const uint64_t *lin_in;
  uint64_t *lin_out;
  int64_t *ups, *unsat;
} msb_window_io;

int msb_default_window(const msb_geom *g, int32_t *S, int32_t *P);
int32_t msb_window_parts(const msb_geom *g, int32_t S);   /* default P for a given S */
int64_t msb_window_pieces(const msb_geom *g, int32_t S, int32_t P);
int64_t msb_window_words(const msb_geom *g, int32_t S);
int msb_window_init(const msb_geom *g, uint64_t seed, int32_t S, int32_t P, uint64_t block,
                    const uint32_t *pow_tables, uint32_t *states, void *stream);
int msb_window_sweep(const msb_geom *g, const msb_sweep_params *p, int32_t S, int32_t P,
                     uint32_t *spins, uint32_t *states, const uint32_t *cur, int32_t first,
                     int32_t count, uint32_t *next, uint64_t *flips, const msb_halo *halo,
                     const msb_window_io *io, void *stream);

/* Direct sweeps (MSB_RNG_PHILOX_BITS, FERRO/ANTI tables): no accept planes.
 * One cooperative launch flips n_sweeps sweeps with every warp of every SM;
 * each word's Metropolis tests are decided from its neighbour classes, and
 * only the sites with Delta E > 0 compare their draw (bit planes generated
 * on demand, most significant first) against the Delta E = 4|J| or 8|J|
 * key.  p->block is the stream block of the first sweep's red phase (2 per
 * sweep).  Phases are ordered by p->flags band-group flags when given
 * (grid barriers otherwise); halo / io as in msb_window_sweep.  The draws
 * are those of PhiloxBitStreams, so results equal the window path and the
 * reference Engine fed that stream.  msb_direct_ok: 1 if (g, p) can take
 * this path (n/32 % 32 == 0 or n = 512, rows in bands of 2 x
 * 32/quads-per-row), else 0.  Replaces: engine.py:353-360 (Engine.sweep)
 * for the counter-based stream. */
int msb_direct_ok(const msb_geom *g, const msb_sweep_params *p);
int msb_direct_sweep(const msb_geom *g, const msb_sweep_params *p, uint32_t *spins, int32_t n_sweeps,
                     uint64_t *flips, const msb_halo *halo, const msb_window_io *io, void *stream);

/* ---- a ring of row slabs in ONE launch (several slabs per GPU) ---------- */
/* The slabs of a lattice held by one process on one device (the periodic
 * ring of one lattice in row slabs, or a part of a larger ring): one
 * cooperative launch runs them all, the CTAs split evenly between the
 * slabs, each slab with its own buffers, work counters, flags and msb_halo
 * (neighbour pointers may name slabs of this ring or peer memory).  Same
 * per-slab semantics as msb_window_sweep / msb_direct_sweep with a halo;
 * every slab shares S, P, the table mode and the stream kind.  ctx:
 * device scratch of msb_ring_ctx_bytes(nslabs) bytes (per-slab kernel
 * arguments, copied on the stream).  This is also how the multi-GPU halo
 * protocol is exercised on one GPU: a GPU cannot run several cooperative
 * launches that wait on one another, but one launch over several slabs can. */
typedef struct msb_ring_slab {
  const msb_geom *g;
  const msb_sweep_params *p;
  uint32_t *spins;
  uint32_t *states;      /* window path: piece states (xoshiro); direct: unused */
  const uint32_t *cur;   /* window path: window being flipped; direct: unused */
  uint32_t *next;        /* window path: window being produced (nullable); direct: unused */
  uint64_t *flips;
  const msb_halo *halo;
} msb_ring_slab;
#define MSB_RING_MAX 16
int64_t msb_ring_ctx_bytes(int32_t nslabs);
int msb_window_sweep_ring(int32_t nslabs, const msb_ring_slab *slabs, int32_t S, int32_t P, int32_t first,
                          int32_t count, void *ctx, void *stream);
int msb_direct_sweep_ring(int32_t nslabs, const msb_ring_slab *slabs, int32_t n_sweeps, void *ctx,
                          void *stream);

/* ---- observables (engine.py:372-386) ------------------------------------- */
/* Adds, per replica, the number of +1 spins and the number of unsatisfied
 * bonds owned by the held rows (bonds of red sites) into ups[n_sim] and
 * unsat[n_sim] (device int64; caller zeroes).  |M| = |2 ups/N - 1|,
 * E/N = -J (2N - 2 unsat)/N, evaluated on the host like the reference. */
int msb_observe(const msb_geom *g, const uint32_t *spins, int64_t *ups, int64_t *unsat,
                void *stream);
/* msb_to_linear and msb_observe in one pass over the spins (either output
 * may be NULL; ups and unsat go together).  The layout transpose already
 * holds both colours of a row, so the observables cost only the neighbour
 * rows.  msb_to_linear / msb_observe are this call with one output. */
int msb_export(const msb_geom *g, const uint32_t *spins, uint64_t *lin, int64_t *ups,
               int64_t *unsat, void *stream);

/* ---- record/replay support (reference.py:179-208) ------------------------ */
/* The u23 draws the next `phase` would consume, in the reference block order
 * [n_sim][m/4][4][16][n/32], without advancing the states. */
int msb_draws(const msb_geom *g, const msb_sweep_params *p, int32_t phase, const uint32_t *states,
              uint32_t *out, void *stream);

/* ---- slab halo helpers (row-slab decomposition over GPUs) ----------------- */
/* Pack colour `colour` of the first and last held rows into edge[2][Wp]
 * (send buffers), and unpack received neighbour rows into the ghost rows. */
int msb_pack_edges(const msb_geom *g, int32_t colour, const uint32_t *spins, uint32_t *edge,
                   void *stream);
int msb_unpack_ghosts(const msb_geom *g, int32_t colour, const uint32_t *ghost_rows,
                      uint32_t *spins, void *stream);

/* ---- measurement helpers ---------------------------------------------------- */
/* Issue-bound INT32 microbenchmark (mixed ALU/FMA-pipe ops); ops_out = total
 * integer ops executed, elapsed via CUDA events. */
int msb_bench_int_peak(int32_t blocks, int32_t iters, double *ops_out, float *ms_out,
                       void *stream);

#ifdef __cplusplus
}
#endif
#endif
