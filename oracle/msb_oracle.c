/*
 * msb_oracle.c -- CPU restatement of the reference `multispin` hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product package links, loads or
 * calls this file; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs do, and only as the checker.
 *
 * What it restates (all paths relative to the reference's pkg/src/multispin):
 *   - splitmix64 stream seeding ............. rng.py:53-82   (_mix64, stream_state)
 *   - xoshiro256++ step ..................... rng.py:93-105  (Xoshiro256pp.next_raw64)
 *   - unit-float shaping (23-bit mantissa) .. rng.py:113-115, rng.py:180-183
 *   - random initial lattice ................ engine.py:274-282, rng.py:139-147
 *   - one colour phase of Engine.sweep ...... engine.py:314-351 (_flip_quarter,
 *     _flip_phase): per (sim, cell) stream, draws consumed in the order
 *     quarter -> k = 4i+ii -> word, draw (q,k,w) gating bit t = 4(k%4)+k//4
 *     of the quarter's target array (FLIP_RED / FLIP_BLUE, engine.py:57-68),
 *     accepted iff draw < table[sim, 8*own + n_up] in float64.
 *   - site of a packed bit .................. lattice.py:178-202 (unclassify,
 *     lattice_columns, lattice_rows)
 *   - |M| and E/N ........................... engine.py:372-386
 *
 * The engine's packed eight-array words are an implementation of the
 * neighbour count; the oracle counts neighbours on the plain +/-1 lattice
 * (reference.py:119-129 neighbor_code_brute), which the reference's own
 * tests prove equal (test_engine.py:133-144, test_acceptance.py:94-110).
 *
 * Lattice storage here: int8 spins[sim][c][r], c in [0,m), r in [0,n),
 * linear index c*n + r exactly as the reference (lattice.py:156-175).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#define M64_GOLDEN 0x9E3779B97F4B7C15ULL

/* ---- tiny pthreads parallel-for (no OpenMP runtime in this image) ---- */
static int g_threads = 0;
void orc_set_threads(int t) { g_threads = t; }
int orc_num_threads(void) {
  if (g_threads > 0) return g_threads;
  long c = sysconf(_SC_NPROCESSORS_ONLN);
  return c > 0 ? (int)c : 1;
}
typedef void (*par_fn)(long lo, long hi, void *ctx, uint64_t *acc);
typedef struct { par_fn fn; void *ctx; long n, chunk; long next; pthread_mutex_t mu; uint64_t acc; } par_job;
static void *par_worker(void *arg) {
  par_job *j = (par_job *)arg;
  uint64_t acc = 0;
  for (;;) {
    pthread_mutex_lock(&j->mu);
    long lo = j->next;
    j->next += j->chunk;
    pthread_mutex_unlock(&j->mu);
    if (lo >= j->n) break;
    long hi = lo + j->chunk < j->n ? lo + j->chunk : j->n;
    j->fn(lo, hi, j->ctx, &acc);
  }
  pthread_mutex_lock(&j->mu);
  j->acc += acc;
  pthread_mutex_unlock(&j->mu);
  return NULL;
}
static uint64_t par_for(long n, par_fn fn, void *ctx) {
  int t = orc_num_threads();
  if (t > n) t = (int)(n > 0 ? n : 1);
  par_job j = {fn, ctx, n, 1, 0, PTHREAD_MUTEX_INITIALIZER, 0};
  j.chunk = n / (8L * t) > 0 ? n / (8L * t) : 1;
  if (t <= 1) { par_worker(&j); return j.acc; }
  pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * t);
  for (int i = 0; i < t; i++) pthread_create(&th[i], NULL, par_worker, &j);
  for (int i = 0; i < t; i++) pthread_join(th[i], NULL);
  free(th);
  return j.acc;
}

/* rng.py:53-58 */
static inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

/* rng.py:71-82: stream seed = mix64(master + (stream+1)*phi); state = next 4
 * splitmix64 outputs of that seed; all-zero state patched. */
void orc_stream_state(uint64_t master, uint64_t stream, uint64_t s[4]) {
  uint64_t z = mix64(master + (stream + 1) * M64_GOLDEN);
  for (int i = 0; i < 4; i++) {
    z += M64_GOLDEN;
    s[i] = mix64(z);
  }
  if (!(s[0] | s[1] | s[2] | s[3])) s[0] = M64_GOLDEN;
}

/* rng.py:93-105 */
static inline uint64_t xnext(uint64_t s[4]) {
  uint64_t x = s[0] + s[3];
  uint64_t out = ((x << 23) | (x >> 41)) + s[0];
  uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = (s[3] << 45) | (s[3] >> 19);
  return out;
}

/* Raw outputs of one stream (Xoshiro256pp(master, stream).raw64). */
void orc_raw64(uint64_t master, uint64_t stream, uint64_t skip, uint64_t count, uint64_t *out) {
  uint64_t s[4];
  orc_stream_state(master, stream, s);
  for (uint64_t i = 0; i < skip; i++) xnext(s);
  for (uint64_t i = 0; i < count; i++) out[i] = xnext(s);
}

/* engine.py:274-282 + rng.py:139-147: init="random" draws
 * Xoshiro256pp(seed, 2**48 + sim_offset + sim).bits(m*n); spin +1 iff bit is
 * 1; bit i is bit 63 - i%64 of output i//64 (big-endian unpackbits). */
typedef struct { int m, n; uint64_t seed, sim_offset; int8_t *spins; } init_ctx;
static void init_body(long lo, long hi, void *vctx, uint64_t *acc) {
  (void)acc;
  init_ctx *x = (init_ctx *)vctx;
  const uint64_t sites = (uint64_t)x->m * x->n;
  for (long s = lo; s < hi; s++) {
    uint64_t st[4];
    orc_stream_state(x->seed, (1ULL << 48) + x->sim_offset + (uint64_t)s, st);
    int8_t *lat = x->spins + (uint64_t)s * sites;
    uint64_t word = 0;
    for (uint64_t i = 0; i < sites; i++) {
      if ((i & 63) == 0) word = xnext(st);
      lat[i] = ((word >> (63 - (i & 63))) & 1) ? 1 : -1;
    }
  }
}
void orc_init_random(int n_sim, int m, int n, uint64_t seed, uint64_t sim_offset, int8_t *spins) {
  init_ctx x = {m, n, seed, sim_offset, spins};
  par_for(n_sim, init_body, &x);
}

/* Quarter tables (engine.py:57-68), target arrays only: for each quarter q
 * the target's (forward, even) flags; identical for both colours.
 * Red: RFE, RBO, RBE, RFO.  Blue: BFE, BBO, BBE, BFO. */
static const int Q_FWD[4] = {1, 0, 0, 1};
static const int Q_EVEN[4] = {1, 0, 1, 0};

/* lattice.py:190-196: lattice column of worker cell g (1-based) of an array. */
static inline int target_column(int m, int red, int fwd, int even, int g) {
  int p0 = even ? 0 : 1;
  int cpar = red ? p0 : 1 - p0;
  return fwd ? 2 * (g - 1) + cpar : m - 2 * g + cpar;
}

/* One colour phase over every simulation (engine.py:334-351 with the
 * per-quarter work of engine.py:314-332).
 *   states: [n_sim*cells][4] xoshiro states, advanced in place by 2n draws.
 *   table:  [n_sim][16] float64 acceptance table (engine.py:257, _tables).
 *   flips:  accumulated accepted count (engine.py:331-332).
 * Neighbour values are those before the phase: a phase only writes its own
 * colour and reads the other one, so updating in place is
 * exact. */
typedef struct { int m, n, phase; uint64_t *states; const double *table; int8_t *spins; } phase_ctx;
static void phase_body(long lo, long hi, void *vctx, uint64_t *acc) {
  phase_ctx *x = (phase_ctx *)vctx;
  const int m = x->m, n = x->n, cells = m / 4, words = n / 32, red = x->phase == 0;
  const uint64_t sites = (uint64_t)m * n;
  for (long sg = lo; sg < hi; sg++) {
    const int s = (int)(sg / cells), g = (int)(sg % cells) + 1;
    uint64_t *st = x->states + 4 * sg;
    int8_t *lat = x->spins + (uint64_t)s * sites;
    const double *tab = x->table + 16 * s;
    uint64_t local = 0;
    for (int q = 0; q < 4; q++) {
      const int even = Q_EVEN[q];
      const int c = target_column(m, red, Q_FWD[q], even, g);
      const int p0 = even ? 0 : 1;
      const int8_t *up = lat + (uint64_t)((c + 1) % m) * n, *dn = lat + (uint64_t)((c + m - 1) % m) * n;
      int8_t *row = lat + (uint64_t)c * n;
      for (int k = 0; k < 16; k++) {
        const int t = 4 * (k % 4) + k / 4; /* engine.py:326-330 */
        for (int w = 0; w < words; w++) {
          const uint64_t raw = xnext(st);
          const double u = (double)((raw >> 32) & 0x7FFFFF) * (1.0 / 8388608.0);
          const int r = 32 * w + 2 * t + p0; /* lattice.py:186 */
          const int ru = r + 1 == n ? 0 : r + 1, rd = r == 0 ? n - 1 : r - 1;
          const int own = row[r] > 0;
          const int n_up = (up[r] > 0) + (dn[r] > 0) + (row[ru] > 0) + (row[rd] > 0);
          if (u < tab[8 * own + n_up]) {
            row[r] = (int8_t)-row[r];
            local++;
          }
        }
      }
    }
    *acc += local;
  }
}
void orc_flip_phase(int n_sim, int m, int n, int phase, uint64_t *states, const double *table,
                    int8_t *spins, uint64_t *flips) {
  phase_ctx x = {m, n, phase, states, table, spins};
  *flips += par_for((long)n_sim * (m / 4), phase_body, &x);
}

/* Stream states for an engine slice (engine.py:259-261): stream id
 * (sim_offset + s)*cells + g-1, advanced by `skip_draws` outputs. */
typedef struct { int m; uint64_t seed, sim_offset, skip; uint64_t *states; } st_ctx;
static void states_body(long lo, long hi, void *vctx, uint64_t *acc) {
  (void)acc;
  st_ctx *x = (st_ctx *)vctx;
  const int cells = x->m / 4;
  for (long sg = lo; sg < hi; sg++) {
    const long s = sg / cells, g = sg % cells;
    uint64_t *st = x->states + 4 * sg;
    orc_stream_state(x->seed, (x->sim_offset + (uint64_t)s) * (uint64_t)cells + (uint64_t)g, st);
    for (uint64_t i = 0; i < x->skip; i++) xnext(st);
  }
}
void orc_flip_states(int n_sim, int m, uint64_t seed, uint64_t sim_offset, uint64_t skip_draws,
                     uint64_t *states) {
  st_ctx x = {m, seed, sim_offset, skip_draws, states};
  par_for((long)n_sim * (m / 4), states_body, &x);
}

/* Engine.sweep (engine.py:353-360): red phase then blue phase. */
void orc_sweeps(int n_sim, int m, int n, int n_sweeps, uint64_t *states, const double *table,
                int8_t *spins, uint64_t *flips) {
  for (int k = 0; k < n_sweeps; k++) {
    orc_flip_phase(n_sim, m, n, 0, states, table, spins, flips);
    orc_flip_phase(n_sim, m, n, 1, states, table, spins, flips);
  }
}

/* Integer observables (engine.py:372-386): ups = number of +1 spins; bonds =
 * sum over sites of s*s(c+1) + s*s(r+1).  The float64 expressions are
 * applied by the caller exactly as the reference writes them. */
typedef struct { int m, n; const int8_t *spins; int64_t *ups, *bonds; } obs_ctx;
static void obs_body(long lo, long hi, void *vctx, uint64_t *acc) {
  (void)acc;
  obs_ctx *x = (obs_ctx *)vctx;
  const int m = x->m, n = x->n;
  const uint64_t sites = (uint64_t)m * n;
  for (long s = lo; s < hi; s++) {
    const int8_t *lat = x->spins + (uint64_t)s * sites;
    int64_t u = 0, b = 0;
    for (int c = 0; c < m; c++) {
      const int8_t *row = lat + (uint64_t)c * n, *nxt = lat + (uint64_t)((c + 1) % m) * n;
      for (int r = 0; r < n; r++) {
        u += row[r] > 0;
        b += row[r] * nxt[r] + row[r] * row[r + 1 == n ? 0 : r + 1];
      }
    }
    x->ups[s] = u;
    x->bonds[s] = b;
  }
}
void orc_observe(int n_sim, int m, int n, const int8_t *spins, int64_t *ups, int64_t *bonds) {
  obs_ctx x = {m, n, spins, ups, bonds};
  par_for(n_sim, obs_body, &x);
}

/* Draw map of one sweep for a single simulation (reference.py:179-208,
 * _MapRecorder): map[c*n + r] = the unit draw that gated site (c, r).
 * Advances `states` ([cells][4]) by one sweep. */
void orc_draw_map_sweep(int m, int n, uint64_t *states, double *map) {
  const int cells = m / 4, words = n / 32;
  for (int phase = 0; phase < 2; phase++) {
    const int red = phase == 0;
    for (int g = 1; g <= cells; g++) {
      uint64_t *st = states + 4 * (g - 1);
      for (int q = 0; q < 4; q++) {
        const int c = target_column(m, red, Q_FWD[q], Q_EVEN[q], g);
        const int p0 = Q_EVEN[q] ? 0 : 1;
        for (int k = 0; k < 16; k++) {
          const int t = 4 * (k % 4) + k / 4;
          for (int w = 0; w < words; w++) {
            const uint64_t raw = xnext(st);
            map[(uint64_t)c * n + 32 * w + 2 * t + p0] =
                (double)((raw >> 32) & 0x7FFFFF) * (1.0 / 8388608.0);
          }
        }
      }
    }
  }
}

/* ---- counter-based stream (paper_2404_16990_b200.rng.PhiloxStreams)
 * Philox4x32-10 (Salmon et al., SC'11).  Draw d of stream S under seed K:
 * low 23 bits of word d&3 of Philox(counter = (d>>2 lo, hi, S lo, hi),
 * key = (K lo, K hi)).  Consumed by the reference Engine exactly like its
 * xoshiro streams (engine.py:336): a phase takes the stream's next 2n draws. */
static void philox10(uint32_t c[4], uint32_t k0, uint32_t k1) {
  for (int r = 0; r < 10; r++) {
    const uint64_t p0 = (uint64_t)c[0] * 0xD2511F53u, p1 = (uint64_t)c[2] * 0xCD9E8D57u;
    const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c[1] ^ k0, n2 = (uint32_t)(p0 >> 32) ^ c[3] ^ k1;
    c[1] = (uint32_t)p1;
    c[3] = (uint32_t)p0;
    c[0] = n0;
    c[2] = n2;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

uint32_t orc_philox_draw(uint64_t seed, uint64_t stream, uint64_t d) {
  uint32_t c[4] = {(uint32_t)(d >> 2), (uint32_t)(d >> 34), (uint32_t)stream, (uint32_t)(stream >> 32)};
  philox10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
  return c[d & 3] & 0x7FFFFF;
}

/* Bit-plane variant (paper_2404_16990_b200.rng.PhiloxBitStreams): group
 * g = d >> 5 of a stream has 23 plane words, from Philox blocks j = 0..5 with
 * counter (g lo, (g hi << 3) | j, S lo, S hi | 2^31); draw d = 32g + i is
 * the u23 whose bit 22-b is bit i of plane b. */
static void pbits_planes(uint64_t seed, uint64_t stream, uint64_t g, uint32_t pl[24]) {
  for (int j = 0; j < 6; j++) {
    uint32_t c[4] = {(uint32_t)g, ((uint32_t)(g >> 32) << 3) | (uint32_t)j, (uint32_t)stream,
                     (uint32_t)(stream >> 32) | 0x80000000u};
    philox10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
    for (int e = 0; e < 4; e++) pl[4 * j + e] = c[e];
  }
}
static uint32_t pbits_u23(const uint32_t pl[24], int i) {
  uint32_t u = 0;
  for (int b = 0; b < 23; b++) u |= ((pl[b] >> i) & 1u) << (22 - b);
  return u;
}
uint32_t orc_pbits_draw(uint64_t seed, uint64_t stream, uint64_t d) {
  uint32_t pl[24];
  pbits_planes(seed, stream, d >> 5, pl);
  return pbits_u23(pl, (int)(d & 31));
}

typedef struct { int m, n, phase; uint64_t seed, sim_offset, block; const double *table; int8_t *spins; int bits; }
    pphase_ctx;
static void pphase_body(long lo, long hi, void *vctx, uint64_t *acc) {
  pphase_ctx *x = (pphase_ctx *)vctx;
  const int m = x->m, n = x->n, cells = m / 4, words = n / 32, red = x->phase == 0;
  const uint64_t sites = (uint64_t)m * n;
  for (long sg = lo; sg < hi; sg++) {
    const int s = (int)(sg / cells), g = (int)(sg % cells) + 1;
    const uint64_t stream = (x->sim_offset + (uint64_t)s) * (uint64_t)cells + (uint64_t)(g - 1);
    int8_t *lat = x->spins + (uint64_t)s * sites;
    const double *tab = x->table + 16 * s;
    uint64_t d = x->block * 2 * (uint64_t)n, local = 0;
    uint32_t pl[24];
    uint64_t pg = ~0ull;  /* group whose planes pl holds (bit-plane stream) */
    for (int q = 0; q < 4; q++) {
      const int even = Q_EVEN[q];
      const int c = target_column(m, red, Q_FWD[q], even, g);
      const int p0 = even ? 0 : 1;
      const int8_t *up = lat + (uint64_t)((c + 1) % m) * n, *dn = lat + (uint64_t)((c + m - 1) % m) * n;
      int8_t *row = lat + (uint64_t)c * n;
      for (int k = 0; k < 16; k++) {
        const int t = 4 * (k % 4) + k / 4;
        for (int w = 0; w < words; w++, d++) {
          uint32_t u23;
          if (x->bits) {
            if ((d >> 5) != pg) pbits_planes(x->seed, stream, pg = d >> 5, pl);
            u23 = pbits_u23(pl, (int)(d & 31));
          } else {
            u23 = orc_philox_draw(x->seed, stream, d);
          }
          const double u = (double)u23 * (1.0 / 8388608.0);
          const int r = 32 * w + 2 * t + p0;
          const int ru = r + 1 == n ? 0 : r + 1, rd = r == 0 ? n - 1 : r - 1;
          const int own = row[r] > 0;
          const int n_up = (up[r] > 0) + (dn[r] > 0) + (row[ru] > 0) + (row[rd] > 0);
          if (u < tab[8 * own + n_up]) {
            row[r] = (int8_t)-row[r];
            local++;
          }
        }
      }
    }
    *acc += local;
  }
}
void orc_flip_phase_philox(int n_sim, int m, int n, int phase, uint64_t seed, uint64_t sim_offset, uint64_t block,
                           const double *table, int8_t *spins, uint64_t *flips) {
  pphase_ctx x = {m, n, phase, seed, sim_offset, block, table, spins, 0};
  *flips += par_for((long)n_sim * (m / 4), pphase_body, &x);
}
void orc_flip_phase_philox_bits(int n_sim, int m, int n, int phase, uint64_t seed, uint64_t sim_offset,
                                uint64_t block, const double *table, int8_t *spins, uint64_t *flips) {
  pphase_ctx x = {m, n, phase, seed, sim_offset, block, table, spins, 1};
  *flips += par_for((long)n_sim * (m / 4), pphase_body, &x);
}
