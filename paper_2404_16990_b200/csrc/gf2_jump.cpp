// GF(2) jump-ahead for the reference's xoshiro256++ streams.
//
// The xoshiro256 state transition (rng.py:93-105, the lines after `result`)
// is linear over GF(2): s' = A s for a fixed 256x256 bit matrix A.  Skipping
// J draws is s -> A^J s.  The sweep kernel keeps one persistent state per
// stream *piece* and advances it by one sweep (4n draws) with the constant
// matrix B = A^(4n); piece start states are built from the 64 powers
// A^(2^b).  Matrices are applied on the device through 4-bit "nibble"
// tables: for each of the 64 state nibbles p and value v,
// T[p][v] = M * (v << 4p), so M s = XOR_p T[p][nibble_p(s)] -- 64 lookups of
// 32 bytes.
//
// State bit order: bit i of the 256-bit vector is bit (i % 64) of s[i / 64],
// i.e. 32-bit word i/32 is s[i/64]'s low (even) or high (odd) half.  This is
// the register order the kernels use (s0.lo, s0.hi, s1.lo, ...).
#include <cstdint>
#include <cstring>
#include <mutex>
#include <vector>

#include "gf2_jump.h"

namespace msb {

struct Mat {  // column-major: col[i] = M e_i, a 256-bit vector as 4 u64
  uint64_t col[256][4];
};

static void xoshiro_linear_step(uint64_t s[4]) {  // rng.py:97-104 (state part only)
  uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = (s[3] << 45) | (s[3] >> 19);
}

static void transition(Mat& A) {
  for (int i = 0; i < 256; i++) {
    uint64_t s[4] = {0, 0, 0, 0};
    s[i / 64] = 1ULL << (i % 64);
    xoshiro_linear_step(s);
    std::memcpy(A.col[i], s, sizeof s);
  }
}

static void apply(const Mat& M, const uint64_t v[4], uint64_t out[4]) {
  uint64_t r[4] = {0, 0, 0, 0};
  for (int i = 0; i < 256; i++) {
    if ((v[i / 64] >> (i % 64)) & 1) {
      for (int k = 0; k < 4; k++) r[k] ^= M.col[i][k];
    }
  }
  std::memcpy(out, r, sizeof r);
}

static void mul(const Mat& X, const Mat& Y, Mat& out) {  // out = X Y
  Mat r;
  for (int i = 0; i < 256; i++) apply(X, Y.col[i], r.col[i]);
  out = r;
}

static void identity(Mat& I) {
  std::memset(&I, 0, sizeof I);
  for (int i = 0; i < 256; i++) I.col[i][i / 64] = 1ULL << (i % 64);
}

// A^(2^b), b = 0..63, built once (thread-safe).
static const std::vector<Mat>& powers() {
  static std::vector<Mat> P;
  static std::once_flag once;
  std::call_once(once, [] {
    P.resize(64);
    transition(P[0]);
    for (int b = 1; b < 64; b++) mul(P[b - 1], P[b - 1], P[b]);
  });
  return P;
}

static void jump_matrix(uint64_t J, Mat& out) {
  const auto& P = powers();
  identity(out);
  for (int b = 0; b < 64; b++)
    if ((J >> b) & 1) mul(P[b], out, out);
}

// Nibble table: 64 positions x 16 values x 8 uint32 words = 32 KiB.
static void nibble_table(const Mat& M, uint32_t* out) {
  for (int p = 0; p < 64; p++) {
    for (int v = 0; v < 16; v++) {
      uint64_t r[4] = {0, 0, 0, 0};
      for (int bit = 0; bit < 4; bit++) {
        if ((v >> bit) & 1) {
          const int i = 4 * p + bit;
          for (int k = 0; k < 4; k++) r[k] ^= M.col[i][k];
        }
      }
      uint32_t* e = out + (p * 16 + v) * 8;
      for (int k = 0; k < 4; k++) {
        e[2 * k] = (uint32_t)r[k];
        e[2 * k + 1] = (uint32_t)(r[k] >> 32);
      }
    }
  }
}

void power_tables(uint32_t* out /* 64 * 8192 words */) {
  const auto& P = powers();
  for (int b = 0; b < 64; b++) nibble_table(P[b], out + (size_t)b * 8192);
}

void jump_table(uint64_t J, uint32_t* out) {
  Mat M;
  jump_matrix(J, M);
  nibble_table(M, out);
}

// Host reference of a jump (used by the library's self-check and tests).
void jump_state(uint64_t J, uint64_t s[4]) {
  const auto& P = powers();
  for (int b = 0; b < 64; b++) {
    if ((J >> b) & 1) {
      uint64_t r[4];
      apply(P[b], s, r);
      std::memcpy(s, r, sizeof r);
    }
  }
}

}  // namespace msb
