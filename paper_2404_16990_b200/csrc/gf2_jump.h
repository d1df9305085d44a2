// Host GF(2) jump-ahead for xoshiro256 (see gf2_jump.cpp).
#pragma once
#include <cstdint>

namespace msb {
// 64 nibble tables of A^(2^b): 64 x 8192 uint32 words.
void power_tables(uint32_t* out);
// Nibble table (8192 uint32 words) of A^J.
void jump_table(uint64_t J, uint32_t* out);
// s <- A^J s (host reference).
void jump_state(uint64_t J, uint64_t s[4]);
}  // namespace msb
