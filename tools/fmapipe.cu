// FMA-pipe instruction forms on sm_100a: throughput alone and mixed 1:1 with
// LOP3 (ALU pipe), independent chains, to see which IMAD forms share the
// half-rate heavy sub-pipe (development tool; run on the GPU box).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CH 8
#define ITERS 2048

template <int OP, bool MIX>
__global__ void kb(uint32_t* out, uint32_t seed) {
  uint32_t a[CH], b[CH], c[CH], d[CH];
  uint64_t w[CH];
#pragma unroll
  for (int i = 0; i < CH; i++) {
    a[i] = seed * (threadIdx.x + i + 1); b[i] = a[i] ^ 0x9e3779b9u; c[i] = a[i] + 12345u; d[i] = a[i] * 7u;
    w[i] = ((uint64_t)b[i] << 32) | a[i];
  }
  const uint32_t k1 = seed | 1, k2 = seed >> 3;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < CH; i++) {
      if (MIX) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(d[i]) : "r"(b[i]), "r"(k2));
      if (OP == 0) {  // plain IMAD
        asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[i]) : "r"(k1), "r"(b[i]));
      } else if (OP == 1) {  // IMAD.WIDE with a live 64-bit addend (its own previous result)
        asm volatile("{.reg .b32 lo, hi; mov.b64 {lo, hi}, %0; mad.wide.u32 %0, lo, 131072, %0;}" : "+l"(w[i]));
      } else if (OP == 2) {  // IMAD.X (carry-in add): add.cc on ALU-side input, addc
        asm volatile("{.reg .b32 t; add.cc.u32 t, %1, %2;\n\taddc.u32 %0, %0, %3;}" : "+r"(a[i]) : "r"(b[i]), "r"(c[i]), "r"(k1));
      } else if (OP == 3) {  // IMAD with an immediate multiplier (IMAD.SHL-like)
        asm volatile("mad.lo.u32 %0, %0, 131072, %1;" : "+r"(a[i]) : "r"(b[i]));
      } else if (OP == 4) {  // IMAD.HI
        asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(a[i]) : "r"(k1), "r"(b[i]));
      }
    }
  }
  uint32_t acc = k2;
#pragma unroll
  for (int i = 0; i < CH; i++) acc ^= a[i] ^ b[i] ^ c[i] ^ d[i] ^ (uint32_t)w[i] ^ (uint32_t)(w[i] >> 32);
  if (acc == 0x12345678u) out[threadIdx.x] = acc;
}

template <int OP, bool MIX>
void run(const char* name, uint32_t* d, int blocks) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  kb<OP, MIX><<<blocks, 256>>>(d, 7);
  cudaEventRecord(e0); kb<OP, MIX><<<blocks, 256>>>(d, 7); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double warp_inst = (double)blocks * 8 * ITERS * CH * (MIX ? 2 : 1);
  // per SMSP per clock (148 SMs x 4 SMSPs, 1.965 GHz)
  printf("%-28s %8.3f ms  %.3f warp-inst/clk/SMSP\n", name, ms, warp_inst / (ms * 1e-3) / (148.0 * 4 * 1.965e9));
}

int main() {
  uint32_t* d; cudaMalloc(&d, 4096);
  const int blocks = 148 * 8;
  run<0, false>("IMAD", d, blocks);        run<0, true>("LOP3 + IMAD", d, blocks);
  run<1, false>("IMAD.WIDE (mul.wide)", d, blocks); run<1, true>("LOP3 + IMAD.WIDE", d, blocks);
  run<2, false>("IADD3.cc + IMAD.X", d, blocks);    run<2, true>("LOP3 + IADD3.cc + IMAD.X", d, blocks);
  run<3, false>("IMAD.SHL", d, blocks);    run<3, true>("LOP3 + IMAD.SHL", d, blocks);
  run<4, false>("IMAD.HI", d, blocks);     run<4, true>("LOP3 + IMAD.HI", d, blocks);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
