// INT32 pipe microbenchmark for sm_100a: issue-bound loops of independent
// integer ops, to measure per-instruction-class throughput on the box.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CH 8
#define ITERS 4096

template <int OP>
__global__ void kbench(uint32_t* out, uint32_t seed) {
  uint32_t a[CH], b[CH];
#pragma unroll
  for (int i = 0; i < CH; i++) { a[i] = seed * (threadIdx.x + i + 1); b[i] = a[i] ^ 0x9e3779b9u; }
  uint32_t k1 = seed | 1, k2 = seed >> 3;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < CH; i++) {
      if (OP == 0) {  // LOP3
        asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[i]) : "r"(b[i]), "r"(k1));
      } else if (OP == 1) {  // IADD3
        asm volatile("add.u32 %0, %0, %1;\n\tadd.u32 %0, %0, %2;" : "+r"(a[i]) : "r"(b[i]), "r"(k1));
      } else if (OP == 2) {  // SHF funnel
        asm volatile("shf.l.wrap.b32 %0, %0, %1, 13;" : "+r"(a[i]) : "r"(b[i]));
      } else if (OP == 3) {  // IMAD
        asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[i]) : "r"(k1), "r"(b[i]));
      } else if (OP == 4) {  // IMAD.WIDE.U32
        uint64_t r;
        asm volatile("mad.wide.u32 %0, %1, %2, %3;" : "=l"(r) : "r"(a[i]), "r"(k1), "l"(((uint64_t)b[i] << 32) | a[i]));
        a[i] = (uint32_t)r; b[i] = (uint32_t)(r >> 32);
      } else if (OP == 5) {  // LOP3 + IMAD 1:1
        asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[i]) : "r"(b[i]), "r"(k1));
        asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(b[i]) : "r"(k1), "r"(k2));
      } else if (OP == 6) {  // LOP3 + IMAD.WIDE 1:1
        uint64_t r;
        asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[i]) : "r"(b[i]), "r"(k1));
        asm volatile("mad.wide.u32 %0, %1, %2, %3;" : "=l"(r) : "r"(b[i]), "r"(k1), "l"((uint64_t)k2));
        b[i] = (uint32_t)r ^ (uint32_t)(r >> 32);
      } else if (OP == 7) {  // add.cc / addc pair (64-bit add)
        asm volatile("add.cc.u32 %0, %0, %2;\n\taddc.u32 %1, %1, %3;" : "+r"(a[i]), "+r"(b[i]) : "r"(k1), "r"(k2));
      } else if (OP == 8) {  // 2 LOP3 + 1 IMAD
        asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[i]) : "r"(b[i]), "r"(k1));
        asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(b[i]) : "r"(a[i]), "r"(k2));
        asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(k2) : "r"(k1), "r"(a[i]));
      }
    }
  }
  uint32_t acc = k2;
#pragma unroll
  for (int i = 0; i < CH; i++) acc ^= a[i] ^ b[i];
  if (acc == 0x12345678u) out[threadIdx.x] = acc;
}

// xoshiro256++ draws (the reference stream), plain CUDA C, 64-bit types.
__global__ void kxoshiro(uint32_t* out, uint32_t seed, int nsteps) {
  uint64_t s0 = 0x9E3779B97F4B7C15ull * (blockIdx.x * blockDim.x + threadIdx.x + 1) ^ seed;
  uint64_t s1 = s0 * 3 + 1, s2 = s0 ^ 0xdeadbeef12345ull, s3 = s1 * 7 + 11;
  uint32_t acc = 0, K = 0x400000u << 9;
  for (int i = 0; i < nsteps; i++) {
    uint64_t x = s0 + s3;
    uint64_t r = ((x << 23) | (x >> 41)) + s0;
    uint64_t t = s1 << 17;
    s2 ^= s0; s3 ^= s1; s1 ^= s2; s0 ^= s3; s2 ^= t; s3 = (s3 << 45) | (s3 >> 19);
    uint32_t hi = (uint32_t)(r >> 32) << 9;
    acc = acc * 2 + (hi < K);
  }
  if (acc == 0x12345678u) out[0] = acc;
}

int main() {
  uint32_t* d; cudaMalloc(&d, 4096);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int dev; cudaGetDevice(&dev); cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("SMs %d clock %d kHz\n", p.multiProcessorCount, clk);
  const char* names[] = {"LOP3", "IADD(2)", "SHF", "IMAD", "IMAD.WIDE", "LOP3+IMAD", "LOP3+IMAD.WIDE(+LOP)", "ADDCC+ADDC", "2LOP3+IMAD"};
  int ops_per[] = {1, 2, 1, 1, 1, 2, 3, 2, 3};
  int blocks = p.multiProcessorCount * 8, threads = 256;
  for (int rep = 0; rep < 2; rep++)
  for (int op = 0; op < 9; op++) {
    auto launch = [&]() {
      switch (op) {
        case 0: kbench<0><<<blocks, threads>>>(d, 7); break;
        case 1: kbench<1><<<blocks, threads>>>(d, 7); break;
        case 2: kbench<2><<<blocks, threads>>>(d, 7); break;
        case 3: kbench<3><<<blocks, threads>>>(d, 7); break;
        case 4: kbench<4><<<blocks, threads>>>(d, 7); break;
        case 5: kbench<5><<<blocks, threads>>>(d, 7); break;
        case 6: kbench<6><<<blocks, threads>>>(d, 7); break;
        case 7: kbench<7><<<blocks, threads>>>(d, 7); break;
        case 8: kbench<8><<<blocks, threads>>>(d, 7); break;
      }
    };
    launch(); cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)blocks * threads * ITERS * CH * ops_per[op];
    if (rep) printf("%-24s %8.3f ms  %8.2f Tops/s (ptx-level ops)\n", names[op], ms, ops / ms / 1e9);
  }
  for (int bl : {148 * 2, 148 * 4, 148 * 8, 148 * 16}) {
    int ns = 1 << 14;
    kxoshiro<<<bl, 256>>>(d, 3, ns);
    cudaEventRecord(e0); kxoshiro<<<bl, 256>>>(d, 3, ns); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("xoshiro blocks=%d: %.3f ms  %.3f T draws/s\n", bl, ms, (double)bl * 256 * ns / ms / 1e9);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
