// INT32 pipe microbenchmark for sm_100a: issue-bound loops of independent
// integer ops, to measure per-instruction-class throughput on the box, plus
// xoshiro256++ draw-generation variants (the reference stream's hot loop).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CH 8
#define ITERS 2048

template <int OP>
__global__ void kbench(uint32_t* out, uint32_t seed) {
  uint32_t a[CH], b[CH], c[CH];
#pragma unroll
  for (int i = 0; i < CH; i++) {
    a[i] = seed * (threadIdx.x + i + 1);
    b[i] = a[i] ^ 0x9e3779b9u;
    c[i] = a[i] + 12345u;
  }
  uint32_t k1 = seed | 1, k2 = seed >> 3;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < CH; i++) {
      if (OP == 0) {  // LOP3
        asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[i]) : "r"(b[i]), "r"(k1));
      } else if (OP == 1) {  // SHF funnel
        asm volatile("shf.l.wrap.b32 %0, %0, %1, 13;" : "+r"(a[i]) : "r"(b[i]));
      } else if (OP == 2) {  // IMAD
        asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[i]) : "r"(k1), "r"(b[i]));
      } else if (OP == 3) {  // IMAD.WIDE.U32 with a live 64-bit addend {c,b}
        asm volatile("{.reg .b64 t; mov.b64 t, {%1, %2}; mad.wide.u32 t, %0, %3, t; mov.b64 {%1, %2}, t;}"
                     : "+r"(a[i]), "+r"(b[i]), "+r"(c[i]) : "r"(k1));
      } else if (OP == 4) {  // IMAD.HI
        asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(a[i]) : "r"(k1), "r"(b[i]));
      } else if (OP == 5) {  // IADD3 carry-out + carry-in add (add.cc / addc)
        asm volatile("add.cc.u32 %0, %0, %2;\n\taddc.u32 %1, %1, %3;" : "+r"(a[i]), "+r"(b[i]) : "r"(k1), "r"(k2));
      } else if (OP == 6) {  // sub.cc + addc accumulate (the compare idiom)
        asm volatile("{.reg .b32 t; sub.cc.u32 t, %1, %2;\n\taddc.u32 %0, %0, %0;}" : "+r"(a[i]) : "r"(b[i]), "r"(k1));
        b[i] += 0x9e3779b9u;
      } else if (OP == 7) {  // LOP3 + IMAD.WIDE 1:1
        asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[i]) : "r"(c[i]), "r"(k1));
        asm volatile("{.reg .b64 t; mov.b64 t, {%0, %1}; mad.wide.u32 t, %2, %3, t; mov.b64 {%0, %1}, t;}"
                     : "+r"(b[i]), "+r"(c[i]) : "r"(a[i]), "r"(k2));
      }
    }
  }
  uint32_t acc = k2;
#pragma unroll
  for (int i = 0; i < CH; i++) acc ^= a[i] ^ b[i] ^ c[i];
  if (acc == 0x12345678u) out[threadIdx.x] = acc;
}

__device__ __forceinline__ uint32_t fsl(uint32_t lo, uint32_t hi, int s) { return __funnelshift_l(lo, hi, s); }

// 64-bit (hi:lo) = a * m + (chi:clo) on the FMA pipe (IMAD.WIDE.U32); m is a
// runtime 1 so ptxas cannot strength-reduce it into an IADD3 pair.
__device__ __forceinline__ void madw(uint32_t& lo, uint32_t& hi, uint32_t a, uint32_t m, uint32_t clo, uint32_t chi) {
  asm("{.reg .b64 t; mov.b64 t, {%2, %3}; mad.wide.u32 t, %4, %5, t; mov.b64 {%0, %1}, t;}"
      : "=r"(lo), "=r"(hi) : "r"(clo), "r"(chi), "r"(a), "r"(m));
}

// VAR 0: plain 64-bit C (compiler's choice).  VAR 1: 32-bit halves, funnel
// shifts, carry-chain compares (ALU heavy).  VAR 2: compares through
// IMAD.WIDE.  VAR 3: VAR 2 + s0+s3 through IMAD.WIDE.  VAR 4: VAR 3 + the
// output add through IMAD.WIDE.
template <int VAR>
__global__ void kxoshiro(uint32_t* out, uint32_t seed, int nsteps, uint32_t one) {
  uint64_t s0 = 0x9E3779B97F4B7C15ull * (blockIdx.x * blockDim.x + threadIdx.x + 1) ^ seed;
  uint64_t s1 = s0 * 3 + 1, s2 = s0 ^ 0xdeadbeef12345ull, s3 = s1 * 7 + 11;
  uint32_t acc0 = 0, acc1 = 0, K0 = 0x300000u << 9, K1 = 0x80000u << 9;
  uint32_t nK0 = 0u - K0, nK1 = 0u - K1;
  if (VAR == 0) {
    for (int i = 0; i < nsteps; i++) {
      uint64_t x = s0 + s3;
      uint64_t r = ((x << 23) | (x >> 41)) + s0;
      uint64_t t = s1 << 17;
      s2 ^= s0; s3 ^= s1; s1 ^= s2; s0 ^= s3; s2 ^= t; s3 = (s3 << 45) | (s3 >> 19);
      uint32_t hi = (uint32_t)(r >> 32) << 9;
      acc0 = acc0 * 2 + (hi >= K0);
      acc1 = acc1 * 2 + (hi >= K1);
    }
  } else {
    uint32_t a0 = (uint32_t)s0, a1 = s0 >> 32, b0 = (uint32_t)s1, b1 = s1 >> 32;
    uint32_t c0 = (uint32_t)s2, c1 = s2 >> 32, d0 = (uint32_t)s3, d1 = s3 >> 32;
#pragma unroll 4
    for (int i = 0; i < nsteps; i++) {
      uint32_t x0, x1, o1;
      if (VAR >= 3) {
        uint32_t h;
        madw(x0, h, a0, one, d0, d1);
        x1 = h + a1;
      } else {
        asm("add.cc.u32 %0, %2, %3;\n\taddc.u32 %1, %4, %5;" : "=r"(x0), "=r"(x1) : "r"(a0), "r"(d0), "r"(a1), "r"(d1));
      }
      uint32_t r1 = fsl(x0, x1, 23), r0 = fsl(x1, x0, 23);
      if (VAR >= 4) {
        uint32_t l, h;
        madw(l, h, r0, one, a0, a1);
        o1 = h + r1;
      } else {
        asm("{.reg .b32 t; add.cc.u32 t, %1, %2;\n\taddc.u32 %0, %3, %4;}" : "=r"(o1) : "r"(r0), "r"(a0), "r"(r1), "r"(a1));
      }
      uint32_t hi9 = o1 << 9;
      if (VAR == 1) {
        asm("{.reg .b32 t; sub.cc.u32 t, %1, %2;\n\taddc.u32 %0, %0, %0;}" : "+r"(acc0) : "r"(hi9), "r"(K0));
        asm("{.reg .b32 t; sub.cc.u32 t, %1, %2;\n\taddc.u32 %0, %0, %0;}" : "+r"(acc1) : "r"(hi9), "r"(K1));
      } else {
        uint32_t l, h;
        madw(l, h, hi9, one, nK0, 0u);
        acc0 = acc0 * 2 + h;
        madw(l, h, hi9, one, nK1, 0u);
        acc1 = acc1 * 2 + h;
      }
      uint32_t t0 = b0 << 17, t1 = fsl(b0, b1, 17);
      uint32_t nc0 = c0 ^ a0 ^ t0, nc1 = c1 ^ a1 ^ t1;
      uint32_t nd0 = d0 ^ b0, nd1 = d1 ^ b1;
      uint32_t nb0 = b0 ^ c0 ^ a0, nb1 = b1 ^ c1 ^ a1;
      uint32_t na0 = a0 ^ d0 ^ b0, na1 = a1 ^ d1 ^ b1;
      a0 = na0; a1 = na1; b0 = nb0; b1 = nb1; c0 = nc0; c1 = nc1;
      d1 = fsl(nd1, nd0, 13);
      d0 = fsl(nd0, nd1, 13);
    }
  }
  if ((acc0 ^ acc1) == 0x12345678u) out[0] = acc0;
}

__device__ __forceinline__ uint32_t lop3x(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d; asm("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(d) : "r"(a), "r"(b), "r"(c)); return d;
}
// 64-bit product of a 32-bit value and an immediate power of two through
// the FMA pipe (mul.wide.u32); lo/hi halves.
template <int K>
__device__ __forceinline__ void wide_pow2(uint32_t x, uint32_t& lo, uint32_t& hi) {
  uint64_t r;
  asm("mul.wide.u32 %0, %1, %2;" : "=l"(r) : "r"(x), "n"(1u << K));
  lo = (uint32_t)r; hi = (uint32_t)(r >> 32);
}

// VAR 5: t via WIDE; VAR 6: + rotl13 via WIDE+IMAD; VAR 7: + r0 via WIDE+IMAD
template <int VAR>
__global__ void kxo2(uint32_t* out, uint32_t seed, int nsteps) {
  uint64_t s0 = 0x9E3779B97F4B7C15ull * (blockIdx.x * blockDim.x + threadIdx.x + 1) ^ seed;
  uint64_t s1 = s0 * 3 + 1, s2 = s0 ^ 0xdeadbeef12345ull, s3 = s1 * 7 + 11;
  uint32_t acc0 = 0, acc1 = 0, K0 = 0x300000u << 9, K1 = 0x80000u << 9;
  uint32_t a0 = (uint32_t)s0, a1 = s0 >> 32, b0 = (uint32_t)s1, b1 = s1 >> 32;
  uint32_t c0 = (uint32_t)s2, c1 = s2 >> 32, d0 = (uint32_t)s3, d1 = s3 >> 32;
#pragma unroll 8
  for (int i = 0; i < nsteps; i++) {
    uint32_t x0, x1, o1;
    asm("add.cc.u32 %0, %2, %3;\n\taddc.u32 %1, %4, %5;" : "=r"(x0), "=r"(x1) : "r"(a0), "r"(d0), "r"(a1), "r"(d1));
    uint32_t r1 = fsl(x0, x1, 23), r0;
    if (VAR >= 7) { uint32_t wl, wh; wide_pow2<23>(x1, wl, wh); r0 = x0 * (1u << 23) + wh; }
    else r0 = fsl(x1, x0, 23);
    asm("{.reg .b32 t; add.cc.u32 t, %1, %2;\n\taddc.u32 %0, %3, %4;}" : "=r"(o1) : "r"(r0), "r"(a0), "r"(r1), "r"(a1));
    uint32_t hi9 = o1 << 9;
    asm("{.reg .b32 t; sub.cc.u32 t, %1, %2;\n\taddc.u32 %0, %0, %0;}" : "+r"(acc0) : "r"(hi9), "r"(K0));
    asm("{.reg .b32 t; sub.cc.u32 t, %1, %2;\n\taddc.u32 %0, %0, %0;}" : "+r"(acc1) : "r"(hi9), "r"(K1));
    uint32_t t0, t1;
    { uint32_t wh; wide_pow2<17>(b0, t0, wh); t1 = b1 * (1u << 17) + wh; }
    const uint32_t nc0 = lop3x(c0, a0, t0), nc1 = lop3x(c1, a1, t1);
    const uint32_t nd0 = d0 ^ b0, nd1 = d1 ^ b1;
    const uint32_t nb0 = lop3x(b0, c0, a0), nb1 = lop3x(b1, c1, a1);
    const uint32_t na0 = lop3x(a0, d0, b0), na1 = lop3x(a1, d1, b1);
    a0 = na0; a1 = na1; b0 = nb0; b1 = nb1; c0 = nc0; c1 = nc1;
    if (VAR >= 6) {
      uint32_t l0, h0, l1, h1;
      wide_pow2<13>(nd0, l0, h0);
      wide_pow2<13>(nd1, l1, h1);
      d1 = nd0 * (1u << 13) + h1;   // (nd0 << 13) | (nd1 >> 19)
      d0 = nd1 * (1u << 13) + h0;   // (nd1 << 13) | (nd0 >> 19)
    } else {
      d1 = fsl(nd1, nd0, 13);
      d0 = fsl(nd0, nd1, 13);
    }
  }
  if ((acc0 ^ acc1) == 0x12345678u) out[0] = acc0 ^ a0 ^ b1 ^ c0 ^ d1;
}

// VAR 8: VAR 5 + 64-bit adds through IMAD.WIDE with a dead pair addend and a
// runtime multiplier of 1 (state update computed first so s0/s3 die there)
template <int VAR>
__global__ void kxo3(uint32_t* out, uint32_t seed, int nsteps, const uint32_t* onep) {
  uint64_t s0 = 0x9E3779B97F4B7C15ull * (blockIdx.x * blockDim.x + threadIdx.x + 1) ^ seed;
  uint64_t s1 = s0 * 3 + 1, s2 = s0 ^ 0xdeadbeef12345ull, s3 = s1 * 7 + 11;
  uint32_t acc0 = 0, acc1 = 0, K0 = 0x300000u << 9, K1 = 0x80000u << 9;
  const uint32_t one = onep[threadIdx.x & 7];
  uint32_t a0 = (uint32_t)s0, a1 = s0 >> 32, b0 = (uint32_t)s1, b1 = s1 >> 32;
  uint32_t c0 = (uint32_t)s2, c1 = s2 >> 32, d0 = (uint32_t)s3, d1 = s3 >> 32;
#pragma unroll 8
  for (int i = 0; i < nsteps; i++) {
    uint32_t t0, t1;
    { uint32_t wh; wide_pow2<17>(b0, t0, wh); t1 = b1 * (1u << 17) + wh; }
    const uint32_t nc0 = lop3x(c0, a0, t0), nc1 = lop3x(c1, a1, t1);
    const uint32_t nd0 = d0 ^ b0, nd1 = d1 ^ b1;
    const uint32_t nb0 = lop3x(b0, c0, a0), nb1 = lop3x(b1, c1, a1);
    const uint32_t na0 = lop3x(a0, d0, b0), na1 = lop3x(a1, d1, b1);
    // x = s0 + s3 (old values), addend pair d dies here
    uint64_t xd = ((uint64_t)d1 << 32) | d0;
    uint64_t x;
    asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(x) : "r"(a0), "r"(one), "l"(xd));
    const uint32_t x0 = (uint32_t)x, x1 = (uint32_t)(x >> 32) + a1;
    const uint32_t r1 = fsl(x0, x1, 23), r0 = fsl(x1, x0, 23);
    uint32_t o1;
    if (VAR >= 9) {
      uint64_t ap = ((uint64_t)a1 << 32) | a0, o;
      asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(o) : "r"(r0), "r"(one), "l"(ap));
      o1 = (uint32_t)(o >> 32) + r1;
    } else {
      asm("{.reg .b32 t; add.cc.u32 t, %1, %2;\n\taddc.u32 %0, %3, %4;}" : "=r"(o1) : "r"(r0), "r"(a0), "r"(r1), "r"(a1));
    }
    const uint32_t hi9 = o1 << 9;
    asm("{.reg .b32 t; sub.cc.u32 t, %1, %2;\n\taddc.u32 %0, %0, %0;}" : "+r"(acc0) : "r"(hi9), "r"(K0));
    asm("{.reg .b32 t; sub.cc.u32 t, %1, %2;\n\taddc.u32 %0, %0, %0;}" : "+r"(acc1) : "r"(hi9), "r"(K1));
    a0 = na0; a1 = na1; b0 = nb0; b1 = nb1; c0 = nc0; c1 = nc1;
    d1 = fsl(nd1, nd0, 13);
    d0 = fsl(nd0, nd1, 13);
  }
  if ((acc0 ^ acc1) == 0x12345678u) out[0] = acc0 ^ a0 ^ b1 ^ c0 ^ d1;
}

int main() {
  uint32_t* d; cudaMalloc(&d, 4096);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int dev; cudaGetDevice(&dev); cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("SMs %d clock %d kHz\n", p.multiProcessorCount, clk);
  const char* names[] = {"LOP3", "SHF", "IMAD", "IMAD.WIDE", "IMAD.HI", "ADD.CC+ADDC", "SUB.CC+ADDC", "LOP3+IMAD.WIDE"};
  int ops_per[] = {1, 1, 1, 1, 1, 2, 2, 2};
  int blocks = p.multiProcessorCount * 8, threads = 256;
  for (int rep = 0; rep < 2; rep++)
  for (int op = 0; op < 8; op++) {
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
      }
    };
    launch(); cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)blocks * threads * ITERS * CH * ops_per[op];
    if (rep) printf("%-24s %8.3f ms  %8.2f Tops/s (ptx-level ops)\n", names[op], ms, ops / ms / 1e9);
  }
  for (int var = 0; var < 5; var++)
  for (int bl : {148 * 4, 148 * 8}) {
    int ns = 1 << 13;
    auto launch = [&]() {
      switch (var) {
        case 0: kxoshiro<0><<<bl, 256>>>(d, 3, ns, 1); break;
        case 1: kxoshiro<1><<<bl, 256>>>(d, 3, ns, 1); break;
        case 2: kxoshiro<2><<<bl, 256>>>(d, 3, ns, 1); break;
        case 3: kxoshiro<3><<<bl, 256>>>(d, 3, ns, 1); break;
        case 4: kxoshiro<4><<<bl, 256>>>(d, 3, ns, 1); break;
      }
    };
    launch();
    cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("xoshiro VAR %d blocks=%d: %.3f ms  %.3f T draws/s\n", var, bl, ms, (double)bl * 256 * ns / ms / 1e9);
  }
  for (int var = 5; var < 8; var++)
  for (int bl : {148 * 4, 148 * 8}) {
    int ns = 1 << 13;
    auto launch = [&]() {
      switch (var) {
        case 5: kxo2<5><<<bl, 256>>>(d, 3, ns); break;
        case 6: kxo2<6><<<bl, 256>>>(d, 3, ns); break;
        case 7: kxo2<7><<<bl, 256>>>(d, 3, ns); break;
      }
    };
    launch();
    cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("xoshiro VAR %d blocks=%d: %.3f ms  %.3f T draws/s\n", var, bl, ms, (double)bl * 256 * ns / ms / 1e9);
  }
  for (int wps : {2, 3, 4, 6, 8, 16, 32}) {   // warps per SM for VAR 5
    int ns = 1 << 13;
    int threads = wps * 32;                         // 1 block per SM
    int bl = 148;
    kxo2<5><<<bl, threads>>>(d, 3, ns);
    cudaEventRecord(e0); kxo2<5><<<bl, threads>>>(d, 3, ns); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("VAR5 warps/SM=%d: %.3f T draws/s\n", wps, (double)bl * threads * ns / ms / 1e9);
  }
  uint32_t* onep; cudaMalloc(&onep, 64);
  { uint32_t h[8] = {1,1,1,1,1,1,1,1}; cudaMemcpy(onep, h, 32, cudaMemcpyHostToDevice); }
  for (int var = 8; var < 10; var++)
  for (int bl : {148 * 4, 148 * 8}) {
    int ns = 1 << 13;
    auto launch = [&]() {
      if (var == 8) kxo3<8><<<bl, 256>>>(d, 3, ns, onep); else kxo3<9><<<bl, 256>>>(d, 3, ns, onep);
    };
    launch();
    cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("xoshiro VAR %d blocks=%d: %.3f ms  %.3f T draws/s\n", var, bl, ms, (double)bl * 256 * ns / ms / 1e9);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
