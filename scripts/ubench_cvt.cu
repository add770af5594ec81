// ubench_cvt.cu -- E4M3 -> fp16 conversion throughput on sm_100a (FP8 KV variant,
// DESIGN.md §5): cycles per converted pair for the hardware unpack
// (cvt.rn.f16x2.e4m3x2 = F2FP.F16.E4M3.UNPACK_B), an integer path (PRMT with
// sign replication, two LOP3, one IMAD) and mixes, with W warps per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubench_cvt scripts/ubench_cvt.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint2 hw(uint32_t w) {
  uint2 r;
  asm volatile("{\n\t.reg .b16 lo, hi;\n\tmov.b32 {lo, hi}, %2;\n\t"
               "cvt.rn.f16x2.e4m3x2 %0, lo;\n\tcvt.rn.f16x2.e4m3x2 %1, hi;\n\t}"
               : "=r"(r.x), "=r"(r.y) : "r"(w));
  return r;
}
// fp16 bits of code*2^-8: sign at bit 15, (code & 0x7F) << 7
__device__ __forceinline__ uint2 sw(uint32_t w) {
  uint32_t a, b;
  asm volatile("prmt.b32 %0, %1, 0, 0x9180;" : "=r"(a) : "r"(w));   // [sgn c1][c1][sgn c0][c0]
  asm volatile("prmt.b32 %0, %1, 0, 0xB3A2;" : "=r"(b) : "r"(w));   // [sgn c3][c3][sgn c2][c2]
  uint2 r;
  r.x = ((a & 0x007F007Fu) << 7) | (a & 0x80008000u);
  r.y = ((b & 0x007F007Fu) << 7) | (b & 0x80008000u);
  return r;
}

__device__ __forceinline__ uint2 hw_scaled(uint32_t w) {   // hw cvt, then x 2^-8 (HMUL2, exact)
  uint2 r = hw(w);
  asm volatile("mul.rn.f16x2 %0, %0, %1;" : "+r"(r.x) : "r"(0x1C001C00u));
  asm volatile("mul.rn.f16x2 %0, %0, %1;" : "+r"(r.y) : "r"(0x1C001C00u));
  return r;
}

__global__ void check(int* bad) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;   // 2^16 code pairs
  const uint32_t w = i | (i << 16);
  const uint2 a = hw_scaled(w), b = sw(w);
  const uint32_t lo = i & 0xFF, hi = (i >> 8) & 0xFF;
  const bool nan = (lo & 0x7F) == 0x7F || (hi & 0x7F) == 0x7F;
  if (!nan && (a.x != b.x || a.y != b.y)) atomicAdd(bad, 1);
}

template <int MODE>
__global__ void k(uint32_t* out, long long* cyc, int iters, uint32_t seed) {
  uint32_t w[8];
  for (int i = 0; i < 8; ++i) w[i] = seed * (threadIdx.x + 1 + i) ^ (0x9E3779B9u * i);
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      uint2 r;
      if (MODE == 0) r = hw(w[i]);
      else if (MODE == 1) r = sw(w[i]);
      else if (MODE == 2) r = (i & 1) ? sw(w[i]) : hw(w[i]);
      else if (MODE == 3) r = (i % 3 == 0) ? hw(w[i]) : sw(w[i]);
      else r = (i & 1) ? sw(w[i]) : hw_scaled(w[i]);
      acc ^= r.x + r.y;
      w[i] += 0x01010101u;
    }
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  uint32_t* out; long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
  const int iters = 4096;
  const char* names[5] = {"hw cvt", "int path", "mix 1:1", "mix 1:2", "mix hws"};
  int* bad; cudaMalloc(&bad, 4); cudaMemset(bad, 0, 4);
  check<<<256, 256>>>(bad);
  int hbad; cudaMemcpy(&hbad, bad, 4, cudaMemcpyDeviceToHost);
  printf("int path == hw cvt * 2^-8 on all non-NaN code pairs: %s (%d mismatches)\n", hbad ? "NO" : "yes", hbad);
  // check the int path equals hw cvt * 2^-8 (as fp16 values) for all 2^16 pairs on the host side: skipped here
  for (int mode = 0; mode < 5; ++mode)
    for (int warps : {1, 2, 4, 8}) {
      auto f = mode == 0 ? k<0> : mode == 1 ? k<1> : mode == 2 ? k<2> : mode == 3 ? k<3> : k<4>;
      f<<<148, warps * 32>>>(out, cyc, 16, 1);
      f<<<148, warps * 32>>>(out, cyc, iters, 7);
      cudaDeviceSynchronize();
      long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      // pairs converted per SM per clock: warps * 32 lanes * iters * 8 words * 2 pairs / cycles
      double pairs = (double)warps * 32 * iters * 16;
      printf("%-9s warps/SM %d: %.2f pairs/clk/SM (%.1f cyc per warp-pair-instr)\n", names[mode], warps,
             pairs / c, (double)c / (iters * 16.0));
    }
  return 0;
}
