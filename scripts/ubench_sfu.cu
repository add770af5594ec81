// Micro-benchmark (not part of the library): per-SM throughput of the softmax
// instruction mix on this GPU — MUFU.EX2, FFMA, FFMA2, F2FP pack, FMNMX3 and the
// FMA-pipe polynomial exp2 — measured with clock64 in one CTA per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_sfu ubench_sfu.cu
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdint>

constexpr int kIters = 4096;
constexpr int kChains = 16;

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float2 poly2(float2 x) {
  x.x = fmaxf(x.x, -126.f);
  x.y = fmaxf(x.y, -126.f);
  const float2 t = __fadd2_rn(x, make_float2(12582912.f, 12582912.f));
  const float2 r = __fadd2_rn(t, make_float2(-12582912.f, -12582912.f));
  const float2 f = __fadd2_rn(x, make_float2(-r.x, -r.y));
  float2 q = __ffma2_rn(make_float2(0.0551716685f, 0.0551716685f), f, make_float2(0.2426111549f, 0.2426111549f));
  q = __ffma2_rn(q, f, make_float2(0.6932609677f, 0.6932609677f));
  q = __ffma2_rn(q, f, make_float2(0.9999280572f, 0.9999280572f));
  return make_float2(__uint_as_float(__float_as_uint(q.x) + (__float_as_uint(t.x) << 23)),
                     __uint_as_float(__float_as_uint(q.y) + (__float_as_uint(t.y) << 23)));
}

template <int kOp>
__global__ void bench(float* out, long long* cyc, float seed) {
  float a[kChains];
  for (int i = 0; i < kChains; ++i) a[i] = seed * (threadIdx.x + i) * 1e-3f - 1.f;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < kChains; i += 2) {
      if (kOp == 0) {          // MUFU.EX2
        a[i] = ex2(a[i]) - 1.0f;      // FADD keeps the chain in range; counted separately
        a[i + 1] = ex2(a[i + 1]) - 1.0f;
      } else if (kOp == 1) {   // FFMA
        a[i] = fmaf(a[i], 0.999f, 0.001f);
        a[i + 1] = fmaf(a[i + 1], 0.999f, 0.001f);
      } else if (kOp == 2) {   // FFMA2
        float2 v = __ffma2_rn(make_float2(a[i], a[i + 1]), make_float2(0.999f, 0.999f), make_float2(1e-3f, 1e-3f));
        a[i] = v.x;
        a[i + 1] = v.y;
      } else if (kOp == 3) {   // poly exp2 pair (+ 2 FADD to stay in range)
        float2 v = poly2(make_float2(a[i], a[i + 1]));
        a[i] = v.x - 1.0f;
        a[i + 1] = v.y - 1.0f;
      } else if (kOp == 4) {   // F2FP pack + unpack
        __nv_bfloat162 b = __floats2bfloat162_rn(a[i], a[i + 1]);
        uint32_t u = *reinterpret_cast<uint32_t*>(&b);
        a[i] = __uint_as_float(u << 16) + 1e-3f;
        a[i + 1] = __uint_as_float(u & 0xffff0000u) + 1e-3f;
      } else if (kOp == 5) {   // FMNMX3
        a[i] = fmaxf(a[i], fmaxf(a[i + 1], a[(i + 2) % kChains])) - 1e-3f;
        a[i + 1] = fmaxf(a[i + 1], fmaxf(a[i], a[(i + 3) % kChains])) - 1e-3f;
      } else if (kOp == 6) {   // FADD2
        float2 v = __fadd2_rn(make_float2(a[i], a[i + 1]), make_float2(1e-3f, -1e-3f));
        a[i] = v.x;
        a[i + 1] = v.y;
      }
    }
  }
  const long long t1 = clock64();
  float s = 0.f;
  for (int i = 0; i < kChains; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * sizeof(float));
  cudaMalloc(&cyc, 148 * sizeof(long long));
  const char* names[] = {"ex2(+FADD)", "FFMA", "FFMA2", "poly2(+FADD)", "F2FP+2 FADD", "FMNMX3(+FADD)", "FADD2"};
  for (int threads : {128, 256, 512}) {
    for (int op = 0; op < 7; ++op) {
      for (int rep = 0; rep < 2; ++rep) {
        switch (op) {
          case 0: bench<0><<<148, threads>>>(out, cyc, 1.f); break;
          case 1: bench<1><<<148, threads>>>(out, cyc, 1.f); break;
          case 2: bench<2><<<148, threads>>>(out, cyc, 1.f); break;
          case 3: bench<3><<<148, threads>>>(out, cyc, 1.f); break;
          case 4: bench<4><<<148, threads>>>(out, cyc, 1.f); break;
          case 5: bench<5><<<148, threads>>>(out, cyc, 1.f); break;
          case 6: bench<6><<<148, threads>>>(out, cyc, 1.f); break;
        }
      }
      cudaDeviceSynchronize();
      long long c;
      cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
      const double elems = (double)threads * kIters * kChains;
      printf("threads %3d  %-14s  %.2f elements/clk/SM  (%.3f clk per warp-instr-of-32-elems)\n", threads,
             names[op], elems / c, 32.0 / (elems / c) * (threads / 32) / (threads / 32) );
    }
  }
  return 0;
}
