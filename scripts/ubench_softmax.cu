// Micro-benchmark (not part of the library): the tcgen05 kernel's per-tile
// softmax exp loop in isolation (one row of 128 fp32 scores per thread ->
// FFMA2 scale/shift, 2x MUFU.EX2, FADD2 row sum, F2FP bf16 pack), timed with
// clock64 at 1 and 2 warps per SMSP.  Shows whether the loop itself can run at
// the MUFU bound (128 ex2 x 8 cycles = 1024 cycles per warp per tile).
#include <cuda_bf16.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float ex2v(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ void fence32(float* r) {
  asm volatile(""
               : "+f"(r[0]), "+f"(r[1]), "+f"(r[2]), "+f"(r[3]), "+f"(r[4]), "+f"(r[5]), "+f"(r[6]), "+f"(r[7]),
                 "+f"(r[8]), "+f"(r[9]), "+f"(r[10]), "+f"(r[11]), "+f"(r[12]), "+f"(r[13]), "+f"(r[14]),
                 "+f"(r[15]), "+f"(r[16]), "+f"(r[17]), "+f"(r[18]), "+f"(r[19]), "+f"(r[20]), "+f"(r[21]),
                 "+f"(r[22]), "+f"(r[23]), "+f"(r[24]), "+f"(r[25]), "+f"(r[26]), "+f"(r[27]), "+f"(r[28]),
                 "+f"(r[29]), "+f"(r[30]), "+f"(r[31]));
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
__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}

template <int kVariant>
__global__ void softmax_loop(const float* in, uint32_t* out, long long* cyc, int tiles) {
  float sv[128];
#pragma unroll
  for (int i = 0; i < 128; ++i) sv[i] = in[(threadIdx.x * 7 + i) & 1023];
  uint32_t acc = 0;
  float l = 0.f;
  const float c = 0.127f;
  __syncthreads();
  const long long t0 = clock64();
  for (int t = 0; t < tiles; ++t) {
    const float mc = 0.5f + t * 1e-7f;
    const float2 c2 = make_float2(c, c), nmc2 = make_float2(-mc, -mc);
    float2 sum4[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
    uint32_t pk[64];
    if (kVariant >= 5) {
      constexpr int kPoly = kVariant - 4;   // poly pairs of every 8
#pragma unroll
      for (int i = 0; i < 64; ++i) {
        const float2 x = __ffma2_rn(make_float2(sv[2 * i], sv[2 * i + 1]), c2, nmc2);
        const float2 e = ((i & 7) >= 8 - kPoly) ? poly2(x) : make_float2(ex2(x.x), ex2(x.y));
        sum4[i & 3] = __fadd2_rn(sum4[i & 3], e);
        pk[i] = pack_bf16(e.x, e.y);
      }
    } else if (kVariant <= 1) {
#pragma unroll
      for (int i = 0; i < 64; ++i) {
        const float2 x = __ffma2_rn(make_float2(sv[2 * i], sv[2 * i + 1]), c2, nmc2);
        const float2 e = make_float2(ex2(x.x), ex2(x.y));
        if (kVariant == 0) sum4[i & 3] = __fadd2_rn(sum4[i & 3], e);
        pk[i] = pack_bf16(e.x, e.y);
      }
    } else {
      // chunked software pipeline: ex2 of chunk q (volatile, in order), then the
      // pack/sum of chunk q-1 -- consumers sit >= 32 MUFU ops after producers
      float ev[128];
      constexpr int kCh = kVariant == 2 ? 128 : (kVariant == 3 ? 32 : 16);
#pragma unroll
      for (int q = 0; q <= 128 / kCh; ++q) {
        if (q < 128 / kCh) {
#pragma unroll
          for (int i = q * kCh / 2; i < (q + 1) * kCh / 2; ++i) {
            const float2 x = __ffma2_rn(make_float2(sv[2 * i], sv[2 * i + 1]), c2, nmc2);
            ev[2 * i] = ex2v(x.x);
            ev[2 * i + 1] = ex2v(x.y);
          }
        }
        if (q > 0) {
#pragma unroll
          for (int f = (q - 1) * kCh; f < q * kCh; f += 32) fence32(ev + f);
#pragma unroll
          for (int i = (q - 1) * kCh / 2; i < q * kCh / 2; ++i) {
            const float2 e = make_float2(ev[2 * i], ev[2 * i + 1]);
            sum4[i & 3] = __fadd2_rn(sum4[i & 3], e);
            pk[i] = pack_bf16(e.x, e.y);
          }
        }
      }
    }
#pragma unroll
    for (int i = 0; i < 64; ++i) acc ^= pk[i];
    const float2 s = __fadd2_rn(__fadd2_rn(sum4[0], sum4[1]), __fadd2_rn(sum4[2], sum4[3]));
    l += s.x + s.y;
    sv[0] += 1e-3f;
  }
  const long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc ^ __float_as_uint(l);
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  float* in;
  uint32_t* out;
  long long* cyc;
  cudaMalloc(&in, 1024 * 4);
  cudaMemset(in, 0, 1024 * 4);
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 148 * 8);
  const int tiles = 256;
  for (int threads : {128, 256}) {
    for (int v : {0, 5, 6, 7}) {
      for (int rep = 0; rep < 2; ++rep) {
        if (v == 0) softmax_loop<0><<<148, threads>>>(in, out, cyc, tiles);
        else if (v == 1) softmax_loop<1><<<148, threads>>>(in, out, cyc, tiles);
        else if (v == 2) softmax_loop<2><<<148, threads>>>(in, out, cyc, tiles);
        else if (v == 3) softmax_loop<3><<<148, threads>>>(in, out, cyc, tiles);
        else if (v == 4) softmax_loop<4><<<148, threads>>>(in, out, cyc, tiles);
        else if (v == 5) softmax_loop<5><<<148, threads>>>(in, out, cyc, tiles);
        else if (v == 6) softmax_loop<6><<<148, threads>>>(in, out, cyc, tiles);
        else softmax_loop<7><<<148, threads>>>(in, out, cyc, tiles);
      }
      cudaDeviceSynchronize();
      long long c;
      cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      printf("warps/SMSP %d variant %d (%s): %.0f cycles per tile per warp (MUFU bound %d)\n", threads / 128, v,
             v == 0 ? "exp+sum+pack" : v == 1 ? "exp+pack" : v == 2 ? "all ex2 then pack/sum" : v == 3 ? "32-col chunk pipeline" : v == 4 ? "16-col chunk pipeline" : v == 5 ? "1/8 poly" : v == 6 ? "2/8 poly" : "3/8 poly", (double)c / tiles, 1024 * threads / 128);
    }
  }
  return 0;
}
