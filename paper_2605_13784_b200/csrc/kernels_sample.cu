// kernels_sample.cu — on-device greedy sampling for sm_100a.
//
// For every row of logits: the argmax token (ties toward the lowest id, SPEC
// greedy_sample), its logit l1, the second-highest logit value l2 and the
// logit gap l1 - l2 (Eq. flash-cache, Eq. logit-gap), so
// the host never reads the vocabulary-sized logits back.  Optionally a window
// of draft tokens is verified in the same call: n_accept = the number of
// leading rows whose argmax equals the draft ("batched variant for
// accepting or rejecting a window of speculated tokens").
//
// HBM-bound (one read of the logits): the grid is rows x splits CTAs, each
// streaming a contiguous chunk of one row with 16-byte loads and reducing a
// (max, argmax, second max) triple per thread, per warp (shuffles) and per CTA
// (shared memory); the last CTA of a row (atomic ticket) merges the row's
// partials, and the last row to finish computes n_accept.  NaN logits are
// ignored (they compare below every number).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include "store.h"

namespace ssa {

namespace {

struct Top2 {   // SampleParams::partials element
  float m1;   // highest value
  int32_t i1; // its lowest index
  float m2;   // second-highest value (== m1 when the top value occurs twice)
};

__device__ __forceinline__ void top2_push(Top2& t, float x, int32_t i) {
  // elements of one thread arrive in increasing index order; i1 < 0 = empty
  if (t.i1 < 0 || x > t.m1) {
    t.m2 = t.m1;
    t.m1 = x;
    t.i1 = i;
  } else if (x > t.m2) {
    t.m2 = x;
  }
}

__device__ __forceinline__ Top2 top2_merge(const Top2& a, const Top2& b) {
  if (b.i1 < 0) return a;
  if (a.i1 < 0) return b;
  const bool a_top = a.m1 > b.m1 || (a.m1 == b.m1 && a.i1 < b.i1);
  const Top2& t = a_top ? a : b;
  const Top2& o = a_top ? b : a;
  // the runner-up is the top's own second or the other's first (equal tops: gap 0)
  return Top2{t.m1, t.i1, fmaxf(t.m2, o.m1)};
}

__device__ __forceinline__ Top2 warp_top2(Top2 t) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    Top2 u;
    u.m1 = __shfl_xor_sync(0xffffffffu, t.m1, o);
    u.i1 = __shfl_xor_sync(0xffffffffu, t.i1, o);
    u.m2 = __shfl_xor_sync(0xffffffffu, t.m2, o);
    t = top2_merge(t, u);
  }
  return t;
}

template <typename T>
__device__ __forceinline__ void load8(const T* p, float (&v)[8]);
template <>
__device__ __forceinline__ void load8<float>(const float* p, float (&v)[8]) {
  const float4 a = __ldcs(reinterpret_cast<const float4*>(p));
  const float4 b = __ldcs(reinterpret_cast<const float4*>(p) + 1);
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
  v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
template <>
__device__ __forceinline__ void load8<__nv_bfloat16>(const __nv_bfloat16* p, float (&v)[8]) {
  const uint4 a = __ldcs(reinterpret_cast<const uint4*>(p));
  const uint32_t w[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    v[2 * i] = __uint_as_float(w[i] << 16);
    v[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
  }
}
template <typename T>
__device__ __forceinline__ float to_f(T x);
template <>
__device__ __forceinline__ float to_f<float>(float x) { return x; }
template <>
__device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 x) { return __bfloat162float(x); }

constexpr int kThreads = 256;

template <typename T>
__global__ void __launch_bounds__(kThreads) greedy_kernel(const SampleParams p) {
  const int row = blockIdx.y;
  const int split = blockIdx.x;
  const T* x = static_cast<const T*>(p.logits) + (int64_t)row * p.row_stride;
  // contiguous chunk of this split, a multiple of 8 elements except the last
  const int64_t per = ((p.vocab + p.splits - 1) / p.splits + 7) / 8 * 8;
  const int64_t lo = (int64_t)split * per;
  const int64_t hi = lo + per < (int64_t)p.vocab ? lo + per : (int64_t)p.vocab;
  Top2 t{-CUDART_INF_F, -1, -CUDART_INF_F};
  const bool aligned = (reinterpret_cast<uintptr_t>(x) & 15) == 0;   // lo is a multiple of 8 elements
  int64_t i = lo + (int64_t)threadIdx.x * 8;
  constexpr int64_t kStep = (int64_t)kThreads * 8;
  if (aligned) {
    // four 8-element groups in flight per thread (memory-level parallelism)
    for (; i + 3 * kStep + 8 <= hi; i += 4 * kStep) {
      float v[4][8];
#pragma unroll
      for (int u = 0; u < 4; ++u) load8<T>(x + i + u * kStep, v[u]);
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (v[u][j] == v[u][j]) top2_push(t, v[u][j], (int32_t)(i + u * kStep + j));
    }
  }
  for (; i < hi; i += kStep) {
    if (aligned && i + 8 <= hi) {
      float v[8];
      load8<T>(x + i, v);
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (v[j] == v[j]) top2_push(t, v[j], (int32_t)(i + j));
    } else {   // ragged tail or unaligned row: element by element, still increasing
      for (int j = 0; j < 8 && i + j < hi; ++j) {
        const float v = to_f<T>(x[i + j]);
        if (v == v) top2_push(t, v, (int32_t)(i + j));
      }
    }
  }
  t = warp_top2(t);
  __shared__ Top2 red[kThreads / 32];
  __shared__ int last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) red[warp] = t;
  __syncthreads();
  if (warp == 0) {
    t = lane < kThreads / 32 ? red[lane] : Top2{-CUDART_INF_F, -1, -CUDART_INF_F};
    t = warp_top2(t);
    if (lane == 0) {
      Top2* part = static_cast<Top2*>(p.partials) + (int64_t)row * p.splits + split;
      *part = t;
      __threadfence();
      const int ticket = atomicAdd(p.row_counters + row, 1);
      last = ticket == p.splits - 1;
    }
  }
  __syncthreads();
  if (!last) return;
  // ---- last CTA of the row: merge the row's partials (lowest split first)
  __threadfence();
  if (warp == 0) {
    Top2 m{-CUDART_INF_F, -1, -CUDART_INF_F};
    for (int s = lane; s < p.splits; s += 32) {
      const Top2* q = static_cast<const Top2*>(p.partials) + (int64_t)row * p.splits + s;
      Top2 u;
      u.m1 = __ldcg(&q->m1);
      u.i1 = __ldcg(&q->i1);
      u.m2 = __ldcg(&q->m2);
      m = top2_merge(m, u);
    }
    m = warp_top2(m);
    if (lane == 0) {
      p.out_ids[row] = m.i1;
      if (p.out_gap) p.out_gap[row] = m.i1 >= 0 ? m.m1 - m.m2 : 0.f;   // fp32 subtraction
      if (p.out_top) {
        p.out_top[2 * row] = m.m1;
        p.out_top[2 * row + 1] = m.m2;
      }
      p.row_counters[row] = 0;   // ready for the next call
      if (p.draft) {
        __threadfence();
        const int done = atomicAdd(p.row_counters + p.n_rows, 1);
        if (done == p.n_rows - 1) {
          // every row is final: the accepted prefix of the draft window
          __threadfence();
          int n = 0;
          while (n < p.n_rows && __ldcg(p.out_ids + n) == p.draft[n]) ++n;
          *p.out_n_accept = n;
          p.row_counters[p.n_rows] = 0;
        }
      }
    }
  }
}

}  // namespace

size_t sample_partial_bytes() { return sizeof(Top2); }

cudaError_t launch_greedy(const SampleParams& p, bool bf16, cudaStream_t s) {
  dim3 grid(p.splits, p.n_rows);
  if (bf16) greedy_kernel<__nv_bfloat16><<<grid, kThreads, 0, s>>>(p);
  else greedy_kernel<float><<<grid, kThreads, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace ssa
