// kernels_simt.cu — CUDA-core kernels of the session-attention path (sm_100a).
//
//   attn_simt     split-KV attention of a q tile over paged cached keys plus the
//                 segment's own keys (causal), online softmax in fp32.  Used for
//                 fp32 mode (KS, 1e-5 parity) and for small-row bf16 work (KD,
//                 e.g. 1-token queries at 4 FLOP/B where tensor cores do not pay).
//   combine       log-sum-exp merge of split partials (KC; reading R-11).
//   scatter       append of new K/V rows into pages (KA; bit-exact, Alg. 1).
//   gather        read-back of pages (tests / digest only).
//
// Math (Eq. attention): s = scale*q.k, p = exp(s - m),
// o = sum p v / sum p.  We fold scale*log2(e) into q and use exp2.
#include <cuda_bf16.h>
#include <math_constants.h>
#include <stdint.h>

#include "ssa_internal.h"

namespace ssa {

namespace {

constexpr int kThreads = 128;
constexpr int kBK = 64;   // keys per SIMT tile
constexpr int kRT = 32;   // rows per SIMT unit

__device__ __forceinline__ float ld_f(const float* p, int64_t i) { return p[i]; }
__device__ __forceinline__ float ld_f(const __nv_bfloat16* p, int64_t i) { return __bfloat162float(p[i]); }
__device__ __forceinline__ void st_f(float* p, int64_t i, float v) { p[i] = v; }
__device__ __forceinline__ void st_f(__nv_bfloat16* p, int64_t i, float v) { p[i] = __float2bfloat16_rn(v); }

// 16-byte vector load of VEC = 16 / sizeof(T) consecutive elements, as floats.
__device__ __forceinline__ void ld_vec16(const float* p, int64_t i, float (&out)[4]) {
  const float4 x = __ldg(reinterpret_cast<const float4*>(p + i));
  out[0] = x.x; out[1] = x.y; out[2] = x.z; out[3] = x.w;
}
__device__ __forceinline__ void ld_vec16(const __nv_bfloat16* p, int64_t i, float (&out)[8]) {
  const uint4 x = __ldg(reinterpret_cast<const uint4*>(p + i));
  const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    out[2 * k] = __uint_as_float(w[k] << 16);
    out[2 * k + 1] = __uint_as_float(w[k] & 0xFFFF0000u);
  }
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <typename T, int D>
__global__ void __launch_bounds__(kThreads) attn_simt_kernel(const AttnParams p) {
  constexpr int NV = kRT * D / kThreads;      // O accumulators per thread
  constexpr int KS = D + 1;                   // padded K row (bank-conflict free dots)
  extern __shared__ float smem[];
  float* Qs = smem;                           // [kRT][D]
  float* Ks = Qs + kRT * D;                   // [kBK][D+1]
  float* Vs = Ks + kBK * KS;                  // [kBK][D]
  float* Ss = Vs + kBK * D;                   // [kRT][kBK]
  float* mrow = Ss + kRT * kBK;               // running max (log2 domain)
  float* lrow = mrow + kRT;                   // running sum
  float* arow = lrow + kRT;                   // rescale factor of this tile

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int u = blockIdx.x, ly = blockIdx.y;
  const WorkUnit wu = p.units[u];
  const SegDesc sg = p.segs[wu.seg];
  const int G = p.G;
  const int rows = wu.q_ntok * G;
  const int64_t layer = p.layer0 + ly;
  const int64_t in_row0 = (p.in_layer_stride ? (int64_t)ly * p.rows_per_layer : 0) + sg.row0;
  const T* Q = static_cast<const T*>(p.Q);
  const T* Kt = static_cast<const T*>(p.Kt);
  const T* Vt = static_cast<const T*>(p.Vt);
  const T* PK = static_cast<const T*>(p.poolK);
  const T* PV = static_cast<const T*>(p.poolV);

  constexpr int VEC = 16 / sizeof(T);           // elements per 16-byte load
  for (int idx = tid; idx < kRT * D / VEC; idx += kThreads) {
    const int r = idx * VEC / D, e = idx * VEC % D;
    float v[VEC];
#pragma unroll
    for (int c = 0; c < VEC; ++c) v[c] = 0.f;
    if (r < rows) {
      const int64_t row = in_row0 + wu.q_tok0 + r / G;
      const int h = wu.kv_head * G + r % G;
      ld_vec16(Q, (row * p.Hq + h) * D + e, v);
    }
#pragma unroll
    for (int c = 0; c < VEC; ++c) Qs[r * D + e + c] = v[c] * p.scale_log2;
  }
  if (tid < kRT) { mrow[tid] = -CUDART_INF_F; lrow[tid] = 0.f; }
  float acc[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) acc[i] = 0.f;

  const int n_pool_tiles = (sg.n_slots + kBK - 1) / kBK;
  for (int tile = wu.tile_lo; tile < wu.tile_hi; ++tile) {
    const bool is_pool = tile < n_pool_tiles;
    const int key0 = (is_pool ? tile : tile - n_pool_tiles) * kBK;
    __syncthreads();
    for (int idx = tid; idx < kBK * D / VEC; idx += kThreads) {   // 16-byte loads
      const int j = idx * VEC / D, e = idx * VEC % D;
      float kv[VEC], vv[VEC];
#pragma unroll
      for (int c = 0; c < VEC; ++c) kv[c] = vv[c] = 0.f;
      const int key = key0 + j;
      if (is_pool) {
        if (key < sg.n_slots && !(key >= sg.hole_lo && key < sg.hole_hi)) {
          const int64_t page = sg.pages[key / p.P];
          const int64_t off = (((layer * p.num_pages + page) * p.Hkv + wu.kv_head) * p.P + key % p.P) * D + e;
          ld_vec16(PK, off, kv);
          ld_vec16(PV, off, vv);
        }
      } else if (key < sg.tail_m) {
        const int64_t off = ((in_row0 + key) * p.Hkv + wu.kv_head) * D + e;
        ld_vec16(Kt, off, kv);
        ld_vec16(Vt, off, vv);
      }
#pragma unroll
      for (int c = 0; c < VEC; ++c) {
        Ks[j * KS + e + c] = kv[c];
        Vs[j * D + e + c] = vv[c];
      }
    }
    __syncthreads();
    for (int idx = tid; idx < kRT * kBK; idx += kThreads) {
      const int r = idx / kBK, j = idx % kBK;
      const int key = key0 + j;
      bool valid = r < rows;
      if (is_pool) {
        valid = valid && key < sg.n_slots && !(key >= sg.hole_lo && key < sg.hole_hi);
      } else {
        const int tok = wu.q_tok0 + r / G;
        valid = valid && key < sg.tail_m && (p.fault == 2 ? key < tok : key <= tok);
      }
      float s = -CUDART_INF_F;
      if (valid) {
        const float* q = Qs + r * D;
        const float* k = Ks + j * KS;
        float a = 0.f;
#pragma unroll 16
        for (int e = 0; e < D; ++e) a = fmaf(q[e], k[e], a);
        s = a;
      }
      Ss[idx] = s;
    }
    __syncthreads();
    for (int r = warp; r < kRT; r += kThreads / 32) {
      const float s0 = Ss[r * kBK + lane], s1 = Ss[r * kBK + lane + 32];
      const float m_old = mrow[r];
      const float m_new = fmaxf(m_old, warp_max(fmaxf(s0, s1)));
      float p0 = 0.f, p1 = 0.f, alpha = 1.f;
      if (m_new != -CUDART_INF_F) {
        p0 = exp2f(s0 - m_new);
        p1 = exp2f(s1 - m_new);
        alpha = exp2f(m_old - m_new);
      }
      const float sum = warp_sum(p0 + p1);
      __syncwarp();   // every lane's reads of this row (S, mrow) before the writes below
      Ss[r * kBK + lane] = p0;
      Ss[r * kBK + lane + 32] = p1;
      if (lane == 0) {
        lrow[r] = lrow[r] * alpha + sum;
        mrow[r] = m_new;
        arow[r] = alpha;
      }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int idx = tid + i * kThreads;
      const int r = idx / D, e = idx % D;
      float a = acc[i] * arow[r];
      const float* pr = Ss + r * kBK;
#pragma unroll 8
      for (int j = 0; j < kBK; ++j) a = fmaf(pr[j], Vs[j * D + e], a);
      acc[i] = a;
    }
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int idx = tid + i * kThreads;
    const int r = idx / D, e = idx % D;
    if (r >= rows) continue;
    const float l = lrow[r];
    const float o = l > 0.f ? acc[i] / l : 0.f;
    if (wu.group < 0) {
      const int64_t row = in_row0 + wu.q_tok0 + r / G;
      const int h = wu.kv_head * G + r % G;
      st_f(static_cast<T*>(p.O), (row * p.Hq + h) * D + e, o);
    } else {
      const int64_t slot = (int64_t)ly * p.n_units + u;
      p.part_o[(slot * kRT + r) * D + e] = o;
      if (e == 0) p.part_lse[slot * kRT + r] = l > 0.f ? mrow[r] + log2f(l) : -CUDART_INF_F;
    }
  }
}

// Split-KV merge (KC).  One CTA per (group, layer): per-row weights
// w_s = 2^(lse_s - L) / sum_s 2^(lse_s - L) are computed once into smem, then
// the 128-bit-vectorized weighted sum runs over all (row, 4-column) pairs.
// Partials carry normalized o_s and lse_s in log2 units (reading R-11).
constexpr int kCombineRows = 32;   // rows of a group per combine CTA (max; fewer for small launches)

template <typename T>
__global__ void __launch_bounds__(256) combine_kernel(const CombineParams p) {
  extern __shared__ float wsm[];                       // [n_splits][CR]
  const int CR = p.combine_rows;
  const int g = blockIdx.x, ly = blockIdx.y, r0 = blockIdx.z * CR;
  const Group gr = p.groups[g];
  if (gr.n_splits == 0) return;   // merged inside its attention CTA
  const int rows = gr.q_ntok * p.G;
  if (r0 >= rows) return;
  const int nr = min(CR, rows - r0);
  const SegDesc sg = p.segs[gr.seg];
  const int RT = p.rows_tile;
  const int64_t slot0 = (int64_t)ly * p.n_units + gr.unit0;
  const int NS = gr.n_splits;
  for (int rr = threadIdx.x; rr < nr; rr += blockDim.x) {
    const int r = r0 + rr;
    float L = -CUDART_INF_F;
    for (int s = 0; s < NS; ++s) L = fmaxf(L, p.part_lse[(slot0 + s) * RT + r]);
    float wsum = 0.f;
    for (int s = 0; s < NS; ++s) {
      const float ls = p.part_lse[(slot0 + s) * RT + r];
      const float w = ls == -CUDART_INF_F ? 0.f : exp2f(ls - L);
      wsm[s * CR + rr] = w;
      wsum += w;
    }
    const float inv = wsum > 0.f ? 1.f / wsum : 0.f;
    for (int s = 0; s < NS; ++s) wsm[s * CR + rr] *= inv;
    if (p.lse_out || p.n_peers > 0) {
      const int64_t row = (p.in_layer_stride ? (int64_t)ly * p.rows_per_layer : 0) + sg.row0 + gr.q_tok0 + r / p.G;
      const float lse = wsum > 0.f ? L + log2f(wsum) : -CUDART_INF_F;
      const int64_t at = row * p.Hq + gr.kv_head * p.G + r % p.G;
      if (p.n_peers > 0) {
        for (int q = 0; q < p.n_peers; ++q) reinterpret_cast<float*>(p.peer_chunk[q])[p.lse_off + at] = lse;
      } else {
        p.lse_out[at] = lse;
      }
    }
  }
  __syncthreads();
  if (!p.write_o) return;
  const int64_t in_row0 = (p.in_layer_stride ? (int64_t)ly * p.rows_per_layer : 0) + sg.row0;
  const int d4 = p.D / 4;
  for (int idx = threadIdx.x; idx < nr * d4; idx += blockDim.x) {
    const int rr = idx / d4, r = r0 + rr, e = (idx % d4) * 4;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    const float4* src = reinterpret_cast<const float4*>(p.part_o + ((slot0)*RT + r) * p.D + e);
    const int64_t split_stride4 = (int64_t)RT * p.D / 4;   // float4s between consecutive splits
    int s = 0;
    for (; s + 4 <= NS; s += 4) {   // four independent loads in flight
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = __ldcs(src + (s + u) * split_stride4);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float w = wsm[(s + u) * CR + rr];
        acc.x = fmaf(w, v[u].x, acc.x);
        acc.y = fmaf(w, v[u].y, acc.y);
        acc.z = fmaf(w, v[u].z, acc.z);
        acc.w = fmaf(w, v[u].w, acc.w);
      }
    }
    for (; s < NS; ++s) {
      const float w = wsm[s * CR + rr];
      const float4 v = __ldcs(src + s * split_stride4);
      acc.x = fmaf(w, v.x, acc.x);
      acc.y = fmaf(w, v.y, acc.y);
      acc.z = fmaf(w, v.z, acc.z);
      acc.w = fmaf(w, v.w, acc.w);
    }
    const int64_t row = in_row0 + gr.q_tok0 + r / p.G;
    const int h = gr.kv_head * p.G + r % p.G;
    if (p.n_peers > 0) {
      // the rank partial goes straight into every peer's gathered buffer
      for (int q = 0; q < p.n_peers; ++q)
        *reinterpret_cast<float4*>(reinterpret_cast<float*>(p.peer_chunk[q]) + (row * p.Hq + h) * p.D + e) = acc;
    } else if (p.o_f32) {
      *reinterpret_cast<float4*>(p.o_f32 + (row * p.Hq + h) * p.D + e) = acc;
    } else {
      T* out = static_cast<T*>(p.O) + (row * p.Hq + h) * p.D + e;
      st_f(out, 0, acc.x);
      st_f(out, 1, acc.y);
      st_f(out, 2, acc.z);
      st_f(out, 3, acc.w);
    }
  }
}

// Cross-rank merge (A9): one warp per (row, head); world packed chunks of
// [O fp32 rows*Hq*D | lse rows*Hq] (log2 units), reading R-11.
template <typename T>
__global__ void __launch_bounds__(256) merge_ranks_kernel(const float* parts, int world, int64_t rows, int Hq, int D,
                                                          T* O) {
  const int64_t rh = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (rh >= rows * Hq) return;
  const int64_t chunk = rows * Hq * (int64_t)(D + 1);
  const float* lse = parts + rows * Hq * (int64_t)D;
  float L = -CUDART_INF_F;
  for (int r = 0; r < world; ++r) L = fmaxf(L, lse[r * chunk + rh]);
  float wsum = 0.f;
  for (int r = 0; r < world; ++r) {
    const float l = lse[r * chunk + rh];
    if (l != -CUDART_INF_F) wsum += exp2f(l - L);
  }
  const float inv = wsum > 0.f ? 1.f / wsum : 0.f;
  for (int e = lane; e < D; e += 32) {
    float acc = 0.f;
    for (int r = 0; r < world; ++r) {
      const float l = lse[r * chunk + rh];
      if (l != -CUDART_INF_F) acc = fmaf(exp2f(l - L), parts[r * chunk + rh * D + e], acc);
    }
    st_f(O, rh * D + e, acc * inv);
  }
}

// 16-byte chunks: (token, kv head, chunk).  Bit-exact copy into pages.
__global__ void __launch_bounds__(256) scatter_kernel(const ScatterParams p) {
  const int ly = blockIdx.y;
  const int64_t layer = p.layer0 + ly;
  const int chunks = p.D * p.elem_bytes / 16;
  const int64_t total = p.total_tokens * p.Hkv * chunks;
  const int64_t in_l = p.in_layer_stride ? (int64_t)ly * p.rows_per_layer : 0;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int c = idx % chunks;
    const int h = (idx / chunks) % p.Hkv;
    const int64_t t = idx / ((int64_t)chunks * p.Hkv);
    int lo = 0, hi = p.n_segs;  // find seg with tok_prefix[s] <= t < tok_prefix[s+1]
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (p.tok_prefix[mid] <= t) lo = mid; else hi = mid;
    }
    const SegDesc sg = p.segs[lo];
    const int64_t tl = t - p.tok_prefix[lo];
    const int64_t slot = sg.append_slot0 + tl;
    const int64_t page = sg.pages[slot / p.P];
    const int64_t src = ((in_l + sg.row0 + tl) * p.Hkv + h) * (int64_t)p.D * p.elem_bytes + c * 16;
    const int64_t dst = (((layer * p.num_pages + page) * p.Hkv + h) * p.P + slot % p.P) * (int64_t)p.D * p.elem_bytes + c * 16;
    const int4 kv = *reinterpret_cast<const int4*>(static_cast<const char*>(p.K) + src);
    const int4 vv = *reinterpret_cast<const int4*>(static_cast<const char*>(p.V) + src);
    *reinterpret_cast<int4*>(static_cast<char*>(p.poolK) + dst) = kv;
    *reinterpret_cast<int4*>(static_cast<char*>(p.poolV) + dst) = vv;
  }
}

// FP8 KV variant (reading R-22): code = E4M3(x / scale), the quotient rounded
// once in fp32 (IEEE division), then one round-to-nearest-even to E4M3 with
// saturation at +-448 (cvt.rn.satfinite); 16 elements per thread and tensor.
__device__ __forceinline__ uint32_t e4m3x4(float a, float b, float c, float d) {
  uint32_t lo, hi;
  asm("{\n\t.reg .b16 t;\n\tcvt.rn.satfinite.e4m3x2.f32 t, %2, %1;\n\tcvt.u32.u16 %0, t;\n\t}"
      : "=r"(lo) : "f"(a), "f"(b));
  asm("{\n\t.reg .b16 t;\n\tcvt.rn.satfinite.e4m3x2.f32 t, %2, %1;\n\tcvt.u32.u16 %0, t;\n\t}"
      : "=r"(hi) : "f"(c), "f"(d));
  return lo | (hi << 16);
}
__device__ __forceinline__ uint4 quant16(const uint4 a, const uint4 b, float s) {
  const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
  float f[16];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    f[2 * i] = __fdiv_rn(__uint_as_float(w[i] << 16), s);
    f[2 * i + 1] = __fdiv_rn(__uint_as_float(w[i] & 0xFFFF0000u), s);
  }
  return make_uint4(e4m3x4(f[0], f[1], f[2], f[3]), e4m3x4(f[4], f[5], f[6], f[7]),
                    e4m3x4(f[8], f[9], f[10], f[11]), e4m3x4(f[12], f[13], f[14], f[15]));
}
__global__ void __launch_bounds__(256) quant_e4m3_kernel(const QuantParams p) {
  const int64_t n16 = p.n / 16;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x) {
    const uint4* k = reinterpret_cast<const uint4*>(p.K) + 2 * i;
    const uint4* v = reinterpret_cast<const uint4*>(p.V) + 2 * i;
    reinterpret_cast<uint4*>(p.K8)[i] = quant16(k[0], k[1], p.k_scale);
    reinterpret_cast<uint4*>(p.V8)[i] = quant16(v[0], v[1], p.v_scale);
  }
}

__global__ void __launch_bounds__(256) gather_kernel(const GatherParams p) {
  const int chunks = p.D * p.elem_bytes / 16;
  const int64_t total = p.count * p.Hkv * chunks;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int c = idx % chunks;
    const int h = (idx / chunks) % p.Hkv;
    const int64_t tl = idx / ((int64_t)chunks * p.Hkv);
    const int64_t t = p.start + tl;
    const int64_t slot = (p.n_prefix_slots_pad >= 0 && t >= p.n_prefix) ? p.n_prefix_slots_pad + (t - p.n_prefix) : t;
    const int64_t page = p.pages[slot / p.P];
    const int64_t src = ((((int64_t)p.layer * p.num_pages + page) * p.Hkv + h) * p.P + slot % p.P) * (int64_t)p.D * p.elem_bytes + c * 16;
    const int64_t dst = (tl * p.Hkv + h) * (int64_t)p.D * p.elem_bytes + c * 16;
    *reinterpret_cast<int4*>(static_cast<char*>(p.K) + dst) = *reinterpret_cast<const int4*>(static_cast<const char*>(p.poolK) + src);
    *reinterpret_cast<int4*>(static_cast<char*>(p.V) + dst) = *reinterpret_cast<const int4*>(static_cast<const char*>(p.poolV) + src);
  }
}

template <typename T, int D>
cudaError_t launch_simt_t(const AttnParams& p, int n_layers, cudaStream_t s) {
  const size_t smem = sizeof(float) * (kRT * D + kBK * (D + 1) + kBK * D + kRT * kBK + 3 * kRT);
  cudaError_t e = set_smem_attr_once(reinterpret_cast<const void*>(attn_simt_kernel<T, D>), (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid(p.n_units, n_layers);
  attn_simt_kernel<T, D><<<grid, kThreads, smem, s>>>(p);
  return cudaGetLastError();
}

}  // namespace

int simt_rows_tile(int G, int D) { (void)G; (void)D; return kRT; }

cudaError_t launch_merge_ranks(const float* parts, int world, int64_t rows, int Hq, int D, void* O, bool bf16,
                               cudaStream_t s) {
  const int64_t warps = rows * Hq;
  if (warps == 0) return cudaSuccess;
  const int blocks = (int)((warps + 7) / 8);
  if (bf16)
    merge_ranks_kernel<__nv_bfloat16><<<blocks, 256, 0, s>>>(parts, world, rows, Hq, D, static_cast<__nv_bfloat16*>(O));
  else
    merge_ranks_kernel<float><<<blocks, 256, 0, s>>>(parts, world, rows, Hq, D, static_cast<float*>(O));
  return cudaGetLastError();
}

// Peer-memory exchange flags (A9): one warp; lane q releases `epoch` into slot
// `slot` of peer q's flag array (st.release.sys after a system-scope fence, so
// the stores this stream issued before -- the pushed chunk, or the merge's reads
// being done -- are ordered before the flag).
__global__ void signal_peers_kernel(const uint64_t* peer_flags, int n_peers, int slot, uint32_t epoch) {
  const int q = threadIdx.x;
  if (q >= n_peers) return;
  __threadfence_system();
  uint32_t* f = reinterpret_cast<uint32_t*>(peer_flags[q]) + slot;
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(f), "r"(epoch) : "memory");
}

// One block waits (acquire, system scope) until flags[i] >= epoch for i < n: the
// kernels after it on the stream run only once every peer has released.  A single
// spinning block never starves the peers' kernels of SMs (virtual ranks on one
// GPU); a peer that never signals fails the launch after 10 s instead of hanging.
__global__ void wait_flags_kernel(const uint32_t* flags, int n, uint32_t epoch) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    uint32_t v;
    uint64_t t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    do {
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flags + i) : "memory");
      if ((int32_t)(v - epoch) >= 0) break;
      __nanosleep(256);
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > 10000000000ull) __trap();
    } while (true);
  }
}

cudaError_t launch_signal_peers(const uint64_t* peer_flags, int n_peers, int slot, uint32_t epoch, cudaStream_t s) {
  signal_peers_kernel<<<1, 32 * ((n_peers + 31) / 32), 0, s>>>(peer_flags, n_peers, slot, epoch);
  return cudaGetLastError();
}

cudaError_t launch_wait_flags(const uint32_t* flags, int n, uint32_t epoch, cudaStream_t s) {
  wait_flags_kernel<<<1, 32, 0, s>>>(flags, n, epoch);
  return cudaGetLastError();
}
int simt_key_tile() { return kBK; }

cudaError_t launch_attn_simt(const AttnParams& p, int n_layers, bool bf16, cudaStream_t s) {
  if (p.n_units == 0 || n_layers == 0) return cudaSuccess;
  switch (p.D) {
#define SSA_CASE(DD)                                                                  \
  case DD:                                                                            \
    return bf16 ? launch_simt_t<__nv_bfloat16, DD>(p, n_layers, s) : launch_simt_t<float, DD>(p, n_layers, s);
    SSA_CASE(16)
    SSA_CASE(32)
    SSA_CASE(64)
    SSA_CASE(128)
#undef SSA_CASE
    default:
      return cudaErrorInvalidValue;
  }
}

cudaError_t launch_combine(const CombineParams& p, int n_layers, bool bf16, cudaStream_t s, int max_splits) {
  if (p.n_groups == 0 || n_layers == 0) return cudaSuccess;
  // rows per CTA: 32, or down to 8 when the launch would not fill the SMs (a single-layer
  // query: 8 groups x 4 row blocks = 32 CTAs at 32 rows, 128 at 8)
  CombineParams q = p;
  q.combine_rows = kCombineRows;
  while (q.combine_rows > 8 && (int64_t)p.n_groups * n_layers * ((p.rows_tile + q.combine_rows - 1) / q.combine_rows) < 2 * 148)
    q.combine_rows /= 2;
  dim3 grid(p.n_groups, n_layers, (p.rows_tile + q.combine_rows - 1) / q.combine_rows);
  const size_t smem = sizeof(float) * (size_t)max_splits * q.combine_rows;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(bf16 ? (const void*)combine_kernel<__nv_bfloat16> : (const void*)combine_kernel<float>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  if (bf16) combine_kernel<__nv_bfloat16><<<grid, 256, smem, s>>>(q);
  else combine_kernel<float><<<grid, 256, smem, s>>>(q);
  return cudaGetLastError();
}

cudaError_t launch_scatter(const ScatterParams& p, int n_layers, cudaStream_t s) {
  if (p.total_tokens == 0 || n_layers == 0) return cudaSuccess;
  const int64_t work = p.total_tokens * p.Hkv * (p.D * p.elem_bytes / 16);
  int blocks = (int)((work + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  dim3 grid(blocks, n_layers);
  scatter_kernel<<<grid, 256, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_quant_e4m3(const QuantParams& p, cudaStream_t s) {
  if (p.n == 0) return cudaSuccess;
  const int64_t work = p.n / 16;
  int blocks = (int)((work + 255) / 256);
  if (blocks > 148 * 8) blocks = 148 * 8;
  quant_e4m3_kernel<<<blocks, 256, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_gather(const GatherParams& p, cudaStream_t s) {
  if (p.count == 0) return cudaSuccess;
  const int64_t work = p.count * p.Hkv * (p.D * p.elem_bytes / 16);
  int blocks = (int)((work + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  gather_kernel<<<blocks, 256, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace ssa
