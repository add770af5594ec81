// kernels_qkv.cu — fused data-plane projection before attention (SURVEY §8(f)
// NEXT-2): the `Forward` of Alg. 1 L282 up to the attention inputs,
//     [Q | K | V] = X W_qkv^T          (tcgen05 GEMM, bf16 in, fp32 accumulate)
//     Q, K <- RoPE(Q, K; pos)          (rotate-half convention, reading R-19)
//     K, V -> the append's page slots  (replaces the KA scatter, A2)
// in one launch.  X is [m][hidden] (token rows), W_qkv is the nn.Linear weight
// [(Hq + 2 Hkv) D][hidden] (rows: Q heads, then K heads, then V heads).
//
// Tiling.  A CTA owns a 128-token x 256-output-column tile (two heads of
// D = 128), accumulating fp32 in 256 TMEM columns; both operands are K-major,
// staged by TMA in 128-byte-swizzled 64-element k-blocks (4 stages x 48 KB).
// Short token counts (the 32-token query, a 256-token append) leave too few
// tiles for 148 SMs, so the k range is split over a thread-block cluster of S
// CTAs (split-K).  Each CTA dumps its fp32 partial tile from TMEM into its own
// shared memory; after a cluster barrier CTA r reduces token rows
// [r*128/S, (r+1)*128/S) by reading all S partials through distributed shared
// memory (fixed order, deterministic), applies RoPE in fp32, rounds once to
// bf16 and stores Q / K / V rows (256 contiguous bytes per head) to the dense
// outputs and/or straight into the KV pool pages.
// Warp roles (256 threads): warp 0 TMA producer, warp 1 MMA issuer, warp 2
// TMEM allocator; all 8 warps run the epilogue.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "sm100.cuh"
#include "store.h"

namespace ssa {

namespace {

using namespace sm100;

constexpr int kBM = 128;                       // token rows per tile (TMEM lanes)
constexpr int kBN = 256;                       // output columns per tile (2 heads)
constexpr int kBK = 64;                        // k elements per stage (one 128-B swizzle row)
constexpr int kHeadD = 128;
constexpr int kStages = 4;
constexpr int kABytes = kBM * kBK * 2;         // 16 KB
constexpr int kBBytes = kBN * kBK * 2;         // 32 KB
constexpr int kStageBytes = kABytes + kBBytes;
constexpr int kPitch = kBN + 4;                // fp32 dump row pitch (floats): conflict-free float4 rows
constexpr int kThreads = 256;
constexpr int kMaxSplits = 8;                  // portable cluster size
static_assert(kBM * kPitch * 4 <= kStages * kStageBytes, "fp32 dump must fit in the stage buffers");

struct QkvBars {
  uint64_t full[kStages];
  uint64_t empty[kStages];
  uint64_t acc;
  uint32_t tmem_base;
};

struct QkvMaps {
  CUtensorMap x;   // [m][hidden]      box {64, 128}
  CUtensorMap w;   // [Nout][hidden]   box {64, 256}
};

__device__ __forceinline__ float4 ld_cluster_f4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr)
               : "memory");
  return v;
}

__device__ __forceinline__ uint2 pack4_bf16(float a, float b, float c, float d) {
  __nv_bfloat162 lo = __floats2bfloat162_rn(a, b);
  __nv_bfloat162 hi = __floats2bfloat162_rn(c, d);
  return make_uint2(*reinterpret_cast<uint32_t*>(&lo), *reinterpret_cast<uint32_t*>(&hi));
}

__global__ void __launch_bounds__(kThreads, 1)
qkv_rope_kernel(const QkvParams p, const __grid_constant__ QkvMaps maps) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* tiles = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  QkvBars& bar = *reinterpret_cast<QkvBars*>(tiles + kStages * kStageBytes);
  float* dump = reinterpret_cast<float*>(tiles);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int S = p.splits;
  const int rank = (int)cluster_ctarank();   // == blockIdx.x % S (cluster spans x)
  const int tn = blockIdx.x / S;
  const int tm = blockIdx.y;
  const int nkb = p.hidden / kBK;
  const int kb_lo = rank * nkb / S;
  const int kb_hi = (rank + 1) * nkb / S;
  const int n_kb = kb_hi - kb_lo;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&maps.x);
    tma_prefetch_desc(&maps.w);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&bar.full[s], 1);
      mbar_init(&bar.empty[s], 1);
    }
    mbar_init(&bar.acc, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<256>(&bar.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bar.tmem_base;

  if (warp == 0) {
    // ------------------------------------------------------------- TMA producer
    if (elect_one()) {
      for (int i = 0; i < n_kb; ++i) {
        const int s = i % kStages;
        if (i >= kStages) mbar_wait(&bar.empty[s], ((i / kStages) - 1) & 1);
        uint8_t* a = tiles + s * kStageBytes;
        mbar_arrive_expect_tx(&bar.full[s], kStageBytes);
        const int k0 = (kb_lo + i) * kBK;
        tma_load_2d(a, &maps.x, &bar.full[s], k0, tm * kBM);
        tma_load_2d(a + kABytes, &maps.w, &bar.full[s], k0, tn * kBN);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------- MMA issuer
    if (elect_one()) {
      constexpr uint32_t idesc = idesc_bf16(kBM, kBN, 0, 0);   // X, W both K-major
      const uint64_t ad0 = sdesc_sw128(smem_u32(tiles), 16, 1024);
      const uint64_t bd0 = sdesc_sw128(smem_u32(tiles + kABytes), 16, 1024);
      for (int i = 0; i < n_kb; ++i) {
        const int s = i % kStages;
        mbar_wait(&bar.full[s], (i / kStages) & 1);
        tc_fence_after();
        const uint64_t st = (uint64_t)((s * kStageBytes) >> 4);
#pragma unroll
        for (int kk = 0; kk < kBK / 16; ++kk)   // 16 k-elements = 32 B along the swizzled row
          mma_bf16_ss(tmem, ad0 + st + (uint64_t)(kk * 2), bd0 + st + (uint64_t)(kk * 2), idesc,
                      (i > 0 || kk > 0) ? 1u : 0u);
        mma_commit(&bar.empty[s]);
      }
      mma_commit(&bar.acc);
    }
  }
  __syncwarp();

  // --------------------------------------------------------------- TMEM -> smem
  // warp w reads TMEM lanes 32*(w%4).. (token rows) and columns 128*(w/4)..
  mbar_wait(&bar.acc, 0);
  tc_fence_after();
  {
    const int q = warp & 3;
    const int ch = warp >> 2;
    const int r = q * 32 + lane;
    float* row = dump + (size_t)r * kPitch + ch * 128;
#pragma unroll 1
    for (int c = 0; c < 4; ++c) {
      uint32_t v[32];
      tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(ch * 128 + c * 32), v);
      tmem_wait_ld();
      reg_fence32(v);
#pragma unroll
      for (int e = 0; e < 32; e += 4)
        *reinterpret_cast<float4*>(row + c * 32 + e) =
            make_float4(__uint_as_float(v[e]), __uint_as_float(v[e + 1]), __uint_as_float(v[e + 2]),
                        __uint_as_float(v[e + 3]));
    }
  }
  tc_fence_before();
  cluster_sync_all();   // every partial of the cluster is in shared memory

  // --------------------------------------------------------------- reduce + RoPE + store
  {
    const int r_lo = rank * kBM / S;
    const int r_hi = (rank + 1) * kBM / S;
    const int half = lane >> 4;           // 0: dims [0, 64), 1: dims [64, 128)
    const int j0 = 4 * (lane & 15);       // rotary frequency index of this lane's first dim
    const int dcol = 4 * lane;            // this lane's 4 dims within a head
    const int n_heads = p.Hq + 2 * p.Hkv;
    const bool rope = p.rope_theta > 0.0;
    // inv_freq_j = theta^(-2j/D) in double (R-19); angles are reduced mod 2 pi
    // in double so fp32 sincos sees |a| <= pi at any position.
    double inv_freq[4];
#pragma unroll
    for (int c = 0; c < 4; ++c)
      inv_freq[c] = rope ? exp2(-(2.0 * (j0 + c) / kHeadD) * log2(p.rope_theta)) : 0.0;
    const uint32_t own = smem_u32(dump);
#pragma unroll 1
    for (int r = r_lo + warp; r < r_hi; r += kThreads / 32) {
      const int t = tm * kBM + r;
      if (t >= p.m) break;
      float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a;
      const uint32_t off = (uint32_t)((r * kPitch + dcol) * 4);
      for (int s = 0; s < S; ++s) {
        const uint32_t src = mapa_shared(own + off, (uint32_t)s);
        const float4 x = ld_cluster_f4(src);
        const float4 y = ld_cluster_f4(src + 128 * 4);
        a.x += x.x; a.y += x.y; a.z += x.z; a.w += x.w;
        b.x += y.x; b.y += y.y; b.z += y.z; b.w += y.w;
      }
      float cs[4], sn[4];
      if (rope) {
        const double pos = (double)(p.pos0 + t);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const double ang = pos * inv_freq[c];
          const double k = rint(ang * 0.15915494309189535);   // 1 / (2 pi)
          double red = fma(-k, 6.283185307179586, ang);
          red = fma(-k, 2.4492935982947064e-16, red);          // 2 pi - double(2 pi)
          sincosf((float)red, &sn[c], &cs[c]);
        }
      }
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const int gh = tn * 2 + hh;
        if (gh >= n_heads) break;
        float4 v = hh ? b : a;
        const bool is_v = gh >= p.Hq + p.Hkv;
        if (rope && !is_v) {
          // partner dims d +/- 64 live in lane ^ 16 (rotate-half pairs)
          float4 u;
          u.x = __shfl_xor_sync(0xffffffffu, v.x, 16);
          u.y = __shfl_xor_sync(0xffffffffu, v.y, 16);
          u.z = __shfl_xor_sync(0xffffffffu, v.z, 16);
          u.w = __shfl_xor_sync(0xffffffffu, v.w, 16);
          const float sg = half ? 1.f : -1.f;   // x' = x cos -/+ x_partner sin
          v.x = fmaf(sg * u.x, sn[0], v.x * cs[0]);
          v.y = fmaf(sg * u.y, sn[1], v.y * cs[1]);
          v.z = fmaf(sg * u.z, sn[2], v.z * cs[2]);
          v.w = fmaf(sg * u.w, sn[3], v.w * cs[3]);
        }
        const uint2 packed = pack4_bf16(v.x, v.y, v.z, v.w);
        if (gh < p.Hq) {
          *reinterpret_cast<uint2*>(static_cast<uint8_t*>(p.Q) + (((int64_t)t * p.Hq + gh) * kHeadD + dcol) * 2) =
              packed;
        } else {
          const int kh = is_v ? gh - p.Hq - p.Hkv : gh - p.Hq;
          void* dense = is_v ? p.V : p.K;
          if (dense)
            *reinterpret_cast<uint2*>(static_cast<uint8_t*>(dense) + (((int64_t)t * p.Hkv + kh) * kHeadD + dcol) * 2) =
                packed;
          void* pool = is_v ? p.poolV : p.poolK;
          if (pool) {
            const int64_t slot = (int64_t)p.slot0 + t;
            const int64_t page = __ldg(p.pages + slot / p.P);
            const int64_t prow = ((p.page_base + page) * p.Hkv + kh) * p.P + slot % p.P;
            *reinterpret_cast<uint2*>(static_cast<uint8_t*>(pool) + (prow * kHeadD + dcol) * 2) = packed;
          }
        }
      }
    }
  }
  tc_fence_before();
  cluster_sync_all();   // peers may still be reading this CTA's partial
  if (warp == 2) tmem_dealloc<256>(tmem);
}

}  // namespace

bool qkv_supported(int D, int hidden) { return D == kHeadD && hidden > 0 && hidden % kBK == 0; }

int qkv_choose_splits(int m, int n_heads, int hidden, int num_sms) {
  const int tiles = ((n_heads * kHeadD + kBN - 1) / kBN) * ((m + kBM - 1) / kBM);
  int s = num_sms / (tiles > 0 ? tiles : 1);
  s = s < 1 ? 1 : (s > kMaxSplits ? kMaxSplits : s);
  const int nkb = hidden / kBK;
  return s > nkb ? nkb : s;
}

cudaError_t launch_qkv_rope(const QkvParams& p, cudaStream_t s) {
  if (p.m <= 0) return cudaSuccess;
  if (!qkv_supported(p.D, p.hidden) || p.splits < 1 || p.splits > kMaxSplits || p.splits > p.hidden / kBK)
    return cudaErrorNotSupported;
  const int n_heads = p.Hq + 2 * p.Hkv;
  QkvMaps maps;
  {
    cuuint64_t dims[2] = {(cuuint64_t)p.hidden, (cuuint64_t)p.m};
    cuuint64_t str[1] = {(cuuint64_t)p.hidden * 2};
    cuuint32_t box[2] = {kBK, kBM};
    if (!encode_bf16_map(&maps.x, p.X, 2, dims, str, box)) return cudaErrorInvalidValue;
  }
  {
    cuuint64_t dims[2] = {(cuuint64_t)p.hidden, (cuuint64_t)n_heads * kHeadD};
    cuuint64_t str[1] = {(cuuint64_t)p.hidden * 2};
    cuuint32_t box[2] = {kBK, kBN};
    if (!encode_bf16_map(&maps.w, p.W, 2, dims, str, box)) return cudaErrorInvalidValue;
  }
  const size_t smem = (size_t)kStages * kStageBytes + sizeof(QkvBars) + 1024;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(qkv_rope_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(qkv_rope_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 0);
    (void)e;
    configured = true;
  }
  const int n_tiles_n = (n_heads * kHeadD + kBN - 1) / kBN;
  const int n_tiles_m = (p.m + kBM - 1) / kBM;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(n_tiles_n * p.splits, n_tiles_m, 1);
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = p.splits;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, qkv_rope_kernel, p, maps);
}

}  // namespace ssa
