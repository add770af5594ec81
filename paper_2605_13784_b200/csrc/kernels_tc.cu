// kernels_tc.cu — tensor-core (tcgen05 / TMEM / TMA) attention for sm_100a.
//
// One CTA computes one work unit (plan.cpp): a q tile of 128 rows — 128/G tokens
// x the G query heads sharing one KV head (GQA packing, reading R-5) — against
// key tiles [tile_lo, tile_hi) of its segment: paged cached keys first (Eq.
// query-attention), then the segment's own keys with the causal mask
// (reading R-2).  Per key tile of 128 keys:
//     S = Q K^T            tcgen05.mma  M=128 N=128 K=128, S in TMEM (fp32)
//     P = exp2(S*c - m)    online softmax in registers, P -> smem (bf16)
//     O += P V             tcgen05.mma  M=128 N=128 K=128, O in TMEM (fp32)
// Warp roles (256 threads):
//     warp 0      TMA producer: Q once, then K/V tiles (paged: one box per page
//                 run; tail: dense input) into an NS-stage ring
//     warp 1      MMA issuer (one elected lane)
//     warp 2      TMEM allocator (512 columns: S0 | S1 | O)
//     warps 4-7   softmax + epilogue, one thread per row (TMEM lane)
// S is double-buffered in TMEM so QK^T of tile j+1 overlaps the softmax of tile
// j.  The running max is updated lazily (only when it grows by > 8 in log2
// units), so the O rescale (TMEM ld/st) is rare.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include <mutex>

#include "sm100.cuh"
#include "store.h"

namespace ssa {

namespace {

using namespace sm100;

constexpr int kM = 128;          // rows per q tile
constexpr int kBN = 128;         // keys per tile
constexpr int kD = 128;          // head dim (two 64-column swizzle chunks)
constexpr int kNS = 2;           // K/V pipeline stages
constexpr int kThreads = 256;
constexpr int kChunkBytes = kM * 128;                 // 128 rows x 128 B = 16 KB
constexpr int kTileBytes = 2 * kChunkBytes;           // 128 x 128 bf16 = 32 KB
constexpr float kRescaleThreshold = 8.0f;             // log2 units

struct TcSmem {
  uint8_t q[kTileBytes];
  uint8_t k[kNS][kTileBytes];
  uint8_t v[kNS][kTileBytes];
  uint8_t p[kTileBytes];
  uint64_t q_full;
  uint64_t k_full[kNS];
  uint64_t v_full[kNS];
  uint64_t kv_empty[kNS];
  uint64_t s_full[2];
  uint64_t p_full;
  uint64_t o_done;
  uint32_t tmem_base;
};

struct TcMaps {
  CUtensorMap q;       // [rows][Hq][D]   box {64, G, 128/G}
  CUtensorMap kt;      // [rows][Hkv][D]  box {64, 1, 128}
  CUtensorMap vt;
  CUtensorMap pk;      // [L*num_pages*Hkv*P][D] box {64, BR}
  CUtensorMap pv;
};

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}

__global__ void __launch_bounds__(kThreads, 1)
attn_tc_kernel(const AttnParams p, const __grid_constant__ TcMaps maps, const int box_rows) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  TcSmem& sm = *reinterpret_cast<TcSmem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int u = blockIdx.x, ly = blockIdx.y;
  const WorkUnit wu = p.units[u];
  const SegDesc sg = p.segs[wu.seg];
  const int G = p.G;
  const int64_t layer = p.layer0 + ly;
  const int64_t in_row0 = (p.in_layer_stride ? (int64_t)ly * p.rows_per_layer : 0) + sg.row0;
  const int n_pool_tiles = (sg.n_slots + kBN - 1) / kBN;
  const int nt = wu.tile_hi - wu.tile_lo;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&maps.q);
    tma_prefetch_desc(&maps.kt);
    tma_prefetch_desc(&maps.vt);
    tma_prefetch_desc(&maps.pk);
    tma_prefetch_desc(&maps.pv);
    mbar_init(&sm.q_full, 1);
    for (int s = 0; s < kNS; ++s) {
      mbar_init(&sm.k_full[s], 1);
      mbar_init(&sm.v_full[s], 1);
      mbar_init(&sm.kv_empty[s], 1);
    }
    mbar_init(&sm.s_full[0], 1);
    mbar_init(&sm.s_full[1], 1);
    mbar_init(&sm.p_full, 4);
    mbar_init(&sm.o_done, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(&sm.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;

  if (warp == 0) {
    // ------------------------------------------------------------- TMA producer
    if (elect_one()) {
      const int T = kM / G;
      mbar_arrive_expect_tx(&sm.q_full, kTileBytes);
      const int32_t qrow = (int32_t)(in_row0 + wu.q_tok0);
      for (int c = 0; c < 2; ++c)
        tma_load_3d(sm.q + c * kChunkBytes, &maps.q, &sm.q_full, c * 64, wu.kv_head * G, qrow);
      (void)T;
      const int64_t head_base = layer * p.num_pages;  // page row base = ((head_base + page)*Hkv + h)*P
      for (int j = 0; j < nt; ++j) {
        const int s = j % kNS;
        if (j >= kNS) mbar_wait(&sm.kv_empty[s], ((j / kNS) - 1) & 1);
        const int tile = wu.tile_lo + j;
        mbar_arrive_expect_tx(&sm.k_full[s], kTileBytes);
        if (tile < n_pool_tiles) {
          const int key0 = tile * kBN;
          for (int b = 0; b < kBN / box_rows; ++b) {
            const int slot = key0 + b * box_rows;
            int32_t row;
            if (slot < sg.n_slots) {
              const int64_t page = __ldg(sg.pages + slot / p.P);
              row = (int32_t)(((head_base + page) * p.Hkv + wu.kv_head) * p.P + (slot % p.P));
            } else {
              row = 0x7FFFFFF0;  // fully out of bounds -> TMA zero fill
            }
            for (int c = 0; c < 2; ++c)
              tma_load_2d(sm.k[s] + c * kChunkBytes + b * box_rows * 128, &maps.pk, &sm.k_full[s], c * 64, row);
          }
          mbar_arrive_expect_tx(&sm.v_full[s], kTileBytes);
          for (int b = 0; b < kBN / box_rows; ++b) {
            const int slot = key0 + b * box_rows;
            int32_t row;
            if (slot < sg.n_slots) {
              const int64_t page = __ldg(sg.pages + slot / p.P);
              row = (int32_t)(((head_base + page) * p.Hkv + wu.kv_head) * p.P + (slot % p.P));
            } else {
              row = 0x7FFFFFF0;
            }
            for (int c = 0; c < 2; ++c)
              tma_load_2d(sm.v[s] + c * kChunkBytes + b * box_rows * 128, &maps.pv, &sm.v_full[s], c * 64, row);
          }
        } else {
          const int32_t krow = (int32_t)(in_row0 + (tile - n_pool_tiles) * kBN);
          for (int c = 0; c < 2; ++c)
            tma_load_3d(sm.k[s] + c * kChunkBytes, &maps.kt, &sm.k_full[s], c * 64, wu.kv_head, krow);
          mbar_arrive_expect_tx(&sm.v_full[s], kTileBytes);
          for (int c = 0; c < 2; ++c)
            tma_load_3d(sm.v[s] + c * kChunkBytes, &maps.vt, &sm.v_full[s], c * 64, wu.kv_head, krow);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------- MMA issuer
    constexpr uint32_t idesc_s = idesc_bf16(kM, kBN, 0, 0);   // Q K-major, K K-major
    constexpr uint32_t idesc_o = idesc_bf16(kM, kD, 0, 1);    // P K-major, V MN-major
    const uint32_t q_addr = smem_u32(sm.q);
    const uint32_t p_addr = smem_u32(sm.p);
    const bool leader = elect_one();
    if (leader) mbar_wait(&sm.q_full, 0);
    tc_fence_after();
    auto issue_pv = [&](int i) {
      const int s = i % kNS;
      if (leader) {
        mbar_wait(&sm.v_full[s], (i / kNS) & 1);
        mbar_wait(&sm.p_full, i & 1);
        tc_fence_after();
        const uint32_t v_addr = smem_u32(sm.v[s]);
#pragma unroll
        for (int kk = 0; kk < kBN / 16; ++kk) {
          // A = P[128 rows][16 keys]: key chunk kk/4, 32-byte step inside the swizzle atom
          const uint64_t a = sdesc_sw128(p_addr + (kk >> 2) * kChunkBytes + (kk & 3) * 32, 16, 1024);
          // B = V[16 keys][128 d] MN-major: 16 keys = 2048 B into each 64-column chunk
          const uint64_t b = sdesc_sw128(v_addr + kk * 2048, kChunkBytes, 1024);
          mma_bf16_ss(tmem + 256, a, b, idesc_o, (i > 0 || kk > 0) ? 1u : 0u);
        }
        mma_commit(&sm.kv_empty[s]);
        mma_commit(&sm.o_done);
      }
      __syncwarp();
    };
    for (int j = 0; j < nt; ++j) {
      const int s = j % kNS;
      if (leader) {
        mbar_wait(&sm.k_full[s], (j / kNS) & 1);
        tc_fence_after();
        const uint32_t k_addr = smem_u32(sm.k[s]);
        const uint32_t d_tmem = tmem + (uint32_t)(j & 1) * 128;
#pragma unroll
        for (int kk = 0; kk < kD / 16; ++kk) {
          const uint32_t off = (kk >> 2) * kChunkBytes + (kk & 3) * 32;
          const uint64_t a = sdesc_sw128(q_addr + off, 16, 1024);
          const uint64_t b = sdesc_sw128(k_addr + off, 16, 1024);
          mma_bf16_ss(d_tmem, a, b, idesc_s, kk > 0 ? 1u : 0u);
        }
        mma_commit(&sm.s_full[j & 1]);
      }
      __syncwarp();
      if (j >= 1) issue_pv(j - 1);
    }
    if (nt > 0) issue_pv(nt - 1);
  } else if (warp >= 4) {
    // ------------------------------------------------------------- softmax + epilogue
    const int r = threadIdx.x - 128;               // row == TMEM lane
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    const float c = p.scale_log2;
    const int tok = wu.q_tok0 + r / G;             // token of this row within the segment
    float m_run = -CUDART_INF_F;                   // running max of raw scores
    float l_run = 0.f;
    uint8_t* prow = sm.p + r * 128;
    const int sw = r & 7;
    for (int j = 0; j < nt; ++j) {
      const int tile = wu.tile_lo + j;
      const bool is_pool = tile < n_pool_tiles;
      const int key0 = (is_pool ? tile : tile - n_pool_tiles) * kBN;
      mbar_wait(&sm.s_full[j & 1], (j >> 1) & 1);
      tc_fence_after();
      float sv[kBN];
#pragma unroll
      for (int q4 = 0; q4 < 4; ++q4) {
        uint32_t regs[32];
        tmem_ld32(tmem + lane_base + (uint32_t)(j & 1) * 128 + q4 * 32, regs);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 32; ++i) sv[q4 * 32 + i] = __uint_as_float(regs[i]);
      }
      // masking: pool tiles past n_slots / inside the R0 pad hole; tail tiles causal
      int lim_lo = 0, lim_hi = kBN;        // valid key range [lim_lo, lim_hi) relative to key0
      int hole_lo = 0, hole_hi = 0;
      if (is_pool) {
        lim_hi = min(kBN, sg.n_slots - key0);
        hole_lo = max(0, sg.hole_lo - key0);
        hole_hi = max(0, min(kBN, sg.hole_hi - key0));
      } else {
        const int last = p.fault == 2 ? tok - 1 : tok;   // row sees own keys 0..tok
        lim_hi = max(0, min(kBN, min(sg.m, last + 1) - key0));
      }
      float mt = -CUDART_INF_F;
#pragma unroll
      for (int i = 0; i < kBN; ++i) {
        const bool ok = i >= lim_lo && i < lim_hi && !(i >= hole_lo && i < hole_hi);
        sv[i] = ok ? sv[i] : -CUDART_INF_F;
        mt = fmaxf(mt, sv[i]);
      }
      const float m_new = fmaxf(m_run, mt);
      const bool rescale = m_new > m_run + kRescaleThreshold / c || (m_run == -CUDART_INF_F);
      float alpha = 1.f;
      if (rescale) {
        alpha = (m_run == -CUDART_INF_F) ? 0.f : exp2f((m_run - m_new) * c);
        m_run = m_new;
      }
      const float mc = (m_run == -CUDART_INF_F) ? 0.f : m_run * c;
      float sum = 0.f;
#pragma unroll
      for (int i = 0; i < kBN; ++i) {
        sv[i] = exp2f(fmaf(sv[i], c, -mc));
        sum += sv[i];
      }
      // P buffer and O are free once PV(j-1) completed
      if (j >= 1) {
        mbar_wait(&sm.o_done, (j - 1) & 1);
        tc_fence_after();
        if (__any_sync(0xffffffffu, rescale && alpha != 1.f)) {
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            uint32_t regs[32];
            const uint32_t a = tmem + lane_base + 256 + q4 * 32;
            tmem_ld32(a, regs);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) regs[i] = __float_as_uint(__uint_as_float(regs[i]) * alpha);
            tmem_st32(a, regs);
          }
          tmem_wait_st();
        }
      }
      l_run = l_run * alpha + sum;
      // P row -> smem, bf16, 128B-swizzled K-major (two 64-key chunks)
#pragma unroll
      for (int g = 0; g < 16; ++g) {
        const int chunk = g >> 3, gi = g & 7;
        uint4 v;
        v.x = pack_bf16(sv[g * 8 + 0], sv[g * 8 + 1]);
        v.y = pack_bf16(sv[g * 8 + 2], sv[g * 8 + 3]);
        v.z = pack_bf16(sv[g * 8 + 4], sv[g * 8 + 5]);
        v.w = pack_bf16(sv[g * 8 + 6], sv[g * 8 + 7]);
        *reinterpret_cast<uint4*>(prow + chunk * kChunkBytes + ((gi ^ sw) << 4)) = v;
      }
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.p_full);
    }
    // ------------------------------------------------------------- epilogue
    const int rows = wu.q_ntok * G;
    if (nt > 0) {
      mbar_wait(&sm.o_done, (nt - 1) & 1);
      tc_fence_after();
    }
    const float inv_l = l_run > 0.f ? 1.f / l_run : 0.f;
    const int h = wu.kv_head * G + r % G;
    const int64_t orow = in_row0 + tok;
#pragma unroll
    for (int q4 = 0; q4 < 4; ++q4) {
      uint32_t regs[32];
      tmem_ld32(tmem + lane_base + 256 + q4 * 32, regs);
      tmem_wait_ld();
      if (r < rows) {
        if (wu.group < 0) {
          __nv_bfloat16* out = static_cast<__nv_bfloat16*>(p.O) + (orow * p.Hq + h) * kD + q4 * 32;
#pragma unroll
          for (int i = 0; i < 32; i += 8) {
            uint4 v;
            v.x = pack_bf16(__uint_as_float(regs[i + 0]) * inv_l, __uint_as_float(regs[i + 1]) * inv_l);
            v.y = pack_bf16(__uint_as_float(regs[i + 2]) * inv_l, __uint_as_float(regs[i + 3]) * inv_l);
            v.z = pack_bf16(__uint_as_float(regs[i + 4]) * inv_l, __uint_as_float(regs[i + 5]) * inv_l);
            v.w = pack_bf16(__uint_as_float(regs[i + 6]) * inv_l, __uint_as_float(regs[i + 7]) * inv_l);
            *reinterpret_cast<uint4*>(out + i) = v;
          }
        } else {
          const int64_t slot = (int64_t)ly * p.n_units + u;
          float* out = p.part_o + (slot * kM + r) * kD + q4 * 32;
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            float4 v = make_float4(__uint_as_float(regs[i]) * inv_l, __uint_as_float(regs[i + 1]) * inv_l,
                                   __uint_as_float(regs[i + 2]) * inv_l, __uint_as_float(regs[i + 3]) * inv_l);
            *reinterpret_cast<float4*>(out + i) = v;
          }
        }
      }
    }
    if (wu.group >= 0 && r < rows) {
      const int64_t slot = (int64_t)ly * p.n_units + u;
      p.part_lse[slot * kM + r] = l_run > 0.f ? m_run * c + log2f(l_run) : -CUDART_INF_F;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<512>(tmem);
}

// ------------------------------------------------------------------ host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(f);
  });
  return fn;
}

bool encode(CUtensorMap* m, const void* base, int rank, const cuuint64_t* dims, const cuuint64_t* strides_bytes,
            const cuuint32_t* box) {
  EncodeTiledFn fn = get_encode();
  if (!fn) return false;
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(base), dims, strides_bytes, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace

int tc_key_tile() { return kBN; }
int tc_rows_tile() { return kM; }
bool tc_supported_shape(int D, int G, bool bf16) {
  return bf16 && D == kD && G >= 1 && G <= 16 && (kM % G) == 0 && get_encode() != nullptr;
}

cudaError_t launch_attn_tc(const AttnParams& p, int n_layers, int q_tiles_opt, cudaStream_t s) {
  (void)q_tiles_opt;
  if (p.n_units == 0 || n_layers == 0) return cudaSuccess;
  if (!tc_supported_shape(p.D, p.G, true)) return cudaErrorNotSupported;
  TcMaps maps;
  const int G = p.G;
  const cuuint64_t rows = (cuuint64_t)p.rows_per_layer * (p.in_layer_stride ? n_layers : 1);
  {
    cuuint64_t dims[3] = {(cuuint64_t)kD, (cuuint64_t)p.Hq, rows};
    cuuint64_t str[2] = {(cuuint64_t)kD * 2, (cuuint64_t)p.Hq * kD * 2};
    cuuint32_t box[3] = {64, (cuuint32_t)G, (cuuint32_t)(kM / G)};
    if (!encode(&maps.q, p.Q, 3, dims, str, box)) return cudaErrorInvalidValue;
  }
  {
    cuuint64_t dims[3] = {(cuuint64_t)kD, (cuuint64_t)p.Hkv, rows};
    cuuint64_t str[2] = {(cuuint64_t)kD * 2, (cuuint64_t)p.Hkv * kD * 2};
    cuuint32_t box[3] = {64, 1, (cuuint32_t)kBN};
    if (!encode(&maps.kt, p.Kt, 3, dims, str, box)) return cudaErrorInvalidValue;
    if (!encode(&maps.vt, p.Vt, 3, dims, str, box)) return cudaErrorInvalidValue;
  }
  const int box_rows = p.P < kBN ? p.P : kBN;
  {
    // pool rows: all layers (the map is re-encoded per launch; cheap host call)
    const cuuint64_t prow = (cuuint64_t)(p.layer0 + n_layers) * p.num_pages * p.Hkv * p.P;
    cuuint64_t dims[2] = {(cuuint64_t)kD, prow};
    cuuint64_t str[1] = {(cuuint64_t)kD * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
    if (!encode(&maps.pk, p.poolK, 2, dims, str, box)) return cudaErrorInvalidValue;
    if (!encode(&maps.pv, p.poolV, 2, dims, str, box)) return cudaErrorInvalidValue;
  }
  const size_t smem = sizeof(TcSmem) + 1024;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(attn_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  dim3 grid(p.n_units, n_layers);
  attn_tc_kernel<<<grid, kThreads, smem, s>>>(p, maps, box_rows);
  return cudaGetLastError();
}

}  // namespace ssa
