// kernels_qkv.cu — fused data-plane projection before attention (SURVEY §8(f)
// NEXT-2): the `Forward` of Alg. 1 L282 up to the attention inputs,
//     [Q | K | V] = X W_qkv^T          (tcgen05 GEMM, bf16 in, fp32 accumulate)
//     Q, K <- RoPE(Q, K; pos)          (rotate-half convention, reading R-21)
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
#include <stdlib.h>

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
constexpr int kRowBytes = kBN * 4;             // one fp32 partial row (swizzled, no padding)
constexpr int kThreads = 256;
constexpr int kMaxSplits = 8;                  // portable cluster size
constexpr int kTableRows = 64;                 // RoPE (cos, sin) table rows (used when S >= 2)
constexpr int kTableBytes = kTableRows * 64 * 8;
constexpr int kExchangeRows = kStages * kStageBytes / kRowBytes;   // part + recv rows that fit (192)

struct QkvBars {
  uint64_t full[kStages];
  uint64_t empty[kStages];
  uint64_t acc;
  uint64_t recv;   // peers' partial rows landed (bulk-copy complete_tx)
  uint32_t tmem_base;
};

struct QkvMaps {
  CUtensorMap x;   // [m][hidden]      box {64, 128}
  CUtensorMap w;   // [Nout][hidden]   box {64, 256}
};

// Four bf16 values (packed pairs) -> four E4M3 codes of value / scale: the quotient
// rounded once in fp32, then cvt.rn.satfinite (reading R-22; the same arithmetic as
// quant_e4m3_kernel, so pages written here equal pages the scatter writes).
__device__ __forceinline__ uint32_t e4m3x4_of_bf16(uint2 v, float scale) {
  const float a = __fdiv_rn(__uint_as_float(v.x << 16), scale);
  const float b = __fdiv_rn(__uint_as_float(v.x & 0xFFFF0000u), scale);
  const float c = __fdiv_rn(__uint_as_float(v.y << 16), scale);
  const float d = __fdiv_rn(__uint_as_float(v.y & 0xFFFF0000u), scale);
  uint32_t lo, hi;
  asm("{\n\t.reg .b16 t;\n\tcvt.rn.satfinite.e4m3x2.f32 t, %2, %1;\n\tcvt.u32.u16 %0, t;\n\t}"
      : "=r"(lo) : "f"(a), "f"(b));
  asm("{\n\t.reg .b16 t;\n\tcvt.rn.satfinite.e4m3x2.f32 t, %2, %1;\n\tcvt.u32.u16 %0, t;\n\t}"
      : "=r"(hi) : "f"(c), "f"(d));
  return lo | (hi << 16);
}

__device__ __forceinline__ float4 ld_cluster_f4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr)
               : "memory");
  return v;
}

// cos / sin of pos * inv_freq, inv_freq = theta^(-2j/D) (R-21): the angle is formed and reduced mod
// 2 pi in double, so the fp32 sincos sees |a| <= pi at any position.
__device__ __forceinline__ void rope_cs(int64_t pos, double inv_freq, float* c, float* s) {
  const double ang = (double)pos * inv_freq;
  const double k = rint(ang * 0.15915494309189535);   // 1 / (2 pi)
  double red = fma(-k, 6.283185307179586, ang);
  red = fma(-k, 2.4492935982947064e-16, red);          // 2 pi - double(2 pi)
  sincosf((float)red, s, c);
}

__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define QKV_TRACE(i) do { if (p.trace && threadIdx.x == 0) p.trace[(blockIdx.y * gridDim.x + blockIdx.x) * 10 + (i)] = gtimer(); } while (0)
#define QKV_TRACE_T(i) do { if (p.trace) p.trace[(blockIdx.y * gridDim.x + blockIdx.x) * 10 + (i)] = gtimer(); } while (0)

// shared::cta -> shared::cluster bulk copy (TMA engine), completing bytes on
// the destination CTA's mbarrier.
__device__ __forceinline__ void bulk_copy_s2cluster(uint32_t dst, uint32_t src, uint32_t bytes, uint32_t mbar) {
  asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "r"(src), "r"(bytes), "r"(mbar)
               : "memory");
}
__device__ __forceinline__ void bulk_commit_group() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_group_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

__device__ __forceinline__ void st_cluster_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared::cluster.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d)
               : "memory");
}

// Shared-memory accesses by 32-bit shared address: the tile pointers are derived from the
// dynamic smem base by integer arithmetic, so plain dereferences compile to generic
// LD.E / ST.E (longer latency than LDS / STS).
__device__ __forceinline__ float4 lds_f4(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts_u4(uint32_t a, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(x), "r"(y), "r"(z), "r"(w) : "memory");
}
__device__ __forceinline__ void sts_f2(uint32_t a, float x, float y) {
  asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(a), "f"(x), "f"(y) : "memory");
}

__device__ __forceinline__ uint2 pack4_bf16(float a, float b, float c, float d) {
  __nv_bfloat162 lo = __floats2bfloat162_rn(a, b);
  __nv_bfloat162 hi = __floats2bfloat162_rn(c, d);
  return make_uint2(*reinterpret_cast<uint32_t*>(&lo), *reinterpret_cast<uint32_t*>(&hi));
}

__global__ void __launch_bounds__(kThreads, 1)
qkv_rope_kernel(const QkvParams p, const __grid_constant__ QkvMaps maps) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  QKV_TRACE(0);
  griddep_launch_dependents();   // the next grid's prologue may overlap this grid's tail
  uint8_t* tiles = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* table = reinterpret_cast<float*>(tiles + kStages * kStageBytes);   // [rows][64] (cos, sin)
  double* inv_freq = reinterpret_cast<double*>(tiles + kStages * kStageBytes + kTableBytes);   // [64]
  QkvBars& bar = *reinterpret_cast<QkvBars*>(tiles + kStages * kStageBytes + kTableBytes + 64 * 8);
  // after the mainloop: part = this CTA's partial rows [valid][256] (swizzled,
  // rows grouped by owner), recv = the peers' partials of this CTA's own rows
  // [S-1][rows_max][256]
  float* part = reinterpret_cast<float*>(tiles);

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
  // token rows of this tile split evenly over the cluster (only the valid ones)
  const int valid = min(kBM, p.m - tm * kBM);
  auto row_lo = [&](int o) { return o * valid / S; };
  const int rows_max = (valid + S - 1) / S;
  const int own_lo = row_lo(rank);
  const int own_rows = row_lo(rank + 1) - own_lo;
  float* recv = part + (size_t)valid * 256;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&maps.x);
    tma_prefetch_desc(&maps.w);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&bar.full[s], 1);
      mbar_init(&bar.empty[s], 1);
    }
    mbar_init(&bar.acc, 1);
    mbar_init(&bar.recv, 1);
    fence_mbar_init();
    // bytes this CTA will receive: its own rows from each of the S-1 peers
    mbar_arrive_expect_tx(&bar.recv, (uint32_t)((S - 1) * own_rows * kRowBytes));
  }
  if (warp == 2) tmem_alloc<256>(&bar.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bar.tmem_base;
  QKV_TRACE(1);

  if (warp == 0) {
    // ------------------------------------------------------------- TMA producer
    // W is a weight no kernel of the stream writes: under programmatic dependent launch
    // its first kStages stages are requested before griddepcontrol.wait, so the weight
    // stream starts while the previous grid drains; X (the previous layer's output)
    // only after it.
    if (elect_one()) {
      auto load_w = [&](int i) {
        const int s = i % kStages;
        uint8_t* a = tiles + s * kStageBytes;
        mbar_arrive_expect_tx(&bar.full[s], kStageBytes);
        if (p.debug >= 2)   // experiments: contiguous 32 KB W blocks (wrong values, same bytes)
          tma_load_2d(a + kABytes, &maps.w, &bar.full[s], 0, (tn * nkb + kb_lo + i) * kBN);
        else
          tma_load_2d(a + kABytes, &maps.w, &bar.full[s], (kb_lo + i) * kBK, tn * kBN);
      };
      const int n_early = p.debug == 5 ? 0 : min(n_kb, kStages);
      for (int i = 0; i < n_early; ++i) load_w(i);
      griddep_wait();
      for (int i = 0; i < n_kb; ++i) {
        const int s = i % kStages;
        if (i >= kStages) mbar_wait(&bar.empty[s], ((i / kStages) - 1) & 1);
        uint8_t* a = tiles + s * kStageBytes;
        if (p.debug == 5) { mbar_arrive(&bar.full[s]); continue; }   // experiments: no loads
        if (i >= n_early) load_w(i);
        tma_load_2d(a, &maps.x, &bar.full[s], (kb_lo + i) * kBK, tm * kBM);
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
        if (p.debug != 4)   // experiments: 4 = no MMAs
#pragma unroll
        for (int kk = 0; kk < kBK / 16; ++kk)   // 16 k-elements = 32 B along the swizzled row
          mma_bf16_ss(tmem, ad0 + st + (uint64_t)(kk * 2), bd0 + st + (uint64_t)(kk * 2), idesc,
                      (i > 0 || kk > 0) ? 1u : 0u);
        mma_commit(&bar.empty[s]);
      }
      mma_commit(&bar.acc);
    }
  } else if (p.rope_theta > 0.0) {
    // ------------------------------------------------------------- RoPE table (idle warps 2-7)
    // inv_freq_j = theta^(-2j/D) once per j in double, then (cos, sin) of this
    // CTA's rows x 64 frequencies while the mainloop runs.
    const int t2 = threadIdx.x - 64;
    if (t2 < 64) inv_freq[t2] = exp2(-(2.0 * t2 / kHeadD) * log2(p.rope_theta));
    asm volatile("bar.sync 1, %0;" ::"n"(kThreads - 64) : "memory");
    if (own_rows <= kTableRows && t2 < 3 * 64) {
      // thread (j, chunk c of 3): the first row's angle exactly (double reduction),
      // later rows by rotating with (cos, sin) of one position step in fp32
      // (error grows ~1 ulp per row: <= 22 steps, far below bf16)
      const int j = t2 & 63, c = t2 >> 6;
      const int r0 = c * own_rows / 3, r1 = (c + 1) * own_rows / 3;
      if (r0 < r1) {
        float cs, sn, cd, sd;
        rope_cs(p.pos0 + tm * kBM + own_lo + r0, inv_freq[j], &cs, &sn);
        rope_cs(1, inv_freq[j], &cd, &sd);
        for (int r = r0; r < r1; ++r) {
          sts_f2(smem_u32(table + (r * 64 + j) * 2), cs, sn);
          const float cn = fmaf(cs, cd, -sn * sd);
          sn = fmaf(sn, cd, cs * sd);
          cs = cn;
        }
      }
    }
    if (threadIdx.x == 64) QKV_TRACE_T(8);
  }
  __syncwarp();

  // --------------------------------------------------------------- partials -> owners
  // After every CTA of the cluster has finished its mainloop (the receive
  // buffers reuse the stage memory), each thread pushes its TMEM row (one token,
  // 128 of the 256 columns) into the owning CTA's receive buffer
  // recv[src rank][owner-local row] with distributed-shared-memory stores.
  mbar_wait(&bar.acc, 0);
  griddep_wait();   // (returns at once by now) before any global write of this grid
  QKV_TRACE(2);
  tc_fence_after();
  cluster_sync_all();   // all mainloops done: stage memory is free cluster-wide
  QKV_TRACE(7);
  {
    // TMEM -> part (local, float4 index XOR (row & 7): conflict-free per-row stores)
    const int q = warp & 3;
    const int ch = warp >> 2;
    const int r = q * 32 + lane;
    const uint32_t d = smem_u32(part + (size_t)r * 256);
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
      uint32_t v0[32], v1[32];
      const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(ch * 128 + h2 * 64);
      tmem_ld32(ta, v0);
      tmem_ld32(ta + 32, v1);
      tmem_wait_ld();
      reg_fence32(v0);
      reg_fence32(v1);
      if (r < valid) {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int f0 = ch * 32 + h2 * 16 + e, f1 = f0 + 8;
          sts_u4(d + 16u * (uint32_t)(f0 ^ (r & 7)), v0[4 * e], v0[4 * e + 1], v0[4 * e + 2], v0[4 * e + 3]);
          sts_u4(d + 16u * (uint32_t)(f1 ^ (r & 7)), v1[4 * e], v1[4 * e + 1], v1[4 * e + 2], v1[4 * e + 3]);
        }
      }
    }
  }
  tc_fence_before();
  fence_proxy_async_smem();   // the bulk copies below read `part` through the async proxy
  __syncthreads();
  if (threadIdx.x == 0 && S > 1) {
    // one bulk DSMEM copy per peer: the owner's rows, into its recv slot for this rank
    for (int o = 0; o < S; ++o) {
      if (o == rank) continue;
      const int lo = row_lo(o), n = row_lo(o + 1) - lo;
      if (n == 0) continue;
      const int slot = rank < o ? rank : rank - 1;
      const uint32_t dst = mapa_shared(smem_u32(recv + (size_t)slot * rows_max * 256), (uint32_t)o);
      const uint32_t mb = mapa_shared(smem_u32(&bar.recv), (uint32_t)o);
      bulk_copy_s2cluster(dst, smem_u32(part + (size_t)lo * 256), (uint32_t)(n * kRowBytes), mb);
    }
    bulk_commit_group();
  }
  QKV_TRACE(3);
  if (S > 1) mbar_wait_cluster(&bar.recv, 0);   // peers' partials of this CTA's rows are here
  QKV_TRACE(4);
  if (p.debug == 1 || p.debug >= 3) {   // experiments: mainloop + exchange only
    if (threadIdx.x == 0 && S > 1) bulk_wait_group_read0();
    __syncthreads();
    if (warp == 2) tmem_dealloc<256>(tmem);
    return;
  }

  // --------------------------------------------------------------- reduce + RoPE + store
  {
    const int half = lane >> 4;           // 0: dims [0, 64), 1: dims [64, 128)
    const int j0 = 4 * (lane & 15);       // rotary frequency index of this lane's first dim
    const int dcol = 4 * lane;            // this lane's 4 dims within a head
    const int n_heads = p.Hq + 2 * p.Hkv;
    const bool rope = p.rope_theta > 0.0;
    const bool use_table = rope && own_rows <= kTableRows;
    auto load_row = [&](int rl, float4& a, float4& b) {
      const int ra = own_lo + rl;   // tile row (swizzle key)
      a = make_float4(0.f, 0.f, 0.f, 0.f);
      b = a;
      for (int sp = 0; sp < S; ++sp) {   // fixed order of ranks: deterministic sums
        const uint32_t src = smem_u32(sp == rank ? part + (size_t)ra * 256
                                                 : recv + (size_t)((sp < rank ? sp : sp - 1) * rows_max + rl) * 256);
        const float4 x = lds_f4(src + 16u * (uint32_t)(lane ^ (ra & 7)));
        const float4 y = lds_f4(src + 16u * (uint32_t)((32 + lane) ^ (ra & 7)));
        a.x += x.x; a.y += x.y; a.z += x.z; a.w += x.w;
        b.x += y.x; b.y += y.y; b.z += y.z; b.w += y.w;
      }
    };
    float4 na, nb;   // next row, loaded one step ahead (latency overlap)
    if (warp < own_rows) load_row(warp, na, nb);
    for (int rl = warp; rl < own_rows; rl += kThreads / 32) {
      const int t = tm * kBM + own_lo + rl;
      const float4 a = na, b = nb;
      if (rl + kThreads / 32 < own_rows) load_row(rl + kThreads / 32, na, nb);
      float cs[4], sn[4];
      if (use_table) {
        const uint32_t e = smem_u32(table + (rl * 64 + j0) * 2);
        const float4 c01 = lds_f4(e), c23 = lds_f4(e + 16);
        cs[0] = c01.x; sn[0] = c01.y; cs[1] = c01.z; sn[1] = c01.w;
        cs[2] = c23.x; sn[2] = c23.y; cs[3] = c23.z; sn[3] = c23.w;
      } else if (rope) {
#pragma unroll
        for (int c = 0; c < 4; ++c)
          rope_cs(p.pos0 + t, inv_freq[j0 + c], &cs[c], &sn[c]);
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
            if (p.kv_fp8)   // E4M3 pool (R-22): codes of the bf16-rounded values, as the quantize kernel
              *reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(pool) + prow * kHeadD + dcol) =
                  e4m3x4_of_bf16(packed, is_v ? p.v_scale : p.k_scale);
            else
              *reinterpret_cast<uint2*>(static_cast<uint8_t*>(pool) + (prow * kHeadD + dcol) * 2) = packed;
          }
        }
      }
    }
  }
  tc_fence_before();
  QKV_TRACE(5);
  if (threadIdx.x == 0 && S > 1) bulk_wait_group_read0();   // our outgoing copies finished reading
  __syncthreads();
  QKV_TRACE(6);
  if (warp == 2) tmem_dealloc<256>(tmem);
}

}  // namespace

bool qkv_supported(int D, int hidden) { return D == kHeadD && hidden > 0 && hidden % kBK == 0; }

// part (valid rows) + recv ((S-1) x ceil(valid/S) rows) must fit in the stage memory
static bool qkv_exchange_fits(int m, int s) {
  const int v = m < kBM ? m : kBM;
  return v + (s - 1) * ((v + s - 1) / s) <= kExchangeRows;
}

int qkv_choose_splits(int m, int n_heads, int hidden, int num_sms) {
  // the most CTAs (tiles x S) whose clusters are all co-resident (one wave);
  // S = 1 when even that does not fit
  const int tiles = ((n_heads * kHeadD + kBN - 1) / kBN) * ((m + kBM - 1) / kBM);
  const int nkb = hidden / kBK;
  static int max_active[kMaxSplits + 1] = {0};
  int best = 1;
  for (int s = 2; s <= kMaxSplits && s <= nkb; ++s) {
    if (!qkv_exchange_fits(m, s)) continue;
    if (max_active[s] == 0) max_active[s] = qkv_max_active_clusters(s);
    if (tiles <= max_active[s] && tiles * s <= num_sms) best = s;
  }
  return best;
}

static size_t qkv_smem_bytes() {
  return (size_t)kStages * kStageBytes + kTableBytes + 64 * 8 + sizeof(QkvBars) + 1024;
}

// Largest number of co-resident clusters of `splits` CTAs (cudaOccupancyMaxActiveClusters).
int qkv_max_active_clusters(int splits) {
  const size_t smem = qkv_smem_bytes();
  if (cudaFuncSetAttribute(qkv_rope_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return -1;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(splits * 64, 1, 1);
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = splits;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = -1;
  if (cudaOccupancyMaxActiveClusters(&n, qkv_rope_kernel, &cfg) != cudaSuccess) return -1;
  return n;
}

cudaError_t launch_qkv_rope(const QkvParams& p, cudaStream_t s, bool pdl) {
  if (p.m <= 0) return cudaSuccess;
  if (!qkv_supported(p.D, p.hidden) || p.splits < 1 || p.splits > kMaxSplits || p.splits > p.hidden / kBK ||
      !qkv_exchange_fits(p.m, p.splits))
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
    if (p.debug >= 2) {
      dims[0] = kBK;
      dims[1] = (cuuint64_t)n_heads * kHeadD * (p.hidden / kBK);
      str[0] = kBK * 2;
    }
    cuuint32_t box[2] = {kBK, kBN};
    if (!encode_bf16_map(&maps.w, p.W, 2, dims, str, box)) return cudaErrorInvalidValue;
  }
  const size_t smem = qkv_smem_bytes();
  {
    cudaError_t e = set_smem_attr_once(reinterpret_cast<const void*>(qkv_rope_kernel), (int)smem);
    if (e != cudaSuccess) return e;
  }
  const int n_tiles_n = (n_heads * kHeadD + kBN - 1) / kBN;
  const int n_tiles_m = (p.m + kBM - 1) / kBM;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(n_tiles_n * p.splits, n_tiles_m, 1);
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = p.splits;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, qkv_rope_kernel, p, maps);
}

}  // namespace ssa
