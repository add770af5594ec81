// kernels_tc.cu — tensor-core (tcgen05 / TMEM / TMA) attention for sm_100a.
//
// A CTA runs up to two work units ("slots", plan.cpp pair_units) with two
// softmax warpgroups that ping-pong against one MMA issuer.  The first
// n_shared key tiles are common to both slots and loaded once (each K/V tile
// then feeds 256 query rows: the q tiles of an append, or Flash Queries over
// one cached pool); later tiles are private to a slot (own-token tails, or the
// two key ranges of a split pair that shares one q tile).
// Per slot and key tile of 128 keys (Eq. attention P:145 on the rows of Eq.
// query-attention P:150-155; causal tail, reading R-2):
//     S = Q K^T         tcgen05.mma M=128 N=128 K=128 -> TMEM (fp32)
//     P = 2^(S*c - m)   softmax warpgroup, one thread per row (TMEM lane);
//                       P (bf16) is written back into the S columns of TMEM
//     O += P V          tcgen05.mma with A = P from TMEM, B = V from smem
// TMEM (512 columns): slot k uses [256k, 256k+128) for S/P and
// [256k+128, 256k+256) for O.  The running max is updated lazily (only when it
// grows by more than 8 in log2 units), so O is rarely rescaled.
// Warp roles (384 threads): warp 0 TMA producer of Q and the K ring, warp 3 TMA
// producer of the V ring, warp 1 MMA issuer, warp 2 TMEM allocator, warps 4-7
// softmax slot 0, warps 8-11 softmax slot 1.  A warp whose 32 rows are all
// padding (a 1-token GQA query fills 4 of 128 rows) skips its softmax.
//
// Split-KV epilogues (AttnParams::cm_C, cm_gbar, cm_gsplit): a CTA holding its
// whole group writes O (a split pair merges its two slots straight from TMEM);
// a group split over several CTAs of a single-layer call leaves fp32 partials,
// merged through DSMEM inside a thread-block cluster (cm_reduce), by a merge
// kernel right behind the grid (gm_merge_kernel for the one-wave group plan,
// the default of query-plane calls; cm_merge_kernel for groups over several
// clusters), or after a group barrier in global memory (gm_reduce, an option).
//
// FP8 KV variant (template F8, reading R-22): the pools and
// the call's own K/V hold E4M3 codes.  Lanes 0 / 1 of warp 0 load the K / V
// tiles (16 KB of codes) into the upper half of their 32 KB ring slots; warp 2
// (K) and warp 3 (V)
// convert the codes in place to fp16 in the same 128-byte-swizzled layout the
// bf16 tiles use (cvt.rn.f16x2.e4m3x2 is exact), and the MMAs run kind::f16 with
// fp16 operands: Q is converted bf16 -> fp16 in smem once per CTA, P is packed
// as fp16.  The K scale folds into the softmax constant, the V scale into 1/l.
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

constexpr int kM = 128;          // rows per q tile (= TMEM lanes)
constexpr int kBN = 128;         // keys per tile
constexpr int kD = 128;          // head dim: two 64-column (128 B) swizzle chunks
constexpr int kThreads = 384;
constexpr int kChunkBytes = 128 * 128;          // 128 rows x 128 B
constexpr int kSlotBytes = 2 * kChunkBytes;     // one 128 x 128 bf16 tile = 32 KB
constexpr int kNumSlots = 7;                    // 224 KB of tiles
constexpr int kMaxStages = 3;
#ifndef SSA_RESCALE_LOG2
#define SSA_RESCALE_LOG2 8.0f
#endif
constexpr float kRescaleLog2 = SSA_RESCALE_LOG2;   // lazy max threshold (log2 units)
// setmaxnreg budget: the CTA's pool is fixed at launch (168 regs x 384 threads
// from __launch_bounds__(384, 1)); setmaxnreg.inc blocks until registers are
// free, so the rebalanced total must fit the pool or the kernel deadlocks.
constexpr int kLaunchRegs = 168;
constexpr int kRegsWG0 = 56;       // TMA producer / MMA issuer / allocator warpgroup
constexpr int kRegsSoftmax = 224;  // two softmax warpgroups
static_assert(128 * kRegsWG0 + 256 * kRegsSoftmax <= kLaunchRegs * kThreads, "setmaxnreg over the CTA pool");
static_assert(kRegsWG0 % 8 == 0 && kRegsSoftmax % 8 == 0, "setmaxnreg needs multiples of 8");

struct Bars {
  uint64_t q_full;
  uint64_t q_ready;               // F8: Q converted to fp16 (both converter warps)
  uint64_t k_raw[kMaxStages];     // F8: E4M3 codes of a K stage landed (TMA)
  uint64_t v_raw[kMaxStages];
  uint64_t k_full[kMaxStages];
  uint64_t v_full[kMaxStages];
  uint64_t k_empty[kMaxStages];   // K stage consumed by the S MMA(s) of its event
  uint64_t v_empty[kMaxStages];   // V stage consumed by the PV MMA(s) of its event
  uint64_t s_full[2];
  uint64_t p_full[2];
  uint64_t o_final[2];
  uint32_t tmem_base;
};

struct TcMaps {
  CUtensorMap q;       // [rows][Hq][D]   box {64, G, 128/G}
  CUtensorMap q32;     // [rows][Hq][D]   box {64, G, 32/G}  (duplicated small q tiles)
  CUtensorMap kt;      // [rows][Hkv][D]  box {64, 1, 128}
  CUtensorMap vt;
  CUtensorMap pk;      // [L*num_pages*Hkv*P][D] box {64, BR}
  CUtensorMap pv;
};

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ uint32_t pack_f16(float a, float b) {
  uint32_t r;
  asm("cvt.rn.f16x2.f32 %0, %2, %1;" : "=r"(r) : "f"(a), "f"(b));
  return r;
}
template <bool F8>
__device__ __forceinline__ uint32_t pack_p(float a, float b) {
  return F8 ? pack_f16(a, b) : pack_bf16(a, b);
}
// four E4M3 codes (bytes, lowest first) -> two fp16 pairs, exactly
__device__ __forceinline__ uint2 e4m3x4_to_f16x4(uint32_t w) {
  uint2 r;
  asm("{\n\t.reg .b16 lo, hi;\n\tmov.b32 {lo, hi}, %2;\n\t"
      "cvt.rn.f16x2.e4m3x2 %0, lo;\n\tcvt.rn.f16x2.e4m3x2 %1, hi;\n\t}"
      : "=r"(r.x), "=r"(r.y) : "r"(w));
  return r;
}
// bf16 pair -> fp16 pair (Q of the FP8 variant; |q| well inside fp16's range)
__device__ __forceinline__ uint32_t bf16x2_to_f16x2(uint32_t w) {
  return pack_f16(__uint_as_float(w << 16), __uint_as_float(w & 0xFFFF0000u));
}

// 16-byte shared-memory accesses by 32-bit shared address (LDS / STS: the
// aligned generic pointer of the dynamic smem would compile to generic LD / ST)
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts128(uint32_t a, uint4 v) {
  asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

// In-place conversion of one ring slot: codes in [kChunkBytes, 2 kChunkBytes)
// (128 rows x 128 B, 128-byte swizzle) -> fp16 tile [128 rows][128 d] as two
// 64-column swizzled chunks.  Each lane converts whole rows (row 32 it + lane):
// it loads the row's 128 codes into registers before storing its 256 bytes of
// fp16, so the in-place overlap (output chunk 1 of row r is code row r) needs no
// cross-lane ordering and no barrier.  The 8 lanes of a quarter-warp are 8 rows
// with distinct swizzle phases, so every LDS / STS is bank-conflict free.
// (Measured alternatives: 4 lanes per row with a warp barrier per
// row group, half rows per step -- both slower.)
__device__ __forceinline__ void convert_kv_slot(uint32_t slot, int lane) {
  const int sw = lane & 7;
#pragma unroll 1
  for (int it = 0; it < 4; ++it) {
    const int r = it * 32 + lane;
    const uint32_t in = slot + kChunkBytes + r * 128;
    uint4 x[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = lds128(in + ((c ^ sw) << 4));
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const uint32_t out = slot + (c >> 2) * kChunkBytes + r * 128;
      const int cc = 2 * (c & 3);
      const uint2 a0 = e4m3x4_to_f16x4(x[c].x), a1 = e4m3x4_to_f16x4(x[c].y);
      const uint2 a2 = e4m3x4_to_f16x4(x[c].z), a3 = e4m3x4_to_f16x4(x[c].w);
      sts128(out + ((cc ^ sw) << 4), make_uint4(a0.x, a0.y, a1.x, a1.y));
      sts128(out + (((cc + 1) ^ sw) << 4), make_uint4(a2.x, a2.y, a3.x, a3.y));
    }
  }
}
// In-place bf16 -> fp16 of a 32 KB Q tile (same element positions).
__device__ __forceinline__ void convert_q_tile(uint32_t q, int lane) {
#pragma unroll 4
  for (int i = lane; i < kSlotBytes / 16; i += 32) {
    uint4 v = lds128(q + i * 16);
    v.x = bf16x2_to_f16x2(v.x);
    v.y = bf16x2_to_f16x2(v.y);
    v.z = bf16x2_to_f16x2(v.z);
    v.w = bf16x2_to_f16x2(v.w);
    sts128(q + i * 16, v);
  }
}

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// exp2 runs on MUFU (16/clk/SM on B200, one op per element).  Measured
// alternatives that do not help on sm_100a (scripts/ubench_sfu.cu): a degree-3
// polynomial on the FMA pipe (13.8 elements/clk/SM, issue-bound) and
// ex2.approx.bf16x2 (ptxas splits it into two MUFU.EX2.BF16 + PRMT).

// Optional per-tile timestamps (debug builds with -DSSA_TRACE): clock64 of the
// softmax and MMA-issuer events of a few CTAs, read back by ssa_debug_trace().
#ifdef SSA_TRACE
constexpr int kTraceCtas = 4, kTraceTiles = 256, kTraceLayer = 5;
__device__ unsigned long long g_trace[kTraceCtas][12][kTraceTiles][2];
#define TRACE(cond, row, j, w, val) \
  do { if ((cond) && blockIdx.y == kTraceLayer && blockIdx.x < kTraceCtas && (j) < kTraceTiles) \
         g_trace[blockIdx.x][row][j][w] = (val); } while (0)
#else
#define TRACE(cond, row, j, w, val) do { } while (0)
#endif

// Optional launch-phase trace (debug builds with -DSSA_GTRACE): %globaltimer (ns) of
// a few events per CTA, per pool layer (mod 32) of a launch, read back by
// ssa_debug_trace() as [32 layers][256 CTAs][16]; 8-13: CM epilogue (rows staged,
// cluster barrier 1 passed, block reduced, ticket taken, merge done, barrier 2 passed).
// 0 entry, 1 setup done, 2 Q landed (MMA issuer), 3 first K stage landed,
// 4 first S of slot 0 seen by the softmax, 5 last PV of slot 0 done, 6 epilogue
// done, 7 SM id.
#ifdef SSA_GTRACE
constexpr int kGtCtas = 256;
__device__ unsigned long long g_gtrace[32][kGtCtas][16];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define GTRACE(cond, ev) \
  do { if ((cond) && blockIdx.x < kGtCtas) g_gtrace[(p.layer0 + blockIdx.y) & 31][blockIdx.x][ev] = gtime(); } while (0)
#define GTRACE_T(cond, ev) GTRACE((cond) && threadIdx.x == 128, ev)
#else
#define GTRACE(cond, ev) do { } while (0)
#define GTRACE_T(cond, ev) do { } while (0)
#endif

// Optional exp2 offload (SSA_POLY_PAIRS_OF_8 = n > 0): n of every 8 element
// pairs use 2^x = 2^j * p(f) on the FMA pipe (j = rint(x) by the 1.5*2^23 magic
// add, f in [-0.5, 0.5], degree-3 minimax p with relative error 7.5e-5, far
// below bf16's 2^-8 unit roundoff of P; x clamped at -126).
#ifndef SSA_POLY_PAIRS_OF_8
#define SSA_POLY_PAIRS_OF_8 0
#endif
constexpr int kPolyPairsOf8 = SSA_POLY_PAIRS_OF_8;
// Ring stages (per K / V ring) of pool tiles a programmatic launch requests before
// griddepcontrol.wait.  The Q tile, requested after the wait, queues behind them: one
// stage measured best on the per-layer query (31.7 vs 32.5 us/layer with a full ring,
// 32.2 with none; scripts/early_stages_ab.sh)
#ifndef SSA_EARLY_STAGES
#define SSA_EARLY_STAGES 1
#endif

// ---------------------------------------------------------------- cluster merge (CM)
// CM launches (AttnParams::cm_C = C >= 1): every unit belongs to a split group and
// the C CTAs of a thread-block cluster (consecutive blockIdx.x) hold C key ranges
// of one q tile (SPLIT pairs: a CTA's two slots are two further ranges, merged in
// the CTA) or of two q tiles (SHARED pairs).  Each CTA leaves the normalized O rows
// (fp32) and lse of its q tile(s) in its idle ring shared memory; after a cluster
// barrier CTA rank r merges row block r over the C CTAs through DSMEM (log-sum-exp,
// reading R-11) and writes O.  A group spread over K > 1 clusters writes the block
// as a partial instead, and the last of the K CTAs of rank r to arrive (atomic
// ticket, no spin waits) merges the K partials.  No combine launch, no partials in
// HBM when K = 1.
constexpr int kXStride = 132;                 // fp32 row stride: 16-B aligned, conflict-free float4 stores
constexpr int kXFloats = kM * kXStride + kM;   // rows + lse

// Barrier over every thread of the cluster (C > 1) or of the CTA (named barrier
// 4; callers sit at different points of the warp-role branches, so the CTA
// barriers are the non-.aligned `barrier.sync` / `barrier.arrive` forms).
__device__ __forceinline__ void cm_sync(int C) {
  __syncwarp();   // converged warps at the (non-.aligned) CTA barrier / the .aligned cluster barrier
  if (C > 1)
    cluster_sync_all();
  else
    asm volatile("barrier.sync 4, %0;" ::"n"(kThreads) : "memory");
}
// Named barrier 5 orders the end of every warp-0..3 role (TMA issue, E4M3
// conversion writes into the ring) before the epilogue writes its exchange rows
// into the same ring shared memory: warps 0-3 arrive, the softmax warps wait.
__device__ __forceinline__ void ring_free_arrive() {
  __syncwarp();
  asm volatile("barrier.arrive 5, %0;" ::"n"(kThreads) : "memory");
}
__device__ __forceinline__ void ring_free_wait() {
  __syncwarp();
  asm volatile("barrier.sync 5, %0;" ::"n"(kThreads) : "memory");
}

__device__ __forceinline__ float ld_dsmem_f32(uint32_t a) {
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ float4 lds_f4(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ float4 ld_dsmem_v4(uint32_t a) {
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a)
               : "memory");
  return v;
}

__device__ __forceinline__ void store_bf16x4(__nv_bfloat16* out, float4 v) {
  uint2 u;
  u.x = pack_bf16(v.x, v.y);
  u.y = pack_bf16(v.z, v.w);
  *reinterpret_cast<uint2*>(out) = u;
}

// Slot rows -> exchange row `dst` (smem exchange buffer, or a global partial row in a
// group-barrier launch): O * inv_l (zeros for a row with no keys), lse at *dst_lse.
__device__ __forceinline__ void cm_stage_rows(float* dst, float* dst_lse, bool live, uint32_t o_col, float inv_l,
                                              float lse, bool has) {
#pragma unroll
  for (int q4 = 0; q4 < 4; ++q4) {
    uint32_t ro[32];
    tmem_ld32(o_col + q4 * 32, ro);
    tmem_wait_ld();
    if (live) {
#pragma unroll
      for (int i = 0; i < 32; i += 4)
        *reinterpret_cast<float4*>(dst + q4 * 32 + i) =
            has ? make_float4(__uint_as_float(ro[i]) * inv_l, __uint_as_float(ro[i + 1]) * inv_l,
                              __uint_as_float(ro[i + 2]) * inv_l, __uint_as_float(ro[i + 3]) * inv_l)
                : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  if (live) *dst_lse = has ? lse : -CUDART_INF_F;
}
// The same rows into a global partial in the column-major float4 layout of
// cm_merge_rows (group-barrier launches), lse at gpart_lse[rr].
__device__ __forceinline__ void gm_stage_rows(float4* gpart, float* gpart_lse, int rr, bool live, uint32_t o_col,
                                              float inv_l, float lse, bool has) {
#pragma unroll
  for (int q4 = 0; q4 < 4; ++q4) {
    uint32_t ro[32];
    tmem_ld32(o_col + q4 * 32, ro);
    tmem_wait_ld();
    if (live) {
#pragma unroll
      for (int i = 0; i < 32; i += 4)
        gpart[(q4 * 8 + i / 4) * kM + rr] =
            has ? make_float4(__uint_as_float(ro[i]) * inv_l, __uint_as_float(ro[i + 1]) * inv_l,
                              __uint_as_float(ro[i + 2]) * inv_l, __uint_as_float(ro[i + 3]) * inv_l)
                : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  if (live) gpart_lse[rr] = has ? lse : -CUDART_INF_F;
}
__device__ __forceinline__ float* x_row(float* X, int rr) { return X + rr * kXStride; }
__device__ __forceinline__ float* x_lse(float* X, int rr) { return X + kM * kXStride + rr; }

// Split pair: slot 0 merges slot 1's staged rows with its own (R-11), in place --
// or, with `out` (a CTA that holds its whole group: cluster of 1, one cluster per
// group), straight into the bf16 output row, or with `gdst` (a group-barrier
// launch) into this CTA's global partial (column-major float4 layout, element
// (c, row) at gdst[c * kM + row]: a warp's stores are 512 contiguous bytes), lse at *glse.
__device__ __forceinline__ void cm_merge_rows(float* X, int rr, bool live, uint32_t o_col, float inv_l, float lse,
                                              bool has, __nv_bfloat16* out = nullptr, float* gdst = nullptr,
                                              float* glse = nullptr) {
  float a0 = 0.f, a1 = 0.f, lm = -CUDART_INF_F;
  if (live) {
    const float l1 = X[kM * kXStride + rr];
    const float l0 = has ? lse : -CUDART_INF_F;
    const float L = fmaxf(l0, l1);
    if (L != -CUDART_INF_F) {
      const float w0 = l0 == -CUDART_INF_F ? 0.f : exp2f(l0 - L);
      const float w1 = l1 == -CUDART_INF_F ? 0.f : exp2f(l1 - L);
      const float inv = 1.f / (w0 + w1);
      a0 = w0 * inv * inv_l;
      a1 = w1 * inv;
      lm = L + __log2f(w0 + w1);
    }
  }
#pragma unroll
  for (int q4 = 0; q4 < 4; ++q4) {
    uint32_t ro[32];
    tmem_ld32(o_col + q4 * 32, ro);
    tmem_wait_ld();
    if (live) {
      float* dst = X + rr * kXStride + q4 * 32;
#pragma unroll
      for (int i = 0; i < 32; i += 4) {
        const float4 x1 = *reinterpret_cast<const float4*>(dst + i);
        float4 v;
        v.x = (a0 != 0.f ? a0 * __uint_as_float(ro[i]) : 0.f) + a1 * x1.x;
        v.y = (a0 != 0.f ? a0 * __uint_as_float(ro[i + 1]) : 0.f) + a1 * x1.y;
        v.z = (a0 != 0.f ? a0 * __uint_as_float(ro[i + 2]) : 0.f) + a1 * x1.z;
        v.w = (a0 != 0.f ? a0 * __uint_as_float(ro[i + 3]) : 0.f) + a1 * x1.w;
        if (out)
          store_bf16x4(out + q4 * 32 + i, v);
        else if (gdst)
          reinterpret_cast<float4*>(gdst)[(q4 * 8 + i / 4) * kM + rr] = v;
        else
          *reinterpret_cast<float4*>(dst + i) = v;
      }
    }
  }
  if (live && !out) *(gdst ? glse : x_lse(X, rr)) = lm;
}

// Split pair without row duplication: slot 1's O rows sit in the same TMEM lanes as
// slot 0's (columns +256), so slot 0 reads both straight from TMEM; slot 1 only
// leaves its lse and 1/l per row in X (lse area and the next kM floats).  Output
// as cm_merge_rows: bf16 `out`, the global partial `gdst` (+ *glse), or X in place.
__device__ __forceinline__ void cm_merge_tmem(float* X, int rr, bool live, uint32_t o_col, float inv_l, float lse,
                                              bool has, __nv_bfloat16* out, float* gdst, float* glse) {
  float a0 = 0.f, a1 = 0.f, lm = -CUDART_INF_F;
  if (live) {
    const float l1 = *x_lse(X, rr);
    const float il1 = *(x_lse(X, rr) + kM);
    const float l0 = has ? lse : -CUDART_INF_F;
    const float L = fmaxf(l0, l1);
    if (L != -CUDART_INF_F) {
      const float w0 = l0 == -CUDART_INF_F ? 0.f : exp2f(l0 - L);
      const float w1 = l1 == -CUDART_INF_F ? 0.f : exp2f(l1 - L);
      const float inv = 1.f / (w0 + w1);
      a0 = w0 * inv * inv_l;
      a1 = w1 * inv * il1;
      lm = L + __log2f(w0 + w1);
    }
  }
#pragma unroll
  for (int q4 = 0; q4 < 4; ++q4) {
    uint32_t r0[32], r1[32];
    tmem_ld32(o_col + q4 * 32, r0);
    tmem_ld32(o_col + 256 + q4 * 32, r1);
    tmem_wait_ld();
    if (live) {
#pragma unroll
      for (int i = 0; i < 32; i += 4) {
        float4 v;
        v.x = (a0 != 0.f ? a0 * __uint_as_float(r0[i]) : 0.f) + (a1 != 0.f ? a1 * __uint_as_float(r1[i]) : 0.f);
        v.y = (a0 != 0.f ? a0 * __uint_as_float(r0[i + 1]) : 0.f) + (a1 != 0.f ? a1 * __uint_as_float(r1[i + 1]) : 0.f);
        v.z = (a0 != 0.f ? a0 * __uint_as_float(r0[i + 2]) : 0.f) + (a1 != 0.f ? a1 * __uint_as_float(r1[i + 2]) : 0.f);
        v.w = (a0 != 0.f ? a0 * __uint_as_float(r0[i + 3]) : 0.f) + (a1 != 0.f ? a1 * __uint_as_float(r1[i + 3]) : 0.f);
        if (out)
          store_bf16x4(out + q4 * 32 + i, v);
        else if (gdst)
          reinterpret_cast<float4*>(gdst)[(q4 * 8 + i / 4) * kM + rr] = v;
        else
          *reinterpret_cast<float4*>(x_row(X, rr) + q4 * 32 + i) = v;
      }
    }
  }
  if (live && !out) *(gdst ? glse : x_lse(X, rr)) = lm;
}

__device__ __forceinline__ void store_bf16x8(__nv_bfloat16* out, const float* v) {
  uint4 u;
  u.x = pack_bf16(v[0], v[1]);
  u.y = pack_bf16(v[2], v[3]);
  u.z = pack_bf16(v[4], v[5]);
  u.w = pack_bf16(v[6], v[7]);
  *reinterpret_cast<uint4*>(out) = u;
}

// Row block `rank` of one q tile's exchange buffers over the C CTAs of the
// cluster, by warpgroup k.  Warp wq takes rows rank*R + wq + 4i; lane l takes
// columns [4l, 4l+4) -- every (D)SMEM and global access of a warp is one whole
// 512-byte row (coalesced: DSMEM runs at global-memory-like segment rates).
__device__ __forceinline__ float lds_f32(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a) : "memory");
  return v;
}

template <int C>
__device__ __forceinline__ void cm_reduce(const AttnParams& p, const WorkUnit& w, const float* X, int k) {
  constexpr int R = (kM + C - 1) / C;       // rows of this CTA's block (the last blocks may be short)
  constexpr int RB = C >= 16 ? 1 : 16 / C > 0 ? 16 / C : 1;  // rows per warp per batch of loads
  const int t = threadIdx.x - 128 - 128 * k;
  const int wq = t >> 5, lane = t & 31;
  const uint32_t rank = C > 1 ? cluster_ctarank() : 0u;
  const int G = p.G;
  const int ly = blockIdx.y;
  const int row0 = (int)rank * R;
  const int row_end = min(row0 + R, w.q_ntok * G);   // live rows of the block
  const SegDesc sg = p.segs[w.seg];
  const int64_t in_l = p.in_layer_stride ? (int64_t)ly * p.rows_per_layer : 0;
  const Group gr = p.groups[w.group];
  const int K = gr.n_splits;   // clusters holding key ranges of this group
  const uint32_t xa = smem_u32(X);
  const int64_t s0 = (int64_t)ly * p.n_units + gr.unit0;
  auto out_ptr = [&](int row) {
    const int64_t orow = in_l + sg.row0 + w.q_tok0 + row / G;
    return static_cast<__nv_bfloat16*>(p.O) + (orow * p.Hq + w.kv_head * G + row % G) * kD + 4 * lane;
  };
  for (int r0 = row0 + wq; r0 < row_end; r0 += 4 * RB) {
    float lc[RB][C];
    float4 v[RB][C];
#pragma unroll
    for (int b = 0; b < RB; ++b) {
      const int row = min(r0 + 4 * b, row_end - 1);
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const uint32_t la = xa + (uint32_t)(kM * kXStride + row) * 4u;
        const uint32_t va = xa + (uint32_t)(row * kXStride + 4 * lane) * 4u;
        lc[b][c] = C > 1 ? ld_dsmem_f32(mapa_shared(la, (uint32_t)c)) : lds_f32(la);
        v[b][c] = C > 1 ? ld_dsmem_v4(mapa_shared(va, (uint32_t)c)) : lds_f4(va);
      }
    }
#pragma unroll
    for (int b = 0; b < RB; ++b) {
      const int row = r0 + 4 * b;
      if (row >= row_end) break;
      float L = -CUDART_INF_F;
#pragma unroll
      for (int c = 0; c < C; ++c) L = fmaxf(L, lc[b][c]);
      float wsum = 0.f;
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int c = 0; c < C; ++c) {
        // staged rows are finite (zeros for a CTA without keys): zero weights need no branch
        const float wt = lc[b][c] == -CUDART_INF_F ? 0.f : exp2f(lc[b][c] - L);
        wsum += wt;
        acc.x = fmaf(wt, v[b][c].x, acc.x);
        acc.y = fmaf(wt, v[b][c].y, acc.y);
        acc.z = fmaf(wt, v[b][c].z, acc.z);
        acc.w = fmaf(wt, v[b][c].w, acc.w);
      }
      const float inv = wsum > 0.f ? 1.f / wsum : 0.f;
      acc = make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
      if (K == 1) {
        store_bf16x4(out_ptr(row), acc);
      } else {
        *reinterpret_cast<float4*>(p.part_o + ((s0 + w.split) * kM + row) * kD + 4 * lane) = acc;
        if (lane == 0) p.part_lse[(s0 + w.split) * kM + row] = wsum > 0.f ? L + __log2f(wsum) : -CUDART_INF_F;
      }
    }
  }
  GTRACE_T(true, 10);
  if (K > 1 && p.cm_tickets) {
    // In-kernel variant of cm_merge_kernel: the last of the K clusters' rank-r CTAs to
    // arrive (atomic ticket, no spin waits) merges the K block partials of block r.
    __threadfence();
    asm volatile("barrier.sync %0, 128;" ::"r"(1 + k) : "memory");
    __shared__ uint32_t last[2];
    if (t == 0) {
      int* cnt = p.cm_tickets + ((int64_t)ly * p.n_groups + w.group) * C + rank;
      const int old = atomicAdd(cnt, 1);
      last[k] = old == K - 1 ? 1u : 0u;
      if (old == K - 1) *cnt = 0;   // every arrival is in: ready for the next launch
    }
    asm volatile("barrier.sync %0, 128;" ::"r"(1 + k) : "memory");
    GTRACE_T(true, 11);
    if (last[k]) {
      __threadfence();
      constexpr int MB = 4;   // rows per batch of loads
      for (int r0 = row0 + wq; r0 < row_end; r0 += 4 * MB) {
        float m[MB], wsum[MB];
        float4 acc[MB];
#pragma unroll
        for (int b = 0; b < MB; ++b) {
          m[b] = -CUDART_INF_F;
          wsum[b] = 0.f;
          acc[b] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        for (int j0 = 0; j0 < K; j0 += 4) {
          float l[MB][4];
          float4 v[MB][4];
#pragma unroll
          for (int b = 0; b < MB; ++b)
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
              const int row = min(r0 + 4 * b, row_end - 1);
              const int j = min(j0 + jj, K - 1);
              l[b][jj] = j0 + jj < K ? __ldcg(p.part_lse + (s0 + j) * kM + row) : -CUDART_INF_F;
              v[b][jj] = __ldcg(reinterpret_cast<const float4*>(p.part_o + ((s0 + j) * kM + row) * kD) + lane);
            }
#pragma unroll
          for (int b = 0; b < MB; ++b) {
            float mb = m[b];
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) mb = fmaxf(mb, l[b][jj]);
            if (mb == -CUDART_INF_F) continue;
            const float sc = m[b] == -CUDART_INF_F ? 0.f : exp2f(m[b] - mb);
            wsum[b] *= sc;
            acc[b] = make_float4(acc[b].x * sc, acc[b].y * sc, acc[b].z * sc, acc[b].w * sc);
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
              const float wt = l[b][jj] == -CUDART_INF_F ? 0.f : exp2f(l[b][jj] - mb);
              wsum[b] += wt;
              acc[b].x = fmaf(wt, v[b][jj].x, acc[b].x);
              acc[b].y = fmaf(wt, v[b][jj].y, acc[b].y);
              acc[b].z = fmaf(wt, v[b][jj].z, acc[b].z);
              acc[b].w = fmaf(wt, v[b][jj].w, acc[b].w);
            }
            m[b] = mb;
          }
        }
#pragma unroll
        for (int b = 0; b < MB; ++b) {
          const int row = r0 + 4 * b;
          if (row >= row_end) break;
          const float inv = wsum[b] > 0.f ? 1.f / wsum[b] : 0.f;
          store_bf16x4(out_ptr(row), make_float4(acc[b].x * inv, acc[b].y * inv, acc[b].z * inv, acc[b].w * inv));
        }
      }
    }
  }
}

// Group-barrier merge (AttnParams::cm_gbar; single-wave launches of clusters of
// one CTA): every CTA of a group has written its (slot-merged, normalized) rows
// as global partial `split` with their lse; the group's K CTAs meet at a barrier
// in global memory (arrival counter + generation word per (layer, group), the
// last arriver resets the counter and bumps the generation), then CTA `split`
// merges row block `split` of the K partials (log-sum-exp, R-11) and writes O.
// All CTAs of the launch are co-resident (grid <= SMs, one CTA per SM), so the
// spin cannot wait on a CTA that is not running.  Warp wq takes rows
// row0 + wq + 4i, lane l the partial l's lse (K <= 32) and columns [4l, 4l+4).
__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* a) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
  return v;
}
// t in [0, nthr): this thread's index among the nthr threads (one or both softmax
// warpgroups, named barrier `bar_id`) that merge the group's row block.  Partial j
// of the group is part_o[(s0 + j) * kM * kD ...] in the column-major float4 layout
// of cm_merge_rows; item (row, c) = 4 output columns of one row, K loads in flight.
template <int KMAX>
__device__ __forceinline__ void gm_merge_items(const AttnParams& p, const WorkUnit& w, int K, int t, int nthr) {
  const int ly = blockIdx.y;
  const int G = p.G;
  const int rows = w.q_ntok * G;
  const int R = (rows + K - 1) / K;
  const int row0 = w.split * R;
  const int nr = min(row0 + R, rows) - row0;
  const SegDesc sg = p.segs[w.seg];
  const int64_t in_l = p.in_layer_stride ? (int64_t)ly * p.rows_per_layer : 0;
  const int64_t s0 = (int64_t)ly * p.n_units + p.groups[w.group].unit0;
  const float4* po = reinterpret_cast<const float4*>(p.part_o) + s0 * (kM * kD / 4);
  const float* pl = p.part_lse + s0 * kM;
  // items: (row, c) with rows fastest within groups of 8, so a warp reads 4 x 128 B
  for (int it = t; it < ((nr + 7) & ~7) * (kD / 4); it += nthr) {
    const int row = row0 + (it & 7) + 8 * ((it >> 3) / (kD / 4));
    const int c = (it >> 3) % (kD / 4);
    if (row >= row0 + nr) continue;
    float lj[KMAX];
    float4 v[KMAX];
#pragma unroll
    for (int j = 0; j < KMAX; ++j)
      if (j < K) {
        lj[j] = __ldcg(pl + (int64_t)j * kM + row);
        v[j] = __ldcg(po + (int64_t)j * (kM * kD / 4) + c * kM + row);
      }
    float L = -CUDART_INF_F;
#pragma unroll
    for (int j = 0; j < KMAX; ++j)
      if (j < K) L = fmaxf(L, lj[j]);
    float ws = 0.f;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int j = 0; j < KMAX; ++j)
      if (j < K) {
        const float wt = lj[j] == -CUDART_INF_F ? 0.f : exp2f(lj[j] - L);
        ws += wt;
        acc.x = fmaf(wt, v[j].x, acc.x);
        acc.y = fmaf(wt, v[j].y, acc.y);
        acc.z = fmaf(wt, v[j].z, acc.z);
        acc.w = fmaf(wt, v[j].w, acc.w);
      }
    const float inv = ws > 0.f ? 1.f / ws : 0.f;
    const int64_t orow = in_l + sg.row0 + w.q_tok0 + row / G;
    store_bf16x4(static_cast<__nv_bfloat16*>(p.O) + (orow * p.Hq + w.kv_head * G + row % G) * kD + 4 * c,
                 make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv));
  }
}

// gen0: the group's generation word, read by thread t == 0 before this CTA's partial
// rows were written (any time after griddepcontrol.wait and before the arrival: only
// this launch's last arriver changes it), so the read is off the barrier's critical path.
__device__ __forceinline__ uint32_t gm_generation(const AttnParams& p, int group) {
  return ld_acquire_u32(reinterpret_cast<uint32_t*>(p.cm_tickets) + ((int64_t)blockIdx.y * p.n_groups + group) * 2 + 1);
}
__device__ __forceinline__ void gm_reduce(const AttnParams& p, const WorkUnit& w, int t, int nthr, int bar_id,
                                          uint32_t gen0) {
  const int ly = blockIdx.y;
  const int K = p.groups[w.group].n_splits;
  if (t == 0) {
    // arrival: acq_rel atomic (releases this CTA's partial rows, ordered before it by the
    // CTA barrier and the fence); the last arriver resets the counter for the next launch
    // (relaxed: kernel boundaries order it) and releases the bumped generation
    uint32_t* c = reinterpret_cast<uint32_t*>(p.cm_tickets) + ((int64_t)ly * p.n_groups + w.group) * 2;
    __threadfence();
    uint32_t old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(c) : "memory");
    if (old == (uint32_t)K - 1) {
      asm volatile("st.relaxed.gpu.global.u32 [%0], 0;" ::"l"(c) : "memory");
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(c + 1), "r"(gen0 + 1u) : "memory");
    } else {
      while (ld_acquire_u32(c + 1) == gen0) {
      }
    }
  }
  asm volatile("barrier.sync %0, %1;" ::"r"(bar_id), "r"(nthr) : "memory");
  GTRACE_T(true, 11);
  if (K <= 8)
    gm_merge_items<8>(p, w, K, t, nthr);
  else if (K <= 16)
    gm_merge_items<16>(p, w, K, t, nthr);
  else
    gm_merge_items<24>(p, w, K, t, nthr);
}

// Group-split launches (AttnParams::cm_gsplit): the attention CTAs leave their partials
// (column-major float4 layout of cm_merge_rows) and exit; this grid, launched right
// behind with programmatic dependent launch (its CTAs need no shared memory and sit
// in griddepcontrol.wait while the attention grid drains), merges every group:
// block (g, b, layer) takes items b * 256 .. of group g -- (row, 4 columns), rows
// fastest within 8 -- with all K partial loads of an item in flight (R-11).
template <int KMAX>
__global__ void __launch_bounds__(256) gm_merge_kernel(const AttnParams p) {
  griddep_launch_dependents();
  const int g = blockIdx.x;
  const int ly = blockIdx.z;
  const Group gr = p.groups[g];
  const int K = gr.n_splits;
  const int G = p.G;
  const int rows = gr.q_ntok * G;
  const int it = blockIdx.y * 256 + threadIdx.x;
  const int row = (it & 7) + 8 * ((it >> 3) / (kD / 4));
  const int c = (it >> 3) % (kD / 4);
  const SegDesc sg = p.segs[gr.seg];
  griddep_wait();   // the attention grid's partials
  if (K <= 1 || row >= rows) return;
  const int64_t s0 = (int64_t)ly * p.n_units + gr.unit0;
  const float4* po = reinterpret_cast<const float4*>(p.part_o) + s0 * (kM * kD / 4);
  const float* pl = p.part_lse + s0 * kM;
  float lj[KMAX];
  float4 v[KMAX];
#pragma unroll
  for (int j = 0; j < KMAX; ++j)
    if (j < K) {
      lj[j] = __ldcg(pl + (int64_t)j * kM + row);
      v[j] = __ldcg(po + (int64_t)j * (kM * kD / 4) + c * kM + row);
    }
  float L = -CUDART_INF_F;
#pragma unroll
  for (int j = 0; j < KMAX; ++j)
    if (j < K) L = fmaxf(L, lj[j]);
  float ws = 0.f;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int j = 0; j < KMAX; ++j)
    if (j < K) {
      const float wt = lj[j] == -CUDART_INF_F ? 0.f : exp2f(lj[j] - L);
      ws += wt;
      acc.x = fmaf(wt, v[j].x, acc.x);
      acc.y = fmaf(wt, v[j].y, acc.y);
      acc.z = fmaf(wt, v[j].z, acc.z);
      acc.w = fmaf(wt, v[j].w, acc.w);
    }
  const float inv = ws > 0.f ? 1.f / ws : 0.f;
  const int64_t in_l = p.in_layer_stride ? (int64_t)ly * p.rows_per_layer : 0;
  const int64_t orow = in_l + sg.row0 + gr.q_tok0 + row / G;
  store_bf16x4(static_cast<__nv_bfloat16*>(p.O) + (orow * p.Hq + gr.kv_head * G + row % G) * kD + 4 * c,
               make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv));
}

// Groups spread over K > 1 clusters: merge the K block partials of every row
// (log-sum-exp, R-11) -- a small grid launched right behind the attention
// kernel (programmatic dependent launch: its prologue overlaps the attention
// kernel's tail).  Block b of layer y: group b / (32 / RW), rows 4 RW (b % (32 /
// RW)) .. +4 RW; warp wq takes RW of them (rows +wq, +wq+4, ...), lane l columns
// [4l, 4l+4) (coalesced 512-byte rows); loads of RW rows x 4 partials are in
// flight at once, with an online rescale over the partials.  RW = 8 (few CTAs, so
// most SMs stay free for the next grid's CTAs) for up to 8 partials, else 1.
template <int RW>
__global__ void __launch_bounds__(128) cm_merge_kernel(const AttnParams p) {
  griddep_launch_dependents();
  constexpr int kBlocksPerGroup = 32 / RW;
  const int g = blockIdx.x / kBlocksPerGroup;
  const Group gr = p.groups[g];
  const int K = gr.n_splits;
  const int G = p.G;
  const int rows = gr.q_ntok * G;
  const int r0 = (blockIdx.x % kBlocksPerGroup) * 4 * RW + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  const int ly = blockIdx.y;
  const int64_t s0 = (int64_t)ly * p.n_units + gr.unit0;
  const SegDesc sg = p.segs[gr.seg];
  griddep_wait();   // the attention grid's partials
  if (K <= 1 || r0 >= rows) return;
  constexpr int B = 4;
  float m[RW], wsum[RW];
  float4 acc[RW];
#pragma unroll
  for (int b = 0; b < RW; ++b) {
    m[b] = -CUDART_INF_F;
    wsum[b] = 0.f;
    acc[b] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  for (int j0 = 0; j0 < K; j0 += B) {
    float l[RW][B];
    float4 v[RW][B];
#pragma unroll
    for (int b = 0; b < RW; ++b)
#pragma unroll
      for (int jj = 0; jj < B; ++jj) {
        const int row = min(r0 + 4 * b, rows - 1);
        const int j = min(j0 + jj, K - 1);
        l[b][jj] = j0 + jj < K ? __ldcg(p.part_lse + (s0 + j) * kM + row) : -CUDART_INF_F;
        v[b][jj] = __ldcg(reinterpret_cast<const float4*>(p.part_o + ((s0 + j) * kM + row) * kD) + lane);
      }
#pragma unroll
    for (int b = 0; b < RW; ++b) {
      float mb = m[b];
#pragma unroll
      for (int jj = 0; jj < B; ++jj) mb = fmaxf(mb, l[b][jj]);
      if (mb == -CUDART_INF_F) continue;
      const float sc = m[b] == -CUDART_INF_F ? 0.f : exp2f(m[b] - mb);
      wsum[b] *= sc;
      acc[b] = make_float4(acc[b].x * sc, acc[b].y * sc, acc[b].z * sc, acc[b].w * sc);
#pragma unroll
      for (int jj = 0; jj < B; ++jj) {
        const float wt = l[b][jj] == -CUDART_INF_F ? 0.f : exp2f(l[b][jj] - mb);
        wsum[b] += wt;
        acc[b].x = fmaf(wt, v[b][jj].x, acc[b].x);
        acc[b].y = fmaf(wt, v[b][jj].y, acc[b].y);
        acc[b].z = fmaf(wt, v[b][jj].z, acc[b].z);
        acc[b].w = fmaf(wt, v[b][jj].w, acc[b].w);
      }
      m[b] = mb;
    }
  }
  const int64_t in_l = p.in_layer_stride ? (int64_t)ly * p.rows_per_layer : 0;
#pragma unroll
  for (int b = 0; b < RW; ++b) {
    const int row = r0 + 4 * b;
    if (row >= rows) break;
    const float inv = wsum[b] > 0.f ? 1.f / wsum[b] : 0.f;
    const int64_t orow = in_l + sg.row0 + gr.q_tok0 + row / G;
    __nv_bfloat16* out = static_cast<__nv_bfloat16*>(p.O) + (orow * p.Hq + gr.kv_head * G + row % G) * kD + 4 * lane;
    store_bf16x4(out, make_float4(acc[b].x * inv, acc[b].y * inv, acc[b].z * inv, acc[b].w * inv));
  }
}

// D[tmem] (+)= A[tmem] * B[smem desc]  (A = P, K-major in TMEM).
__device__ __forceinline__ void mma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

// Load-event index of (slot k, tile j): shared tiles are one event each; after
// them the two slots' private tiles interleave.
__device__ __forceinline__ int event_of(int k, int j, int nsh, int nt0, int nt1) {
  if (j < nsh) return j;
  const int jj = j - nsh;
  const int m = min(nt0, nt1) - nsh;
  return nsh + (jj < m ? 2 * jj + k : 2 * m + (jj - m));
}

template <bool F8>
__global__ void __launch_bounds__(kThreads, 1)
attn_tc_kernel(const AttnParams p, const __grid_constant__ TcMaps maps, const int box_rows) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* tiles = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  Bars& bar = *reinterpret_cast<Bars*>(tiles + kNumSlots * kSlotBytes);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int ly = blockIdx.y;
  GTRACE(threadIdx.x == 0, 0);
  // the next grid in the stream may be scheduled now (it waits in griddepcontrol.wait
  // before touching memory); its CTAs take SMs as this grid's CTAs exit
  griddep_launch_dependents();
#ifdef SSA_GTRACE
  if (threadIdx.x == 0 && blockIdx.x < kGtCtas) {
    uint32_t smid;
    asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
    g_gtrace[(p.layer0 + blockIdx.y) & 31][blockIdx.x][7] = smid;
  }
#endif
  const TcPair& pr = p.pairs[blockIdx.x];   // units, segments, split counts in one place
  const WorkUnit w0 = pr.wa;
  WorkUnit w1 = w0;
  int nt1 = 0;
  if (pr.ub >= 0) {
    w1 = pr.wb;
    nt1 = w1.tile_hi - w1.tile_lo;
  }
  const int nt0 = w0.tile_hi - w0.tile_lo;
  const int nsh = pr.ub >= 0 ? pr.n_shared : 0;
  const bool two_q = pr.ub >= 0 && !pr.same_q;
  // A split pair of a q tile with <= 32 live rows (e.g. a 1-token GQA query: 4 rows) loads
  // those rows twice, at rows 0.. and 32.., so slot 1 reads its live S rows from TMEM lane
  // quadrant 1 (warp 9, SM sub-partition 1) instead of sharing sub-partition 0's MUFU with
  // slot 0.  Rows 64-127 of the tile are padding.
  const bool dup = pr.ub >= 0 && pr.same_q && w0.q_ntok * p.G <= 32;
  // smem tile slots (7 x 32 KB): Q (1 or 2), a K ring of NK and a V ring of NV
  // stages.  K(e) is released by its S MMA, V(e) by its PV MMA, which run
  // about a tile later, so the rings and their producer warps progress
  // independently (K loads run further ahead).
  // CM CTA whose groups it holds alone (cluster of 1, one cluster per group): the
  // epilogue writes O straight from the slots, no exchange buffer / reduce
  const bool cm_direct = p.cm_C == 1 && pr.splits_a == 1 && (pr.ub < 0 || pr.splits_b == 1);
  // the epilogue stages rows in the ring (exchange buffer, or a split pair's slot merge)
  const bool ring_stage = p.cm_C > 0 && (!cm_direct || (pr.same_q && pr.ub >= 0));
  const int NK = 3;
  const int NV = two_q ? 2 : 3;
  uint8_t* q_buf[2] = {tiles, two_q ? tiles + kSlotBytes : tiles};
  uint8_t* k_base = tiles + (two_q ? 2 : 1) * kSlotBytes;
  uint8_t* v_base = k_base + NK * kSlotBytes;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&maps.q);
    tma_prefetch_desc(&maps.q32);
    tma_prefetch_desc(&maps.kt);
    tma_prefetch_desc(&maps.vt);
    tma_prefetch_desc(&maps.pk);
    tma_prefetch_desc(&maps.pv);
    mbar_init(&bar.q_full, 1);
    mbar_init(&bar.q_ready, 2);
    for (int s = 0; s < kMaxStages; ++s) {
      mbar_init(&bar.k_raw[s], 1);
      mbar_init(&bar.v_raw[s], 1);
      mbar_init(&bar.k_full[s], 1);
      mbar_init(&bar.v_full[s], 1);
      mbar_init(&bar.k_empty[s], 1);
      mbar_init(&bar.v_empty[s], 1);
    }
    for (int k = 0; k < 2; ++k) {
      mbar_init(&bar.s_full[k], 1);
      // one arrival per softmax warp that owns a live row of slot k (padding warps skip)
      const int rows_k = (k ? w1 : w0).q_ntok * p.G;
      const int roff_k = (dup && k == 1) ? 32 : 0;
      int live_warps = 0;
      for (int q = 0; q < 4; ++q) live_warps += (roff_k < 32 * q + 32 && roff_k + rows_k > 32 * q) ? 1 : 0;
      mbar_init(&bar.p_full[k], live_warps);
      mbar_init(&bar.o_final[k], 1);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(&bar.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bar.tmem_base;
  GTRACE(threadIdx.x == 0, 1);

  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegsWG0));
    if (F8 && (warp == 2 || warp == 3)) {
      // ----------------------------------------------------------- F8 converters
      // warp 2: Q tile 0 then the K ring; warp 3: Q tile 1 (two q tiles) then the V ring
      const bool is_k = warp == 2;
      mbar_wait(&bar.q_full, 0);
      if (is_k || two_q) convert_q_tile(smem_u32(is_k ? q_buf[0] : q_buf[1]), lane);
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar.q_ready);
      const int NR = is_k ? NK : NV;
      uint8_t* ring = is_k ? k_base : v_base;
      uint64_t* raw = is_k ? bar.k_raw : bar.v_raw;
      uint64_t* full = is_k ? bar.k_full : bar.v_full;
      const int E = nt0 + nt1 - nsh;
      for (int e = 0; e < E; ++e) {
        const int s = e % NR;
        mbar_wait(&raw[s], (e / NR) & 1);
        convert_kv_slot(smem_u32(ring + s * kSlotBytes), lane);
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&full[s]);
      }
    } else if (warp == 0 || (!F8 && warp == 3)) {
      // ----------------------------------------------------------- TMA producers
      // warp 0: Q and the K ring; warp 3: the V ring.  F8: warps 2-3 convert, so
      // lane 0 of warp 0 loads Q and the K ring and lane 1 the V ring (two
      // independent loops in one warp, so K loads run ahead of V as in bf16).
      if (F8 ? lane < 2 : elect_one()) {
        const int64_t head_base = (int64_t)(p.layer0 + ly) * p.num_pages;
        const int64_t in_l = p.in_layer_stride ? (int64_t)ly * p.rows_per_layer : 0;
        const bool is_k = F8 ? lane == 0 : warp == 0;
        const uint64_t pol = l2_policy_evict_first();
        // With a programmatic launch, warm L1 with both slots' first page-table entries
        // before waiting for the previous grid (page tables are written only by copies,
        // which a programmatic launch never overlaps).
        if (p.pool_early)
          for (int k = 0; k < (pr.ub >= 0 ? 2 : 1); ++k) {
            const WorkUnit& w = k ? w1 : w0;
            const SegDesc& sg = k ? pr.sb : pr.sa;
            if (w.tile_hi > w.tile_lo && w.tile_lo * kBN < sg.n_slots)
              asm volatile("prefetch.global.L1 [%0];" ::"l"(sg.pages + (w.tile_lo * kBN) / p.P));
          }
        const int E = nt0 + nt1 - nsh;
        const int m01 = min(nt0, nt1) - nsh;
        const int NR = is_k ? NK : NV;
        uint8_t* ring = is_k ? k_base : v_base;
        uint64_t* full = F8 ? (is_k ? bar.k_raw : bar.v_raw) : (is_k ? bar.k_full : bar.v_full);
        uint64_t* empty = is_k ? bar.k_empty : bar.v_empty;
        const CUtensorMap* pool_map = is_k ? &maps.pk : &maps.pv;
        const CUtensorMap* tail_map = is_k ? &maps.kt : &maps.vt;
        // load event e: (slot k, tile j) -- K or V tile into ring stage e % NR.  Returns
        // false (nothing issued) for a tail tile when only pool tiles may be loaded yet.
        // F8: codes, one 128-byte chunk per row, into the stage's upper half; the
        // converter warps signal k_full / v_full.
        auto issue = [&](int e, bool pool_only) -> bool {
          int k, j;
          if (e < nsh) { k = 0; j = e; }
          else if (e - nsh < 2 * m01) { k = (e - nsh) & 1; j = nsh + ((e - nsh) >> 1); }
          else { k = nt0 > nt1 ? 0 : 1; j = nsh + m01 + (e - nsh - 2 * m01); }
          const WorkUnit& w = k ? w1 : w0;
          const SegDesc& sg = k ? pr.sb : pr.sa;
          const int tile = w.tile_lo + j;
          const int n_pool_tiles = (sg.n_slots + kBN - 1) / kBN;
          if (pool_only && tile >= n_pool_tiles) return false;
          const int s = e % NR;
          if (e >= NR) mbar_wait_lazy(&empty[s], ((e / NR) - 1) & 1);
          uint8_t* dst = ring + s * kSlotBytes + (F8 ? kChunkBytes : 0);
          constexpr int nchunk = F8 ? 1 : 2;
          mbar_arrive_expect_tx(&full[s], nchunk * kChunkBytes);
          if (tile < n_pool_tiles) {
            const int key0 = tile * kBN;
            const int nb = kBN / box_rows;
            for (int b = 0; b < nb; ++b) {
              const int slot = key0 + b * box_rows;
              int32_t row = 0x7FFFFFF0;   // past the tensor -> TMA zero fill
              if (slot < sg.n_slots) {
                const int64_t page = __ldg(sg.pages + slot / p.P);
                row = (int32_t)(((head_base + page) * p.Hkv + w.kv_head) * p.P + (slot % p.P));
              }
              for (int c = 0; c < nchunk; ++c) {
                if (p.l2_evict_first)
                  tma_load_2d_hint(dst + c * kChunkBytes + b * box_rows * 128, pool_map, &full[s], c * 64, row, pol);
                else
                  tma_load_2d(dst + c * kChunkBytes + b * box_rows * 128, pool_map, &full[s], c * 64, row);
              }
            }
          } else {
            const int32_t krow = (int32_t)(in_l + sg.row0 + (tile - n_pool_tiles) * kBN);
            for (int c = 0; c < nchunk; ++c)
              tma_load_3d(dst + c * kChunkBytes, tail_map, &full[s], c * 64, w.kv_head, krow);
          }
          return true;
        };
        // With p.pool_early (the previous grid does not write the pool) the first ring
        // stages of pool tiles are issued before griddepcontrol.wait, so they land while
        // the previous layer finishes; Q and the tails (inputs) always come after it.
        int e0 = 0;
        if (p.pool_early)
          while (e0 < E && e0 < min(NR, SSA_EARLY_STAGES) && issue(e0, true)) ++e0;
        griddep_wait();
        if (is_k && dup) {
          mbar_arrive_expect_tx(&bar.q_full, 2 * 2 * 32 * 128);
          const int32_t qrow = (int32_t)(in_l + pr.sa.row0 + w0.q_tok0);
          for (int c = 0; c < 2; ++c)
            for (int rb = 0; rb < 2; ++rb)
              tma_load_3d(q_buf[0] + c * kChunkBytes + rb * 32 * 128, &maps.q32, &bar.q_full, c * 64,
                          w0.kv_head * p.G, qrow);
        } else if (is_k) {
          const int nq = two_q ? 2 : 1;
          mbar_arrive_expect_tx(&bar.q_full, nq * kSlotBytes);
          for (int k = 0; k < nq; ++k) {
            const WorkUnit& w = k ? w1 : w0;
            const int32_t qrow = (int32_t)(in_l + (k ? pr.sb : pr.sa).row0 + w.q_tok0);
            for (int c = 0; c < 2; ++c)
              tma_load_3d(q_buf[k] + c * kChunkBytes, &maps.q, &bar.q_full, c * 64, w.kv_head * p.G, qrow);
          }
        }
        for (int e = e0; e < E; ++e) (void)issue(e, false);
      }
    } else if (warp == 1) {
      // ----------------------------------------------------------- MMA issuer
      if (elect_one()) {
        constexpr uint32_t idesc_s = F8 ? idesc_f16(kM, kBN, 0, 0) : idesc_bf16(kM, kBN, 0, 0);   // Q, K K-major
        constexpr uint32_t idesc_o = F8 ? idesc_f16(kM, kD, 0, 1) : idesc_bf16(kM, kD, 0, 1);    // P (TMEM), V MN-major
        // descriptor bases; per-step offsets are compile-time adds on the 16-byte address field
        const uint64_t qd0 = sdesc_sw128(smem_u32(q_buf[0]), 16, 1024);
        const uint64_t qd1 = sdesc_sw128(smem_u32(q_buf[1]), 16, 1024);
        const uint64_t kd0 = sdesc_sw128(smem_u32(k_base), 16, 1024);
        const uint64_t vd0 = sdesc_sw128(smem_u32(v_base), kChunkBytes, 1024);
        constexpr uint64_t kStageStep = kSlotBytes >> 4;
        mbar_wait(F8 ? &bar.q_ready : &bar.q_full, 0);
        GTRACE(true, 2);
        tc_fence_after();
        const int jmax = max(nt0, nt1);
        // prologue: S(k, 0); then per j: PV(k, j) and S(k, j+1) for k = 0, 1
        for (int it = -1; it < jmax; ++it) {
#pragma unroll 1
          for (int k = 0; k < 2; ++k) {
            const int ntk = k ? nt1 : nt0;
            if (it >= 0 && it < ntk) {
              // ---- PV(k, it): O_k += P_k (TMEM) * V
              const int e = event_of(k, it, nsh, nt0, nt1);
              const int s = e % NV;
              mbar_wait(&bar.p_full[k], it & 1);
              TRACE(true, 2 + k, it, 0, clock64());
              mbar_wait(&bar.v_full[s], (e / NV) & 1);
              TRACE(true, 11, it, k, clock64());
              tc_fence_after();
              const uint64_t vd = vd0 + (uint64_t)s * kStageStep;
              const uint32_t o = tmem + 256u * k + 128u;
              const uint32_t pa = tmem + 256u * k;
#pragma unroll
              for (int kk = 0; kk < kBN / 16; ++kk)   // 16 keys = 2048 B down each 64-column V chunk
                mma_bf16_ts(o, pa + 8 * kk, vd + (uint64_t)((kk * 2048) >> 4), idesc_o, (it > 0 || kk > 0) ? 1u : 0u);
              // a shared stage is free after slot 1's PV, a private one after its own
              if (it >= nsh || k == 1) mma_commit(&bar.v_empty[s]);
              if (it == ntk - 1) mma_commit(&bar.o_final[k]);
            }
            const int jn = it + 1;
            if (jn < ntk) {
              // ---- S(k, jn) = Q_k K^T
              const int e = event_of(k, jn, nsh, nt0, nt1);
              const int s = e % NK;
              mbar_wait(&bar.k_full[s], (e / NK) & 1);
              GTRACE(e == 0, 3);
              TRACE(true, 10, jn, k, clock64());
              tc_fence_after();
              const uint64_t qd = k ? qd1 : qd0;
              const uint64_t kd = kd0 + (uint64_t)s * kStageStep;
              const uint32_t d = tmem + 256u * k;
#pragma unroll
              for (int kk = 0; kk < kD / 16; ++kk) {
                const uint64_t off = (uint64_t)(((kk >> 2) * kChunkBytes + (kk & 3) * 32) >> 4);
                mma_bf16_ss(d, qd + off, kd + off, idesc_s, kk > 0 ? 1u : 0u);
              }
              mma_commit(&bar.s_full[k]);
              if (jn >= nsh || k == 1) mma_commit(&bar.k_empty[s]);
              TRACE(true, 2 + k, jn, 1, clock64());
            }
          }
        }
      }
    }
    if (ring_stage) ring_free_arrive();
    if (p.cm_C > 0 && !cm_direct) {   // the two cluster barriers of the CM epilogue
      cm_sync(p.cm_C);
      cm_sync(p.cm_C);
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegsSoftmax));
    // ------------------------------------------------------------- softmax + epilogue
    const int k = (warp - 4) >> 2;                 // slot
    const bool active = (k == 0) || pr.ub >= 0;
    const WorkUnit w = k ? w1 : w0;
    const int nt = k ? nt1 : nt0;
    uint32_t gm_gen0 = 0;   // group-barrier generation (thread t == 0 of a merging group)
    if (active) {
      const SegDesc sg = k ? pr.sb : pr.sa;
      const int r = threadIdx.x - 128 - 128 * k;   // TMEM lane
      const int roff = (dup && k == 1) ? 32 : 0;    // tile row of this slot's first live row
      const int rr = r - roff;                      // row of the unit's q tile
      const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
      const uint32_t s_col = tmem + lane_base + 256u * k;
      const uint32_t o_col = s_col + 128u;
      const float c = p.scale_log2;
      const int G = p.G;
      const int tok = w.q_tok0 + (rr >= 0 ? rr : 0) / G;
      const int last_key = min(sg.tail_m - 1, p.fault == 2 ? tok - 1 : tok);   // own keys 0..tok (R-2)
      // rows >= q_ntok * G of the 128-row tile are padding (1-token GQA query: 4 live rows); a
      // warp whose 32 rows are all padding takes no part in the tile loop (p_full counts only
      // the live warps): no S loads, softmax, P stores or barrier polling.  Its P columns keep
      // stale values that only reach the O rows of its own (discarded) lanes.
      const bool warp_dead = !(roff < (warp & 3) * 32 + 32 && roff + w.q_ntok * G > (warp & 3) * 32);
      const int n_pool_tiles = (sg.n_slots + kBN - 1) / kBN;
      float m_run = -CUDART_INF_F;
      float l_run = 0.f;
      for (int j = 0; j < (warp_dead ? 0 : nt); ++j) {
        const int tile = w.tile_lo + j;
        const bool is_pool = tile < n_pool_tiles;
        const int key0 = (is_pool ? tile : tile - n_pool_tiles) * kBN;
        mbar_wait(&bar.s_full[k], j & 1);
        GTRACE(r == 0 && k == 0 && j == 0, 4);
        TRACE(r == 0, k, j, 0, clock64());
        tc_fence_after();
        {
        float sv[kBN];
        {
          uint32_t ra[32], rb[32], rc[32], rd[32];
          tmem_ld32(s_col + 0, ra);
          tmem_ld32(s_col + 32, rb);
          tmem_ld32(s_col + 64, rc);
          tmem_ld32(s_col + 96, rd);
          tmem_wait_ld();
          TRACE(r == 0, 4 + k, j, 0, clock64());
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            sv[i] = __uint_as_float(ra[i]);
            sv[32 + i] = __uint_as_float(rb[i]);
            sv[64 + i] = __uint_as_float(rc[i]);
            sv[96 + i] = __uint_as_float(rd[i]);
          }
        }
        bool need_mask;
        int lim, hlo = 0, hhi = 0;
        if (is_pool) {
          lim = sg.n_slots - key0;
          hlo = sg.hole_lo - key0;
          hhi = sg.hole_hi - key0;
          need_mask = lim < kBN || (hhi > 0 && hlo < kBN && hhi > hlo);
        } else {
          lim = last_key - key0 + 1;
          need_mask = lim < kBN;
        }
        if (__any_sync(0xffffffffu, need_mask)) {
#pragma unroll
          for (int i = 0; i < kBN; ++i) {
            const bool ok = i < lim && !(i >= hlo && i < hhi);
            sv[i] = ok ? sv[i] : -CUDART_INF_F;
          }
        }
        // row max: 8 independent 3-input max chains (FMNMX3), then a short tree
        float mx8[8];
#pragma unroll
        for (int c8 = 0; c8 < 8; ++c8) mx8[c8] = fmaxf(sv[c8], sv[c8 + 8]);
#pragma unroll
        for (int i = 16; i < kBN; i += 16)
#pragma unroll
          for (int c8 = 0; c8 < 8; ++c8) mx8[c8] = fmaxf(mx8[c8], fmaxf(sv[i + c8], sv[i + 8 + c8]));
        const float mt = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                               fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
        float alpha = 1.f;
        if (mt > m_run + kRescaleLog2 / c || m_run == -CUDART_INF_F) {
          const float m_new = fmaxf(m_run, mt);
          alpha = (m_run == -CUDART_INF_F) ? 0.f : ex2((m_run - m_new) * c);
          m_run = m_new;
        }
        const float mc = (m_run == -CUDART_INF_F) ? 0.f : m_run * c;
        TRACE(r == 0, 6 + k, j, 0, clock64());
        uint32_t pk[kBN / 2];
        float2 sum4[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                          make_float2(0.f, 0.f)};
        const float2 c2 = make_float2(c, c), nmc2 = make_float2(-mc, -mc);
#pragma unroll
        for (int i = 0; i < kBN / 2; ++i) {
          const float2 x = __ffma2_rn(make_float2(sv[2 * i], sv[2 * i + 1]), c2, nmc2);
          const float2 e = ((i & 7) >= 8 - kPolyPairsOf8) ? ex2_poly2(x) : make_float2(ex2(x.x), ex2(x.y));
          sum4[i & 3] = __fadd2_rn(sum4[i & 3], e);
          pk[i] = pack_p<F8>(e.x, e.y);
        }
        const float2 s01 = __fadd2_rn(sum4[0], sum4[1]), s23 = __fadd2_rn(sum4[2], sum4[3]);
        const float2 sum2 = __fadd2_rn(s01, s23);
        TRACE(r == 0, 4 + k, j, 1, clock64());
        l_run = l_run * alpha + (sum2.x + sum2.y);
        // O rescale (PV(j-1) completed: s_full(j) committed after it)
        if (j > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            uint32_t ro[32];
            tmem_ld32(o_col + q4 * 32, ro);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; i += 2) {
              const float2 v = __fmul2_rn(make_float2(__uint_as_float(ro[i]), __uint_as_float(ro[i + 1])),
                                          make_float2(alpha, alpha));
              ro[i] = __float_as_uint(v.x);
              ro[i + 1] = __float_as_uint(v.y);
            }
            tmem_st32(o_col + q4 * 32, ro);
          }
        }
        // P (bf16 pairs) into the first 64 columns of this slot's S region
        {
          uint32_t lo[32], hi[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) { lo[i] = pk[i]; hi[i] = pk[32 + i]; }
          tmem_st32(s_col + 0, lo);
          tmem_st32(s_col + 32, hi);
        }
        tmem_wait_st();
        }
        TRACE(r == 0, 6 + k, j, 1, clock64());
        tc_fence_before();
        __syncwarp();
        TRACE(r == 0, k, j, 1, clock64());
        TRACE(lane == 0 && k == 0 && (warp & 3) < 2, 8 + (warp & 3), j, 0, clock64());
        TRACE(lane == 0 && k == 1 && (warp & 3) < 2, 8 + (warp & 3), j, 1, clock64());
        if (lane == 0) mbar_arrive(&bar.p_full[k]);
      }
      // ----------------------------------------------------------- epilogue
      if (nt > 0) {
        mbar_wait(&bar.o_final[k], 0);
        GTRACE(r == 0 && k == 0, 5);
        GTRACE(r == 0 && k == 1, 14);
        tc_fence_after();
      }
      griddep_wait();   // before the first global write (O / partials of the previous grid's readers)
      // group-barrier launch: the arriving thread of this slot's group reads its generation now
      if (p.cm_gbar && (k ? pr.splits_b : pr.splits_a) > 1 && (threadIdx.x == 128 || (two_q && threadIdx.x == 256)))
        gm_gen0 = gm_generation(p, w.group);
      const float inv_l = (l_run > 0.f ? 1.f / l_run : 0.f) * (F8 ? p.o_scale : 1.f);   // F8: V scale
      const float lse = l_run > 0.f ? m_run * c + __log2f(l_run) : -CUDART_INF_F;
      const int h = w.kv_head * G + (rr >= 0 ? rr : 0) % G;
      const bool live = rr >= 0 && rr < w.q_ntok * G;
      const int64_t in_l = p.in_layer_stride ? (int64_t)ly * p.rows_per_layer : 0;
      const int64_t orow = in_l + sg.row0 + tok;
      const int unit = k ? pr.ub : pr.ua;
      const int64_t pslot = (int64_t)ly * p.n_units + unit;
      if (p.cm_C > 0) {
        // Cluster merge (CM launch): the ring becomes the exchange buffer of the q
        // tile(s) once every MMA of the CTA has completed; rows are left normalized
        // (fp32) with their lse and merged across the cluster after the CTA barrier.
        const int nt_o = k ? nt0 : nt1;
        if (pr.ub >= 0 && nt_o > 0) mbar_wait(&bar.o_final[k ^ 1], 0);
        tc_fence_after();
        if (ring_stage) ring_free_wait();
        float* X0 = reinterpret_cast<float*>(k_base);
        __nv_bfloat16* orow_ptr = static_cast<__nv_bfloat16*>(p.O) + (orow * p.Hq + h) * kD;
        // group-barrier launch, group over several CTAs: this slot's rows go to the
        // group's global partial `split` (merged after the group barrier, gm_reduce)
        float* gdst = nullptr;
        float* glse = nullptr;
        if ((p.cm_gbar || p.cm_gsplit) && !cm_direct && (k ? pr.splits_b : pr.splits_a) > 1) {
          const int64_t ps = (int64_t)ly * p.n_units + (k ? pr.unit0_b : pr.unit0_a) + w.split;
          gdst = p.part_o + ps * kM * kD;
          glse = p.part_lse + ps * kM;
        }
        if (pr.same_q && pr.ub >= 0 && !dup) {
          // split pair: slot 1 leaves its lse and 1/l, slot 0 merges both slots' O rows
          // straight from TMEM (R-11)
          if (k == 1 && live) {
            *x_lse(X0, rr) = l_run > 0.f ? lse : -CUDART_INF_F;
            *(x_lse(X0, rr) + kM) = inv_l;
          }
          GTRACE(threadIdx.x == 256, 15);
          asm volatile("barrier.sync 3, 256;" ::: "memory");
          if (k == 0)
            cm_merge_tmem(X0, rr, live, o_col, inv_l, lse, l_run > 0.f, cm_direct ? orow_ptr : nullptr, gdst,
                          glse ? glse + rr : nullptr);
          GTRACE_T(true, 8);
        } else if (pr.same_q && pr.ub >= 0) {
          // duplicated small q tile (slot 1's rows in lanes 32..): slot 1 stages its rows,
          // slot 0 merges them into its own (R-11)
          if (k == 1) cm_stage_rows(x_row(X0, rr), x_lse(X0, rr), live, o_col, inv_l, lse, l_run > 0.f);
          GTRACE(threadIdx.x == 256, 15);
          asm volatile("barrier.sync 3, 256;" ::: "memory");
          if (k == 0)
            cm_merge_rows(X0, rr, live, o_col, inv_l, lse, l_run > 0.f, cm_direct ? orow_ptr : nullptr, gdst,
                          glse ? glse + rr : nullptr);
          GTRACE_T(true, 8);
        } else if (cm_direct) {
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            uint32_t ro[32];
            tmem_ld32(o_col + q4 * 32, ro);
            tmem_wait_ld();
            if (live)
#pragma unroll
              for (int i = 0; i < 32; i += 8) {
                float v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) v[u] = l_run > 0.f ? __uint_as_float(ro[i + u]) * inv_l : 0.f;
                store_bf16x8(orow_ptr + q4 * 32 + i, v);
              }
          }
        } else if (gdst) {
          gm_stage_rows(reinterpret_cast<float4*>(gdst), glse, rr, live, o_col, inv_l, lse, l_run > 0.f);
        } else {
          float* Xk = X0 + (pr.same_q ? 0 : k) * kXFloats;
          cm_stage_rows(x_row(Xk, rr), x_lse(Xk, rr), live, o_col, inv_l, lse, l_run > 0.f);
        }
      } else {
#pragma unroll
      for (int q4 = 0; q4 < 4; ++q4) {
        uint32_t ro[32];
        tmem_ld32(o_col + q4 * 32, ro);
        tmem_wait_ld();
        if (live) {
          if (w.group < 0) {
            __nv_bfloat16* out = static_cast<__nv_bfloat16*>(p.O) + (orow * p.Hq + h) * kD + q4 * 32;
#pragma unroll
            for (int i = 0; i < 32; i += 8) {
              uint4 v;
              v.x = pack_bf16(__uint_as_float(ro[i + 0]) * inv_l, __uint_as_float(ro[i + 1]) * inv_l);
              v.y = pack_bf16(__uint_as_float(ro[i + 2]) * inv_l, __uint_as_float(ro[i + 3]) * inv_l);
              v.z = pack_bf16(__uint_as_float(ro[i + 4]) * inv_l, __uint_as_float(ro[i + 5]) * inv_l);
              v.w = pack_bf16(__uint_as_float(ro[i + 6]) * inv_l, __uint_as_float(ro[i + 7]) * inv_l);
              *reinterpret_cast<uint4*>(out + i) = v;
            }
          } else {
            float* out = p.part_o + (pslot * kM + rr) * kD + q4 * 32;
            const bool has = l_run > 0.f;
#pragma unroll
            for (int i = 0; i < 32; i += 4) {
              *reinterpret_cast<float4*>(out + i) =
                  has ? make_float4(__uint_as_float(ro[i]) * inv_l, __uint_as_float(ro[i + 1]) * inv_l,
                                    __uint_as_float(ro[i + 2]) * inv_l, __uint_as_float(ro[i + 3]) * inv_l)
                      : make_float4(0.f, 0.f, 0.f, 0.f);
            }
          }
        }
      }
      if (w.group >= 0 && live) p.part_lse[pslot * kM + rr] = lse;
      }   // !cm
    }
    if (!active && ring_stage) ring_free_arrive();
    if (p.cm_C > 0 && !cm_direct) {
      cm_sync(p.cm_C);   // every CTA of the cluster has staged its rows
      GTRACE_T(true, 9);
      const bool gm_k = p.cm_gbar && (k && two_q ? pr.splits_b : pr.splits_a) > 1;
      // group-split launch: the group's partial is written; gm_merge_kernel merges it
      const bool gs_k = p.cm_gsplit && (k && two_q ? pr.splits_b : pr.splits_a) > 1;
      if (gs_k) {
      } else if (gm_k) {
        // group-barrier merge: two q tiles -> warpgroup k merges slot k's group; a split
        // pair's single group is merged by both warpgroups
        const int t = threadIdx.x - 128 - (two_q ? 128 * k : 0);
        gm_reduce(p, two_q && k ? w1 : w0, t, two_q ? 128 : 256, two_q ? 1 + k : 3, gm_gen0);
      } else if (k < (two_q ? 2 : 1)) {
        const float* X = reinterpret_cast<const float*>(k_base) + k * kXFloats;
        const WorkUnit& wk = k ? w1 : w0;
        switch (p.cm_C) {
          case 1: cm_reduce<1>(p, wk, X, k); break;
          case 2: cm_reduce<2>(p, wk, X, k); break;
          case 3: cm_reduce<3>(p, wk, X, k); break;
          case 4: cm_reduce<4>(p, wk, X, k); break;
          case 5: cm_reduce<5>(p, wk, X, k); break;
          case 6: cm_reduce<6>(p, wk, X, k); break;
          case 7: cm_reduce<7>(p, wk, X, k); break;
          case 8: cm_reduce<8>(p, wk, X, k); break;
          default: cm_reduce<16>(p, wk, X, k); break;
        }
      }
      GTRACE_T(true, 12);
      cm_sync(p.cm_C);   // peers have finished reading this CTA's shared memory
      GTRACE_T(true, 13);
    }
  }
  tc_fence_before();
  __syncthreads();
  GTRACE(threadIdx.x == 0, 6);
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

}  // namespace

bool encode_bf16_map(CUtensorMap* m, const void* base, int rank, const cuuint64_t* dims,
                     const cuuint64_t* strides_bytes, const cuuint32_t* box) {
  EncodeTiledFn fn = get_encode();
  if (!fn) return false;
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(base), dims, strides_bytes, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

namespace {
bool encode(CUtensorMap* m, const void* base, int rank, const cuuint64_t* dims, const cuuint64_t* strides_bytes,
            const cuuint32_t* box) {
  return encode_bf16_map(m, base, rank, dims, strides_bytes, box);
}
// bf16, or uint8 (E4M3 codes) when u8; 128-byte swizzle either way
bool encode_map(CUtensorMap* m, const void* base, int rank, const cuuint64_t* dims, const cuuint64_t* strides_bytes,
                const cuuint32_t* box, bool u8) {
  if (!u8) return encode_bf16_map(m, base, rank, dims, strides_bytes, box);
  EncodeTiledFn fn = get_encode();
  if (!fn) return false;
  cuuint32_t es[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, rank, const_cast<void*>(base), dims, strides_bytes, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
}  // namespace

int tc_key_tile() { return kBN; }

int tc_debug_trace(void* host, size_t bytes) {
#if defined(SSA_GTRACE)
  if (bytes < sizeof(g_gtrace)) return -1;
  if (cudaMemcpyFromSymbol(host, g_gtrace, sizeof(g_gtrace)) != cudaSuccess) return -1;
  return (int)sizeof(g_gtrace);
#elif defined(SSA_TRACE)
  if (bytes < sizeof(g_trace)) return -1;
  if (cudaMemcpyFromSymbol(host, g_trace, sizeof(g_trace)) != cudaSuccess) return -1;
  return (int)sizeof(g_trace);
#else
  (void)host; (void)bytes;
  return 0;
#endif
}
int tc_rows_tile() { return kM; }
bool tc_supported_shape(int D, int G, bool bf16) {
  return bf16 && D == kD && G >= 1 && G <= 16 && (kM % G) == 0 && get_encode() != nullptr;
}

cudaError_t launch_attn_tc(const AttnParams& p, int n_layers, bool pdl, cudaStream_t s) {
  if (p.n_pairs == 0 || n_layers == 0) return cudaSuccess;
  if (!tc_supported_shape(p.D, p.G, true)) return cudaErrorNotSupported;
  TcMaps maps;
  const int G = p.G;
  const cuuint64_t rows = (cuuint64_t)p.rows_per_layer * (p.in_layer_stride ? n_layers : 1);
  {
    cuuint64_t dims[3] = {(cuuint64_t)kD, (cuuint64_t)p.Hq, rows};
    cuuint64_t str[2] = {(cuuint64_t)kD * 2, (cuuint64_t)p.Hq * kD * 2};
    cuuint32_t box[3] = {64, (cuuint32_t)G, (cuuint32_t)(kM / G)};
    if (!encode(&maps.q, p.Q, 3, dims, str, box)) return cudaErrorInvalidValue;
    cuuint32_t box32[3] = {64, (cuuint32_t)G, (cuuint32_t)(32 / G)};
    if (!encode(&maps.q32, p.Q, 3, dims, str, box32)) return cudaErrorInvalidValue;
  }
  // K/V element bytes: 2 (bf16) or 1 (E4M3 codes: a row of d = 128 codes is one 128-byte swizzle chunk)
  const int kvb = p.kv_fp8 ? 1 : 2;
  const bool u8 = p.kv_fp8 != 0;
  {
    cuuint64_t dims[3] = {(cuuint64_t)kD, (cuuint64_t)p.Hkv, rows};
    cuuint64_t str[2] = {(cuuint64_t)kD * kvb, (cuuint64_t)p.Hkv * kD * kvb};
    cuuint32_t box[3] = {(cuuint32_t)(128 / kvb), 1, (cuuint32_t)kBN};
    if (!encode_map(&maps.kt, p.Kt, 3, dims, str, box, u8)) return cudaErrorInvalidValue;
    if (!encode_map(&maps.vt, p.Vt, 3, dims, str, box, u8)) return cudaErrorInvalidValue;
  }
  const int box_rows = p.P < kBN ? p.P : kBN;
  {
    const cuuint64_t prow = (cuuint64_t)(p.layer0 + n_layers) * p.num_pages * p.Hkv * p.P;
    cuuint64_t dims[2] = {(cuuint64_t)kD, prow};
    cuuint64_t str[1] = {(cuuint64_t)kD * kvb};
    cuuint32_t box[2] = {(cuuint32_t)(128 / kvb), (cuuint32_t)box_rows};
    if (!encode_map(&maps.pk, p.poolK, 2, dims, str, box, u8)) return cudaErrorInvalidValue;
    if (!encode_map(&maps.pv, p.poolV, 2, dims, str, box, u8)) return cudaErrorInvalidValue;
  }
  auto kern = p.kv_fp8 ? attn_tc_kernel<true> : attn_tc_kernel<false>;
  cudaError_t e = tc_configure(p.kv_fp8 != 0);
  if (e != cudaSuccess) return e;
  if (p.cm_C > 1 && p.n_pairs % p.cm_C) return cudaErrorInvalidValue;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(p.n_pairs, n_layers, 1);
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = tc_smem_bytes();
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (p.cm_C > 1) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = (unsigned)p.cm_C;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  if (pdl) {
    // programmatic dependent launch: the CTA prologue (barriers, TMEM, descriptor and
    // page-id prefetch) overlaps the previous grid's tail; memory is touched only
    // after griddepcontrol.wait
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, kern, p, maps, box_rows);
}

cudaError_t launch_cm_merge(const AttnParams& p, int n_layers, int max_split, bool pdl, cudaStream_t s) {
  const int rw = max_split <= 8 ? 8 : 1;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(p.n_groups * (32 / rw), n_layers, 1);
  cfg.blockDim = dim3(128, 1, 1);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return rw == 8 ? cudaLaunchKernelEx(&cfg, cm_merge_kernel<8>, p) : cudaLaunchKernelEx(&cfg, cm_merge_kernel<1>, p);
}

cudaError_t launch_gm_merge(const AttnParams& p, int n_layers, int max_split, bool pdl, cudaStream_t s) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(p.n_groups, kM / 8, n_layers);   // blocks of 256 items: 8 rows x 32 column groups
  cfg.blockDim = dim3(256, 1, 1);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  if (max_split <= 8) return cudaLaunchKernelEx(&cfg, gm_merge_kernel<8>, p);
  if (max_split <= 16) return cudaLaunchKernelEx(&cfg, gm_merge_kernel<16>, p);
  if (max_split <= 32) return cudaLaunchKernelEx(&cfg, gm_merge_kernel<32>, p);
  return cudaErrorInvalidValue;
}

size_t tc_smem_bytes() { return (size_t)kNumSlots * kSlotBytes + sizeof(Bars) + 1024; }

// cudaFuncSetAttribute is per device: configure each (device, variant) once.
cudaError_t tc_configure(bool f8) {
  static std::mutex mu;
  static uint64_t done[2] = {0, 0};   // bit d: device d configured
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  if (dev < 64 && (done[f8 ? 1 : 0] >> dev) & 1) return cudaSuccess;
  auto kern = f8 ? attn_tc_kernel<true> : attn_tc_kernel<false>;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tc_smem_bytes());
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);   // clusters of 16
  if (e != cudaSuccess) return e;
  if (dev < 64) done[f8 ? 1 : 0] |= 1ull << dev;
  return cudaSuccess;
}

// Clusters of `c` CTAs (one per SM) that can be co-resident on the current device.
int tc_max_active_clusters(int c, bool f8) {
  if (tc_configure(f8) != cudaSuccess) return 0;
  auto kern = f8 ? attn_tc_kernel<true> : attn_tc_kernel<false>;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(c * 64, 1, 1);
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = tc_smem_bytes();
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)c;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

}  // namespace ssa
