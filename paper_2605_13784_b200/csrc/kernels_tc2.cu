// kernels_tc2.cu — data-plane attention on CTA pairs (tcgen05 cta_group::2), sm_100a.
//
// Same math as kernels_tc.cu (Eq. attention P:145 on the rows of Eq.
// query-attention P:150-155; causal tail, reading R-2; lazy running max,
// R-10), different schedule.  A cluster of two CTAs on one TPC runs two work
// units whose key tiles are the same keys (two q tiles of one append /
// stateless prompt over the same key range, plan.cpp pair_units_cta2):
//
//   * every tcgen05.mma is issued once, by CTA 0, with M = 256: rows 0-127 are
//     CTA 0's q tile, rows 128-255 CTA 1's, each in its own TMEM; the B
//     operand is split by N across the pair (K: keys 0-63 in CTA 0, 64-127 in
//     CTA 1; V: d-columns 0-63 / 64-127), so each SM stages half of every
//     K/V tile and the SS-MMA reads 96 B/clk of its SM's shared memory
//     instead of 128;
//   * with one q tile per SM, TMEM holds three S buffers (3 x 128 columns) and
//     O (128): the MMA order is S(0) S(1) S(2) PV(0) S(3) PV(1) ..., so S for
//     the next tiles is computed while the softmax works on S(j) and the
//     softmax runs back to back.  P(j) (bf16) overwrites the first 64 columns
//     of its S buffer and feeds PV(j) from TMEM.
//
// Warp roles (256 threads per CTA): warp 0 TMA producer (both CTAs: own Q, own
// halves of K and V, completing on CTA 0's barriers), warp 1 MMA issuer (CTA 0
// only), warp 2 TMEM allocator (both, cta_group::2), warps 4-11 softmax and
// epilogue for the CTA's 128 rows (two warpgroups splitting each S tile's
// columns).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include "sm100.cuh"
#include "store.h"

namespace ssa {

namespace {

using namespace sm100;

constexpr int kM = 128;                   // rows per CTA (TMEM lanes)
constexpr int kBN = 128;                  // keys per tile (pair)
constexpr int kHalf = 64;                 // keys (K) / d-columns (V) per CTA
constexpr int kD = 128;
constexpr int kThreads = 384;
constexpr int kQBytes = kM * kD * 2;      // 32 KB: own q tile, two 64-column swizzle chunks
constexpr int kKHalfBytes = kHalf * kD * 2;   // 16 KB: 64 keys x 128 d (two chunks of 8 KB)
constexpr int kVHalfBytes = kBN * kHalf * 2;  // 16 KB: 128 keys x 64 d (one chunk)
constexpr int kStages = 5;
constexpr int kStageBytes = kKHalfBytes + kVHalfBytes;
constexpr int kVLag = 2;                  // V loads trail K loads (S runs 2 tiles ahead of PV)
constexpr int kMaxPages = 1536;           // staged page ids per unit (6 KB of smem)
constexpr float kRescaleLog2 = 8.0f;
// exp2 offload: kPolyPairsOf8 of every 8 element pairs on the FMA pipe
// (sm100.cuh ex2_poly2), the rest on MUFU.  Here two softmax warps per SMSP
// keep MUFU busy, so moving part of the exps off it shortens the tile.
#ifndef SSA_TC2_POLY
#define SSA_TC2_POLY 2
#endif
constexpr int kPolyPairsOf8 = SSA_TC2_POLY;
#ifndef SSA_TC2_ALL_LANE_ARRIVE
#define SSA_TC2_ALL_LANE_ARRIVE 0
#endif
constexpr int kSBufs = 3;                      // S buffers at columns 0 / 128 / 256
constexpr uint32_t kColS0 = 0, kColO = 384;   // O at 384

struct Bars {
  uint64_t q_full;                 // CTA 0: both Q tiles landed
  uint64_t k_full[kStages];        // CTA 0: both K halves of the stage landed
  uint64_t v_full[kStages];        // CTA 0: both V halves landed
  uint64_t k_empty[kStages];       // both CTAs (multicast commit): K stage consumed by S
  uint64_t v_empty[kStages];       // both CTAs (multicast commit): V stage consumed by PV
  uint64_t s_full[kSBufs];         // both CTAs (multicast commit): S buffer b computed
  uint64_t p_full[kSBufs];         // CTA 0: P of buffer b written by all 16 softmax warps
  uint64_t o_final;                // both CTAs: last PV done
  uint32_t tmem_base;
};

struct Tc2Maps {
  CUtensorMap q;    // [rows][Hq][D]    box {64, G, 128/G}
  CUtensorMap kt;   // [rows][Hkv][D]   box {64, 1, 64}   (tail K half)
  CUtensorMap vt;   // [rows][Hkv][D]   box {64, 1, 128}  (tail V half: 128 keys, one d-chunk)
  CUtensorMap pk;   // [pool rows][D]   box {64, BR}
  CUtensorMap pv;
};

#ifdef SSA_TRACE
// clock64 timeline of the first CTA pairs of layer 5 (ssa_debug_trace): rows
// [rank][0] softmax S seen / P released, [rank][1] ld done / exps done,
// [0][2] issuer S(j) committed / P(j) seen.
constexpr int kTr2Ctas = 4, kTr2Tiles = 256, kTr2Layer = 5;
__device__ unsigned long long g_trace2[kTr2Ctas][2][4][kTr2Tiles][2];
#define TRACE2(cond, rank, row, j, w, val)                                                                     \
  do {                                                                                                         \
    if ((cond) && blockIdx.y == kTr2Layer && (blockIdx.x >> 1) < kTr2Ctas && (j) < kTr2Tiles)                  \
      g_trace2[blockIdx.x >> 1][rank][row][j][w] = (val);                                                      \
  } while (0)
#else
#define TRACE2(cond, rank, row, j, w, val) do { } while (0)
#endif

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
attn_tc2_kernel(const AttnParams p, const TcPair* __restrict__ pairs2, const __grid_constant__ Tc2Maps maps,
                const int box_rows) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* q_buf = base;
  uint8_t* k_ring = base + kQBytes;
  uint8_t* v_ring = k_ring + kStages * kKHalfBytes;
  Bars& bar = *reinterpret_cast<Bars*>(v_ring + kStages * kVHalfBytes);
  // row-max exchange between the two softmax halves: [tile parity][half][row]
  float (*red_max)[2][kM] = reinterpret_cast<float (*)[2][kM]>(reinterpret_cast<uint8_t*>(&bar) + 256);
  // page ids of the unit's pool tiles, staged once so the producer's TMA
  // coordinates do not wait on a dependent global load per box
  int32_t* pg = reinterpret_cast<int32_t*>(reinterpret_cast<uint8_t*>(red_max) + 2 * 2 * kM * sizeof(float));

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int ly = blockIdx.y;
  const TcPair pr = pairs2[blockIdx.x >> 1];
  const WorkUnit w = p.units[rank ? pr.ub : pr.ua];
  const int nt = w.tile_hi - w.tile_lo;          // identical for both CTAs (planner)

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&maps.q);
    tma_prefetch_desc(&maps.kt);
    tma_prefetch_desc(&maps.vt);
    tma_prefetch_desc(&maps.pk);
    tma_prefetch_desc(&maps.pv);
    mbar_init(&bar.q_full, 1);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&bar.k_full[s], 1);
      mbar_init(&bar.v_full[s], 1);
      mbar_init(&bar.k_empty[s], 1);
      mbar_init(&bar.v_empty[s], 1);
    }
    for (int b = 0; b < kSBufs; ++b) {
      mbar_init(&bar.s_full[b], 1);
      mbar_init(&bar.p_full[b], SSA_TC2_ALL_LANE_ARRIVE ? 16 * 32 : 16);
    }
    mbar_init(&bar.o_final, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc_pair<512>(&bar.tmem_base);
  const SegDesc sg0 = p.segs[w.seg];
  const int pg_lo = w.tile_lo * kBN / p.P;
  const int pg_n = min(kMaxPages, max(0, (min(sg0.n_slots, w.tile_hi * kBN) + p.P - 1) / p.P - pg_lo));
  if (warp == 0)
    for (int i = lane; i < pg_n; i += 32) pg[i] = __ldg(sg0.pages + pg_lo + i);
  tc_fence_before();
  cluster_sync_all();   // barriers of both CTAs initialised, TMEM allocated, page ids staged
  tc_fence_after();
  const uint32_t tmem = bar.tmem_base;

  if (warp == 0 || warp == 3) {
    // ------------------------------------------------------------- TMA producers
    // warp 0: Q and the K ring; warp 3: the V ring (independent progress)
    if (elect_one()) {
      const uint32_t q_full0 = mapa_shared(smem_u32(&bar.q_full), 0);
      const int64_t head_base = (int64_t)(p.layer0 + ly) * p.num_pages;
      const int64_t in_l = p.in_layer_stride ? (int64_t)ly * p.rows_per_layer : 0;
      const SegDesc sg = p.segs[w.seg];
      if (warp == 0 && rank == 0) mbar_arrive_expect_tx(&bar.q_full, 2 * kQBytes);
      if (warp == 0) {
        const int32_t qrow = (int32_t)(in_l + sg.row0 + w.q_tok0);
        for (int c = 0; c < 2; ++c)
          tma_load_3d_pair(q_buf + c * (kQBytes / 2), &maps.q, q_full0, c * 64, w.kv_head * p.G, qrow);
      }
      const int n_pool_tiles = (sg.n_slots + kBN - 1) / kBN;
      auto pool_row = [&](int slot) -> int32_t {
        if (slot >= sg.n_slots) return 0x7FFFFFF0;   // past the tensor -> TMA zero fill
        const int pi = slot / p.P - pg_lo;
        const int64_t page = pi < pg_n ? pg[pi] : __ldg(sg.pages + slot / p.P);
        return (int32_t)(((head_base + page) * p.Hkv + w.kv_head) * p.P + (slot % p.P));
      };
      // K ring and V ring: K(e) is released by S(e) (k_empty), V(e) by PV(e)
      // (v_empty).  S runs two tiles ahead of PV, so V loads trail K loads by
      // kVLag tiles and each ring keeps kStages tiles in flight.
      auto load_k = [&](int e) {
        const int s = e % kStages;
        if (e >= kStages) mbar_wait(&bar.k_empty[s], ((e / kStages) - 1) & 1);
        TRACE2(rank == 0, 1, 2, e, 0, clock64());
        uint8_t* kb = k_ring + s * kKHalfBytes;
        const uint32_t kf0 = mapa_shared(smem_u32(&bar.k_full[s]), 0);
        const int tile = w.tile_lo + e;
        if (rank == 0) mbar_arrive_expect_tx(&bar.k_full[s], 2 * kKHalfBytes);
        if (tile < n_pool_tiles) {
          // K half: keys [key0 + 64 rank, +64), both 64-column d-chunks
          const int key0 = tile * kBN + (int)rank * kHalf;
          for (int b = 0; b < kHalf / box_rows; ++b) {
            const int32_t row = pool_row(key0 + b * box_rows);
            for (int c = 0; c < 2; ++c)
              tma_load_2d_pair(kb + c * (kKHalfBytes / 2) + b * box_rows * 128, &maps.pk, kf0, c * 64, row);
          }
        } else {
          const int32_t trow = (int32_t)(in_l + sg.row0 + (tile - n_pool_tiles) * kBN);
          for (int c = 0; c < 2; ++c)
            tma_load_3d_pair(kb + c * (kKHalfBytes / 2), &maps.kt, kf0, c * 64, w.kv_head, trow + (int)rank * kHalf);
        }
      };
      auto load_v = [&](int e) {
        const int s = e % kStages;
        if (e >= kStages) mbar_wait(&bar.v_empty[s], ((e / kStages) - 1) & 1);
        TRACE2(rank == 0, 1, 2, e, 1, clock64());
        uint8_t* vb = v_ring + s * kVHalfBytes;
        const uint32_t vf0 = mapa_shared(smem_u32(&bar.v_full[s]), 0);
        const int tile = w.tile_lo + e;
        if (rank == 0) mbar_arrive_expect_tx(&bar.v_full[s], 2 * kVHalfBytes);
        if (tile < n_pool_tiles) {
          // V half: all 128 keys of the tile, d-chunk = rank
          for (int b = 0; b < kBN / box_rows; ++b) {
            const int32_t row = pool_row(tile * kBN + b * box_rows);
            tma_load_2d_pair(vb + b * box_rows * 128, &maps.pv, vf0, (int)rank * 64, row);
          }
        } else {
          const int32_t trow = (int32_t)(in_l + sg.row0 + (tile - n_pool_tiles) * kBN);
          tma_load_3d_pair(vb, &maps.vt, vf0, (int)rank * 64, w.kv_head, trow);
        }
      };
      if (warp == 0)
        for (int e = 0; e < nt; ++e) load_k(e);
      else
        for (int e = 0; e < nt; ++e) load_v(e);
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------- MMA issuer (CTA 0)
    if (rank == 0 && elect_one()) {
      constexpr uint32_t idesc_s = idesc_bf16(2 * kM, kBN, 0, 0);   // Q, K both K-major; M = 256 over the pair
      constexpr uint32_t idesc_o = idesc_bf16(2 * kM, kD, 0, 1);    // P K-major (TMEM), V MN-major
      const uint64_t qd = sdesc_sw128(smem_u32(q_buf), 16, 1024);
      const uint64_t kd0 = sdesc_sw128(smem_u32(k_ring), 16, 1024);
      const uint64_t vd0 = sdesc_sw128(smem_u32(v_ring), kVHalfBytes, 1024);
      constexpr uint64_t kKStep = (uint64_t)kKHalfBytes >> 4, kVStep = (uint64_t)kVHalfBytes >> 4;
      mbar_wait(&bar.q_full, 0);
      tc_fence_after();
      auto issue_s = [&](int j) {   // S(j) = Q K(j)^T into buffer j % 3
        const int s = j % kStages;
        mbar_wait(&bar.k_full[s], (j / kStages) & 1);
        TRACE2(true, 0, 3, j, 0, clock64());
        tc_fence_after();
        const uint64_t kd = kd0 + (uint64_t)s * kKStep;
        const uint32_t d = tmem + kColS0 + 128u * (uint32_t)(j % kSBufs);
#pragma unroll
        for (int kk = 0; kk < kD / 16; ++kk) {
          const uint64_t qoff = (uint64_t)(((kk >> 2) * (kQBytes / 2) + (kk & 3) * 32) >> 4);
          const uint64_t koff = (uint64_t)(((kk >> 2) * (kKHalfBytes / 2) + (kk & 3) * 32) >> 4);
          mma_pair_ss(d, qd + qoff, kd + koff, idesc_s, kk > 0 ? 1u : 0u);
        }
        mma_commit_pair(&bar.s_full[j % kSBufs]);
        mma_commit_pair(&bar.k_empty[s]);
        TRACE2(true, 0, 2, j, 0, clock64());
      };
      // S runs two tiles ahead of PV: S(j+2) goes to buffer (j+2)%3, which held
      // P(j-1), consumed by PV(j-1) issued before it (the tensor pipe executes in
      // order), so the softmax finds S(j+1) ready when it finishes tile j.
      if (nt > 0) issue_s(0);
      if (nt > 1) issue_s(1);
      for (int j = 0; j < nt; ++j) {
        if (j + 2 < nt) issue_s(j + 2);
        // ---- PV(j): O += P(j) (TMEM) * V(j)
        const int s = j % kStages;
        mbar_wait_cluster(&bar.p_full[j % kSBufs], (j / kSBufs) & 1);
        TRACE2(true, 0, 2, j, 1, clock64());
        mbar_wait(&bar.v_full[s], (j / kStages) & 1);
        TRACE2(true, 0, 3, j, 1, clock64());
        tc_fence_after();
        const uint64_t vd = vd0 + (uint64_t)s * kVStep;
        const uint32_t pa = tmem + kColS0 + 128u * (uint32_t)(j % kSBufs);
#pragma unroll
        for (int kk = 0; kk < kBN / 16; ++kk)   // 16 keys = 2048 B down the V half's 64-column chunk
          mma_pair_ts(tmem + kColO, pa + 8 * kk, vd + (uint64_t)((kk * 2048) >> 4), idesc_o, (j > 0 || kk > 0) ? 1u : 0u);
        mma_commit_pair(&bar.v_empty[s]);
        TRACE2(true, 1, 3, j, 0, clock64());
        if (j == nt - 1) mma_commit_pair(&bar.o_final);
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------- softmax + epilogue
    // Two warpgroups share the CTA's 128 rows (TMEM lanes): warps 4-7 take key
    // columns 0-63 of each S tile, warps 8-11 columns 64-127, so every SMSP runs
    // two softmax warps (MUFU latency hidden).  The row max is exchanged through
    // shared memory once per tile (named barrier 1, 256 threads); each half keeps
    // its own partial row sum, added in the epilogue.
    const SegDesc sg = p.segs[w.seg];
    const int hf = (warp - 4) >> 2;                   // column half
    const int r = (threadIdx.x - 128) & 127;          // row == TMEM lane
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t o_col = tmem + lane_base + kColO + 64u * (uint32_t)hf;   // this half's O columns
    const uint32_t p_full_c = rank ? mapa_shared(smem_u32(&bar.p_full[0]), 0) : 0;   // CTA 0's p_full[0]
    const float c = p.scale_log2;
    const int G = p.G;
    const int tok = w.q_tok0 + r / G;
    const int last_key = min(sg.tail_m - 1, p.fault == 2 ? tok - 1 : tok);   // own keys 0..tok (R-2)
    const int n_pool_tiles = (sg.n_slots + kBN - 1) / kBN;
    float m_run = -CUDART_INF_F;
    float l_run = 0.f;                                 // partial: this half's columns
    for (int j = 0; j < nt; ++j) {
      const int tile = w.tile_lo + j;
      const bool is_pool = tile < n_pool_tiles;
      const int key0 = (is_pool ? tile : tile - n_pool_tiles) * kBN + 64 * hf;
      const int buf = j % kSBufs;
      const uint32_t s_col = tmem + lane_base + kColS0 + 128u * (uint32_t)buf;
      bool need_mask;
      int lim, hlo = 0, hhi = 0;
      if (is_pool) {
        lim = sg.n_slots - key0;
        hlo = sg.hole_lo - key0;
        hhi = sg.hole_hi - key0;
        need_mask = lim < 64 || (hhi > 0 && hlo < 64 && hhi > hlo);
      } else {
        lim = last_key - key0 + 1;
        need_mask = lim < 64;
      }
      const bool any_mask = __any_sync(0xffffffffu, need_mask);
      TRACE2(r == 0 && hf == 0, rank, 1, j, 0, clock64());
      mbar_wait(&bar.s_full[buf], (j / kSBufs) & 1);
      TRACE2(r == 0 && hf == 0, rank, 0, j, 0, clock64());
      tc_fence_after();
      float sv[64];
      {
        uint32_t ra[32], rb[32];
        tmem_ld32(s_col + 64 * hf, ra);
        tmem_ld32(s_col + 64 * hf + 32, rb);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          sv[i] = __uint_as_float(ra[i]);
          sv[32 + i] = __uint_as_float(rb[i]);
        }
      }
      if (any_mask) {
#pragma unroll
        for (int i = 0; i < 64; ++i) {
          const bool ok = i < lim && !(i >= hlo && i < hhi);
          sv[i] = ok ? sv[i] : -CUDART_INF_F;
        }
      }
      float mx8[8];
#pragma unroll
      for (int c8 = 0; c8 < 8; ++c8) mx8[c8] = fmaxf(sv[c8], sv[c8 + 8]);
#pragma unroll
      for (int i = 16; i < 64; i += 16)
#pragma unroll
        for (int c8 = 0; c8 < 8; ++c8) mx8[c8] = fmaxf(mx8[c8], fmaxf(sv[i + c8], sv[i + 8 + c8]));
      const float mh = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                             fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
      // exchange the half-row maxima (double-buffered by tile parity, so one
      // barrier per tile suffices); the barrier also orders both halves' S loads
      // before either half writes P over columns 0-63
      red_max[j & 1][hf][r] = mh;
      asm volatile("bar.sync 1, 256;" ::: "memory");
      const float mt = fmaxf(mh, red_max[j & 1][hf ^ 1][r]);
      float alpha = 1.f;
      if (mt > m_run + kRescaleLog2 / c || m_run == -CUDART_INF_F) {
        const float m_new = fmaxf(m_run, mt);
        alpha = (m_run == -CUDART_INF_F) ? 0.f : ex2((m_run - m_new) * c);
        m_run = m_new;
      }
      // O rescale (this half's 64 columns) needs PV(j-1) complete: it committed
      // v_empty of its stage, whose latest possible completion is that PV (the
      // producer refills the stage only after it), so the parity is unambiguous.
      if (j > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {
        mbar_wait(&bar.v_empty[(j - 1) % kStages], ((j - 1) / kStages) & 1);
        tc_fence_after();
#pragma unroll
        for (int q2 = 0; q2 < 2; ++q2) {
          uint32_t ro[32];
          tmem_ld32(o_col + q2 * 32, ro);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; i += 2) {
            const float2 v = __fmul2_rn(make_float2(__uint_as_float(ro[i]), __uint_as_float(ro[i + 1])),
                                        make_float2(alpha, alpha));
            ro[i] = __float_as_uint(v.x);
            ro[i + 1] = __float_as_uint(v.y);
          }
          tmem_st32(o_col + q2 * 32, ro);
        }
      }
      const float mc = (m_run == -CUDART_INF_F) ? 0.f : m_run * c;
      uint32_t pk[32];
      float2 sum4[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                        make_float2(0.f, 0.f)};
      const float2 c2 = make_float2(c, c), nmc2 = make_float2(-mc, -mc);
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const float2 x = __ffma2_rn(make_float2(sv[2 * i], sv[2 * i + 1]), c2, nmc2);
        const float2 e = ((i & 7) >= 8 - kPolyPairsOf8) ? ex2_poly2(x) : make_float2(ex2(x.x), ex2(x.y));
        sum4[i & 3] = __fadd2_rn(sum4[i & 3], e);
        pk[i] = pack_bf16(e.x, e.y);
      }
      const float2 s01 = __fadd2_rn(sum4[0], sum4[1]), s23 = __fadd2_rn(sum4[2], sum4[3]);
      const float2 sum2 = __fadd2_rn(s01, s23);
      l_run = l_run * alpha + (sum2.x + sum2.y);
      TRACE2(r == 0 && hf == 0, rank, 1, j, 1, clock64());
      tmem_st32(s_col + 32 * hf, pk);   // P of keys 64hf..64hf+63 -> columns 32hf..32hf+31
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      TRACE2(r == 0 && hf == 0, rank, 0, j, 1, clock64());
#if SSA_TC2_ALL_LANE_ARRIVE
      // every lane arrives (no divergent branch for the warp to reconverge on)
      if (rank == 0) mbar_arrive(&bar.p_full[buf]);
      else mbar_arrive_remote(p_full_c + buf * (uint32_t)sizeof(uint64_t));
#else
      if (lane == 0) {
        if (rank == 0) mbar_arrive(&bar.p_full[buf]);
        else mbar_arrive_remote(p_full_c + buf * (uint32_t)sizeof(uint64_t));
      }
#endif
    }
    // ------------------------------------------------------------- epilogue
    red_max[0][hf][r] = l_run;                         // partial row sums
    if (nt > 0) {
      mbar_wait(&bar.o_final, 0);
      tc_fence_after();
    }
    asm volatile("bar.sync 1, 256;" ::: "memory");
    const float l_tot = l_run + red_max[0][hf ^ 1][r];
    const int rows = w.q_ntok * G;
    const float inv_l = l_tot > 0.f ? 1.f / l_tot : 0.f;
    const int h = w.kv_head * G + r % G;
    const int64_t in_l = p.in_layer_stride ? (int64_t)ly * p.rows_per_layer : 0;
    const int64_t orow = in_l + sg.row0 + tok;
    const int unit = rank ? pr.ub : pr.ua;
    const int64_t pslot = (int64_t)ly * p.n_units + unit;
#pragma unroll
    for (int q2 = 0; q2 < 2; ++q2) {
      uint32_t ro[32];
      tmem_ld32(o_col + q2 * 32, ro);
      tmem_wait_ld();
      const int col0 = 64 * hf + 32 * q2;
      if (r < rows) {
        if (w.group < 0) {
          __nv_bfloat16* out = static_cast<__nv_bfloat16*>(p.O) + (orow * p.Hq + h) * kD + col0;
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
          float* out = p.part_o + (pslot * kM + r) * kD + col0;
#pragma unroll
          for (int i = 0; i < 32; i += 4)
            *reinterpret_cast<float4*>(out + i) =
                make_float4(__uint_as_float(ro[i]) * inv_l, __uint_as_float(ro[i + 1]) * inv_l,
                            __uint_as_float(ro[i + 2]) * inv_l, __uint_as_float(ro[i + 3]) * inv_l);
        }
      }
    }
    if (hf == 0 && w.group >= 0 && r < rows)
      p.part_lse[pslot * kM + r] = l_tot > 0.f ? m_run * c + __log2f(l_tot) : -CUDART_INF_F;
  }
  tc_fence_before();
  cluster_sync_all();   // the pair's MMAs, TMA and remote arrives are all done
  tc_fence_after();
  if (warp == 2) tmem_dealloc_pair<512>(tmem);
}

}  // namespace

int tc2_debug_trace(void* host, size_t bytes) {
#ifdef SSA_TRACE
  if (bytes < sizeof(g_trace2)) return -1;
  if (cudaMemcpyFromSymbol(host, g_trace2, sizeof(g_trace2)) != cudaSuccess) return -1;
  return (int)sizeof(g_trace2);
#else
  (void)host; (void)bytes;
  return 0;
#endif
}

cudaError_t launch_attn_tc2(const AttnParams& p, const TcPair* d_pairs2, int n_pairs2, int n_layers, cudaStream_t s) {
  if (n_pairs2 == 0 || n_layers == 0) return cudaSuccess;
  if (!tc_supported_shape(p.D, p.G, true)) return cudaErrorNotSupported;
  Tc2Maps maps;
  const int G = p.G;
  const cuuint64_t rows = (cuuint64_t)p.rows_per_layer * (p.in_layer_stride ? n_layers : 1);
  {
    cuuint64_t dims[3] = {(cuuint64_t)kD, (cuuint64_t)p.Hq, rows};
    cuuint64_t str[2] = {(cuuint64_t)kD * 2, (cuuint64_t)p.Hq * kD * 2};
    cuuint32_t box[3] = {64, (cuuint32_t)G, (cuuint32_t)(kM / G)};
    if (!encode_bf16_map(&maps.q, p.Q, 3, dims, str, box)) return cudaErrorInvalidValue;
  }
  {
    cuuint64_t dims[3] = {(cuuint64_t)kD, (cuuint64_t)p.Hkv, rows};
    cuuint64_t str[2] = {(cuuint64_t)kD * 2, (cuuint64_t)p.Hkv * kD * 2};
    cuuint32_t boxk[3] = {64, 1, (cuuint32_t)kHalf};
    cuuint32_t boxv[3] = {64, 1, (cuuint32_t)kBN};
    if (!encode_bf16_map(&maps.kt, p.Kt, 3, dims, str, boxk)) return cudaErrorInvalidValue;
    if (!encode_bf16_map(&maps.vt, p.Vt, 3, dims, str, boxv)) return cudaErrorInvalidValue;
  }
  const int box_rows = p.P < kHalf ? p.P : kHalf;
  {
    const cuuint64_t prow = (cuuint64_t)(p.layer0 + n_layers) * p.num_pages * p.Hkv * p.P;
    cuuint64_t dims[2] = {(cuuint64_t)kD, prow};
    cuuint64_t str[1] = {(cuuint64_t)kD * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
    if (!encode_bf16_map(&maps.pk, p.poolK, 2, dims, str, box)) return cudaErrorInvalidValue;
    if (!encode_bf16_map(&maps.pv, p.poolV, 2, dims, str, box)) return cudaErrorInvalidValue;
  }
  static_assert(sizeof(Bars) <= 256, "Bars overlaps the row-max exchange");
  const size_t smem = (size_t)kQBytes + (size_t)kStages * (kKHalfBytes + kVHalfBytes) + 256 +
                      2 * 2 * kM * sizeof(float) + kMaxPages * sizeof(int32_t) + 1024;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(attn_tc2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  dim3 grid(2 * n_pairs2, n_layers);
  attn_tc2_kernel<<<grid, kThreads, smem, s>>>(p, d_pairs2, maps, box_rows);
  return cudaGetLastError();
}

}  // namespace ssa
