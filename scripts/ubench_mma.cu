// Micro-benchmark (not part of the library): tcgen05.mma issue-to-completion
// throughput for the attention kernels' shapes on one SM (cta_group::1,
// M128 N128 K16) and on a CTA pair (cta_group::2, M256 N128 K16), SS (A and B
// from shared memory) and TS (A from TMEM).  Cycles per MMA from clock64.
#include <cstdint>
#include <cstdio>

#include "../paper_2605_13784_b200/csrc/sm100.cuh"

using namespace ssa::sm100;

constexpr int kRounds = 512;   // rounds of 8 MMAs (K = 128)

template <bool kPair, bool kTS, int kLdWarps, bool kBulk = false, int kN = 128>
__global__ void __launch_bounds__(256, 1) mma_bench(long long* out, const uint8_t* gsrc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* a = base;                 // 128 x 128 bf16, two 64-column chunks (32 KB)
  uint8_t* b = base + 32768;         // 128 (or 64 per CTA) x 128 bf16 (32 KB)
  __shared__ uint64_t done, bulk_bar;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(base)[i] = 0;
  fence_proxy_async_smem();
  uint32_t rank = 0;
  if (kPair) rank = cluster_ctarank();
  if (threadIdx.x == 0) {
    mbar_init(&bulk_bar, 1);
    mbar_init(&done, 1);
    fence_mbar_init();
  }
  if (warp == 0) {
    if (kPair) tmem_alloc_pair<512>(&tmem_base);
    else tmem_alloc<512>(&tmem_base);
  }
  tc_fence_before();
  if (kPair) cluster_sync_all(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;
  long long t0 = 0, t1 = 0;
  if (warp == 1 && rank == 0 && elect_one()) {
    const uint32_t M = kPair ? 256 : 128;
    const uint32_t idesc = idesc_bf16(M, kN, 0, kTS ? 1 : 0);
    const uint64_t ad = sdesc_sw128(smem_u32(a), 16, 1024);
    const uint64_t bd = sdesc_sw128(smem_u32(b), 16, 1024);
    t0 = clock64();
    for (int r = 0; r < kRounds; ++r) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint64_t off = (uint64_t)(((kk >> 2) * 16384 + (kk & 3) * 32) >> 4);
        const uint64_t offb = (uint64_t)(((kk >> 2) * (kN * 128) + (kk & 3) * 32) >> 4);
        if (kTS) {
          if (kPair) mma_pair_ts(tmem + 256, tmem + 8 * kk, bd + (uint64_t)((kk * 2048) >> 4), idesc, 1u);
          else asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem + 256),
              "r"(tmem + 8 * kk), "l"(bd + (uint64_t)((kk * 2048) >> 4)), "r"(idesc));
        } else {
          if (kPair) mma_pair_ss(tmem, ad + off, bd + off, idesc, 1u);
          else mma_bf16_ss(tmem, ad + off, bd + offb, idesc, 1u);
        }
      }
    }
    if (kPair) mma_commit_pair(&done); else mma_commit(&done);
    mbar_wait(&done, 0);
    t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  } else if (kPair && warp == 1 && rank == 1) {
    mbar_wait(&done, 0);
  } else if (kBulk && warp == 2 && elect_one()) {
    // TMA-like traffic: 32 KB bulk copies global -> a third smem region, back to back
    uint8_t* dst = base + 65536;
    for (int it = 0; it < kRounds / 2; ++it) {
      mbar_arrive_expect_tx(&bulk_bar, 32768);
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       smem_u32(dst)), "l"(gsrc + (size_t)((blockIdx.x * 977 + it * 131) % 4096) * 32768), "r"(32768),
                   "r"(smem_u32(&bulk_bar))
                   : "memory");
      mbar_wait(&bulk_bar, it & 1);
    }
  } else if (warp >= 4 && warp < 4 + kLdWarps) {
    // softmax-like TMEM readers: 128 columns of a region the MMAs do not touch
    const uint32_t lb = (uint32_t)((warp & 3) * 32) << 16;
    uint32_t acc = 0;
    for (int it = 0; it < kRounds * 6; ++it) {
      uint32_t r0[32], r1[32], r2[32], r3[32];
      tmem_ld32(tmem + lb + 384, r0);
      tmem_ld32(tmem + lb + 416, r1);
      tmem_ld32(tmem + lb + 448, r2);
      tmem_ld32(tmem + lb + 480, r3);
      tmem_wait_ld();
      acc += r0[it & 31] + r1[3] + r2[5] + r3[7];
      if (it % 4 == 0) { tmem_st32(tmem + lb + 384, r0); tmem_st32(tmem + lb + 416, r1); tmem_wait_st(); }
    }
    if (acc == 0x12345678) out[255] = acc;
  }
  tc_fence_before();
  if (kPair) cluster_sync_all(); else __syncthreads();
  if (warp == 0) {
    if (kPair) tmem_dealloc_pair<512>(tmem);
    else tmem_dealloc<512>(tmem);
  }
}

template <bool kPair, bool kTS, int kLd = 0, bool kBulk = false, int kN = 128>
void run(const char* name, long long* d, const uint8_t* g) {
  auto k = mma_bench<kPair, kTS, kLd, kBulk, kN>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(kPair ? 2 * 74 : 148);
  cfg.blockDim = dim3(kLd ? 256 : 128);
  cfg.dynamicSmemBytes = 100 * 1024;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kPair ? 2 : 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  for (int rep = 0; rep < 3; ++rep) cudaLaunchKernelEx(&cfg, k, d, g);
  cudaError_t e = cudaDeviceSynchronize();
  long long c = 0;
  cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  printf("%-28s %s: %.1f cycles per MMA (floor 64)\n", name, cudaGetErrorString(e), (double)c / (kRounds * 8));
}

int main() {
  long long* d;
  cudaMalloc(&d, 256 * 8);
  uint8_t* g;
  cudaMalloc(&g, (size_t)4096 * 32768);
  cudaMemset(g, 0, (size_t)4096 * 32768);
  run<false, false>("1-CTA SS M128N128K16", d, g);
  run<false, false, 0, false, 256>("1-CTA SS M128N256K16 (floor 128)", d, g);
  run<false, false, 0, false, 64>("1-CTA SS M128N64K16 (floor 32)", d, g);
  run<false, true>("1-CTA TS M128N128K16", d, g);
  run<true, false>("2-CTA SS M256N128K16", d, g);
  run<true, true>("2-CTA TS M256N128K16", d, g);
  run<false, false, 4>("1-CTA SS + 4 TMEM readers", d, g);
  run<false, true, 4>("1-CTA TS + 4 TMEM readers", d, g);
  run<true, false, 4>("2-CTA SS + 4 TMEM readers", d, g);
  run<true, true, 4>("2-CTA TS + 4 TMEM readers", d, g);
  run<false, false, 0, true>("1-CTA SS + bulk copies", d, g);
  run<true, false, 0, true>("2-CTA SS + bulk copies", d, g);
  run<false, false, 4, true>("1-CTA SS + readers + bulk", d, g);
  run<true, false, 4, true>("2-CTA SS + readers + bulk", d, g);
  return 0;
}
