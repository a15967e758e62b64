// Microbenchmarks for the tcgen05 GEMM's two feeds, measured separately on one B200:
//   tma  : a persistent producer/consumer ring of TMA box loads (no MMA) -> bytes/clk/SM
//          for the operand box shapes the conv GEMMs use (2-D K-major tiles, 4-D NHWC
//          rectangles with 64 B or 128 B rows);
//   mma  : back-to-back tcgen05.mma.kind::tf32 from shared memory (no TMA) -> MAC/clk/SM
//          for M = 128 and N = 64 .. 256, committing per K block like the real kernel.
// Build: nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -I paper_1511_06051_b200/csrc
//        tools/tma_bench.cu -o tools/tma_bench -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "tc_gemm.cuh"

using namespace psg;

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess) {                                                          \
      std::fprintf(stderr, "%s: %s (%s:%d)\n", #x, cudaGetErrorString(e_), __FILE__, \
                   __LINE__);                                                         \
      std::exit(1);                                                                   \
    }                                                                                 \
  } while (0)

constexpr int kMaxStages = 32;

// mode 0: 2-D box {bc, br} at (k, row); mode 1: 4-D box {bc, bw, bh, 1} at (c, w, h, n)
struct TmaJob {
  int mode, bc, bw, bh, iters, bytes, stages, per_stage, producers, lanes;
  int cdim, wdim, hdim, ndim;  // coordinate ranges to walk
};

__global__ void __launch_bounds__(320, 1) tma_only(const __grid_constant__ CUtensorMap map, TmaJob j) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  __shared__ __align__(8) uint64_t full[kMaxStages], empty[kMaxStages];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < j.stages; ++s) {
      tc::mbar_init(tc::smem_u32(&full[s]), j.lanes ? 1 : j.producers);
      tc::mbar_init(tc::smem_u32(&empty[s]), 1);
    }
    tc::fence_barrier_init();
  }
  __syncthreads();
  if (j.lanes && warp == 2 && lane < j.producers) {
    // producers = lanes of one warp: lane 0 posts the stage's bytes, every lane issues
    if (lane == 0) tc::tma_prefetch(&map);
    const int mine = j.per_stage / j.producers;
    for (int it = 0; it < j.iters; ++it) {
      const int s = it % j.stages;
      tc::mbar_wait(tc::smem_u32(&empty[s]), ((it / j.stages) & 1) ^ 1);
      const uint32_t bar = tc::smem_u32(&full[s]);
      if (lane == 0) tc::mbar_arrive_expect_tx(bar, j.bytes * j.per_stage);
      __syncwarp((1u << j.producers) - 1);
      for (int q = lane * mine; q < (lane + 1) * mine; ++q) {
        const uint32_t dst = tc::smem_u32(smem + (s * j.per_stage + q) * j.bytes);
        const int t = blockIdx.x * 7919 + (it * j.per_stage + q) * 13;
        if (j.mode == 0)
          tc::tma_load_2d(dst, &map, bar, (t % j.cdim) * j.bc, ((t / j.cdim) % j.wdim) * j.bw);
        else
          tc::tma_load_4d(dst, &map, bar, (t % j.cdim) * j.bc, ((t / 3) % j.wdim) * j.bw - 2,
                          ((t / 7) % j.hdim) * j.bh - 2, (t / 11) % j.ndim);
      }
    }
  } else if (!j.lanes && warp >= 2 && warp < 2 + j.producers && lane == 0) {
    tc::tma_prefetch(&map);
    const int pw = warp - 2, mine = j.per_stage / j.producers;
    for (int it = 0; it < j.iters; ++it) {
      const int s = it % j.stages;
      tc::mbar_wait(tc::smem_u32(&empty[s]), ((it / j.stages) & 1) ^ 1);
      const uint32_t bar = tc::smem_u32(&full[s]);
      tc::mbar_arrive_expect_tx(bar, j.bytes * mine);
      for (int q = pw * mine; q < (pw + 1) * mine; ++q) {
        const uint32_t dst = tc::smem_u32(smem + (s * j.per_stage + q) * j.bytes);
        const int t = blockIdx.x * 7919 + (it * j.per_stage + q) * 13;
        if (j.mode == 0)
          tc::tma_load_2d(dst, &map, bar, (t % j.cdim) * j.bc, ((t / j.cdim) % j.wdim) * j.bw);
        else
          tc::tma_load_4d(dst, &map, bar, (t % j.cdim) * j.bc, ((t / 3) % j.wdim) * j.bw - 2,
                          ((t / 7) % j.hdim) * j.bh - 2, (t / 11) % j.ndim);
      }
    }
  } else if (warp == 1 && lane == 0) {
    for (int it = 0; it < j.iters; ++it) {
      const int s = it % j.stages;
      tc::mbar_wait(tc::smem_u32(&full[s]), (it / j.stages) & 1);
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(&empty[s]))
                   : "memory");
    }
  }
}

// Back-to-back MMAs: KB K blocks of KBLK (8-column steps), commit per K block.
__global__ void __launch_bounds__(128, 1) mma_only(int n, int kblk, int kblocks, int mn_major,
                                                   int nacc = 0) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  __shared__ __align__(8) uint64_t done, fin;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  // zero the operand tiles so the accumulators stay finite
  for (int i = threadIdx.x; i < (128 + 256) * kblk; i += blockDim.x)
    reinterpret_cast<float*>(smem)[i] = 0.f;
  if (threadIdx.x == 0) {
    tc::mbar_init(tc::smem_u32(&done), 1);
    tc::mbar_init(tc::smem_u32(&fin), 1);
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc(tc::smem_u32(&tbase), 512);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  if (warp == 0 && lane == 0) {
    const uint32_t sa = tc::smem_u32(smem), sb = sa + 128 * kblk * 4;
    const uint32_t idesc = tc::idesc_tf32(128, n, mn_major, mn_major);
    const uint32_t sw = kblk == 32 ? tc::kSw128 : tc::kSw64;
    for (int kb = 0; kb < kblocks; ++kb) {
      for (int q = 0; q < kblk / 8; ++q) {
        const uint64_t ad = mn_major ? tc::smem_desc(sa + q * 1024, kblk * 128, 512, tc::kSw128Base32)
                                     : tc::smem_desc(sa + q * 32, 16, 8 * kblk * 4, sw);
        const uint64_t bd = mn_major ? tc::smem_desc(sb + q * 1024, kblk * 128, 512, tc::kSw128Base32)
                                     : tc::smem_desc(sb + q * 32, 16, 8 * kblk * 4, sw);
        if (nacc)  // independent accumulators round robin (each K block -> acc kb % nacc)
          tc::mma_tf32(tbase + (kb % nacc) * n, ad, bd, idesc, q | (kb >= nacc));
        else
          tc::mma_tf32(tbase + (kb & 1) * 256, ad, bd, idesc, q | (kb > 1));
      }
      tc::mma_commit(tc::smem_u32(&done));  // per-K-block commit, as in the real kernel
    }
    tc::mma_commit(tc::smem_u32(&fin));
    tc::mbar_wait(tc::smem_u32(&fin), 0);  // all issued MMAs complete
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 1) {
    tc::fence_after_sync();
    tc::tmem_dealloc(tbase, 512);
  }
}

// Same loop with cta_group::2: a CTA pair computes M = 256 (128 rows of A per CTA) x N
// (N/2 columns of B per CTA); only the leader issues, the commit multicasts to both.
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    mma_pair(int n, int kblocks) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  __shared__ __align__(8) uint64_t fin;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  for (int i = threadIdx.x; i < (128 + 128) * 32; i += blockDim.x)
    reinterpret_cast<float*>(smem)[i] = 0.f;
  if (threadIdx.x == 0) {
    tc::mbar_init(tc::smem_u32(&fin), 1);
    tc::fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     tc::smem_u32(&tbase)), "r"(512) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc::fence_before_sync();
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  tc::fence_after_sync();
  if (rank == 0 && warp == 0 && lane == 0) {
    const uint32_t sa = tc::smem_u32(smem), sb = sa + 128 * 32 * 4;
    const uint32_t idesc = tc::idesc_tf32(256, n, false, false);
    for (int kb = 0; kb < kblocks; ++kb)
      for (int q = 0; q < 4; ++q) {
        const uint64_t ad = tc::smem_desc(sa + q * 32, 16, 1024, tc::kSw128);
        const uint64_t bd = tc::smem_desc(sb + q * 32, 16, 1024, tc::kSw128);
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(
                tbase + (kb & 1) * 256), "l"(ad), "l"(bd), "r"(idesc), "r"(uint32_t(q | (kb > 1)))
            : "memory");
      }
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
        ::"r"(tc::smem_u32(&fin)), "h"(uint16_t(3)) : "memory");
  }
  if (threadIdx.x == 0) tc::mbar_wait(tc::smem_u32(&fin), 0);
  tc::fence_before_sync();
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 1) {
    tc::fence_after_sync();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(512) : "memory");
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
}

int main() {
  int sms = 0, clk = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
  const double ghz = clk / 1e6;
  float* buf = nullptr;
  const size_t elems = size_t(1) << 28;  // 1 GiB
  CK(cudaMalloc(&buf, elems * 4));
  CK(cudaMemset(buf, 0, elems * 4));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  auto enc = encode();
  struct Case {
    const char* name;
    int mode, bc, bw, bh, C;  // C: channels (4-D) or columns (2-D)
    CUtensorMapSwizzle sw;
  };
  const Case cases[] = {
      {"2d_k32_rows128_sw128", 0, 32, 128, 1, 4096, CU_TENSOR_MAP_SWIZZLE_128B},
      {"2d_k16_rows128_sw64", 0, 16, 128, 1, 4096, CU_TENSOR_MAP_SWIZZLE_64B},
      {"4d_c32_32x4_C256", 1, 32, 32, 4, 256, CU_TENSOR_MAP_SWIZZLE_128B},
      {"4d_c16_32x4_C96", 1, 16, 32, 4, 96, CU_TENSOR_MAP_SWIZZLE_64B},
      {"4d_c32_16x8_C384", 1, 32, 16, 8, 384, CU_TENSOR_MAP_SWIZZLE_128B},
      {"2d_mn32_rows32_sw128b32", 0, 32, 32, 1, 4096, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B},
  };
  for (int lanes : {0})
  for (int prod : {1, 2, 4, 8})
  for (int per : {2, 4, 8})
  for (int stages : {3, 6})
  for (const Case& c : cases) {
    CUtensorMap m;
    uint32_t estr[5] = {1, 1, 1, 1, 1};
    TmaJob j{};
    j.mode = c.mode;
    j.bc = c.bc;
    j.bw = c.bw;
    j.bh = c.bh;
    j.iters = 4000;
    j.bytes = c.bc * c.bw * c.bh * 4;
    j.stages = stages;
    j.per_stage = per;
    j.producers = prod;
    j.lanes = lanes;
    if (per % prod) continue;
    if (size_t(stages) * per * j.bytes > 200 * 1024) continue;
    if (c.mode == 0) {
      const uint64_t rows = elems / c.C;
      const uint64_t dims[2] = {uint64_t(c.C), rows};
      const uint64_t str[1] = {uint64_t(c.C) * 4};
      const uint32_t box[2] = {uint32_t(c.bc), uint32_t(c.bw)};
      if (enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, buf, dims, str, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, c.sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
        std::printf("{\"case\": \"%s\", \"error\": \"encode\"}\n", c.name);
        continue;
      }
      j.cdim = c.C / c.bc;
      j.wdim = int(std::min<uint64_t>(rows, 2048) / c.bw);  // ~32 MB window: L2-resident
    } else {
      const int W = 27, H = 27;
      const uint64_t n = elems / (uint64_t(c.C) * W * H);
      const uint64_t dims[4] = {uint64_t(c.C), W, H, n};
      const uint64_t str[3] = {uint64_t(c.C) * 4, uint64_t(c.C) * W * 4, uint64_t(c.C) * W * H * 4};
      const uint32_t box[4] = {uint32_t(c.bc), uint32_t(c.bw), uint32_t(c.bh), 1};
      if (enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, buf, dims, str, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, c.sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
        std::printf("{\"case\": \"%s\", \"error\": \"encode\"}\n", c.name);
        continue;
      }
      j.cdim = c.C / c.bc;
      j.wdim = (W + c.bw - 1) / c.bw;
      j.hdim = (H + c.bh - 1) / c.bh;
      j.ndim = int(std::min<uint64_t>(n, 48));  // L2-resident window
    }
    const size_t smem = size_t(stages) * per * j.bytes + 1024;
    CK(cudaFuncSetAttribute(tma_only, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    tma_only<<<sms, 320, smem>>>(m, j);
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0));
    tma_only<<<sms, 320, smem>>>(m, j);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    const double bytes = double(sms) * j.iters * j.bytes * per;
    std::printf("{\"case\": \"%s\", \"stages\": %d, \"per_stage\": %d, \"producers\": %d, \"lanes\": %d, \"box_bytes\": %d, \"TB_per_s\": %.2f, \"B_per_clk_per_sm\": %.1f}\n",
                c.name, stages, per, prod, lanes, j.bytes, bytes / (ms * 1e-3) / 1e12, bytes / (ms * 1e-3) / (ghz * 1e9) / sms);
  }
  if (std::getenv("MMA_BENCH") == nullptr) return 0;
  for (int mn = 0; mn < 2; ++mn)
    for (int kblk : {16, 32})
      for (int n : {64, 128, 192, 256}) {
        if (mn && kblk != 32) continue;
        const int kblocks = 4000;
        const size_t smem = size_t(128 + 256) * kblk * 4 + 2048;
        CK(cudaFuncSetAttribute(mma_only, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        mma_only<<<sms, 128, smem>>>(n, kblk, 10, mn);
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(e0));
        mma_only<<<sms, 128, smem>>>(n, kblk, kblocks, mn);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        const double macs = double(sms) * kblocks * 128.0 * n * kblk;
        std::printf("{\"case\": \"mma_tf32_m128_n%d_k%d_%s\", \"TFLOPs\": %.1f, \"MAC_per_clk_per_sm\": %.0f}\n",
                    n, kblk, mn ? "mn" : "k", 2 * macs / (ms * 1e-3) / 1e12,
                    macs / (ms * 1e-3) / (ghz * 1e9) / sms);
      }
  for (int n : {64, 128, 256})
    for (int nacc : {1, 2, 4, 8}) {
      if (n * nacc > 512) continue;
      const int kblocks = 4000;
      const size_t smem = size_t(128 + 256) * 32 * 4 + 2048;
      CK(cudaFuncSetAttribute(mma_only, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
      mma_only<<<sms, 128, smem>>>(n, 32, 10, 0, nacc);
      CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(e0));
      mma_only<<<sms, 128, smem>>>(n, 32, kblocks, 0, nacc);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      const double macs = double(sms) * kblocks * 128.0 * n * 32;
      std::printf("{\"case\": \"mma_tf32_m128_n%d_k32_k_acc%d\", \"TFLOPs\": %.1f, \"MAC_per_clk_per_sm\": %.0f}\n",
                  n, nacc, 2 * macs / (ms * 1e-3) / 1e12, macs / (ms * 1e-3) / (ghz * 1e9) / sms);
    }
  for (int n : {64, 128, 256}) {
    const int kblocks = 4000, grid = sms / 2 * 2;
    const size_t smem = size_t(256) * 32 * 4 + 2048;
    CK(cudaFuncSetAttribute(mma_pair, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    mma_pair<<<grid, 128, smem>>>(n, 10);
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0));
    mma_pair<<<grid, 128, smem>>>(n, kblocks);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    const double macs = double(grid / 2) * kblocks * 256.0 * n * 32;
    std::printf("{\"case\": \"mma_tf32_pair_m256_n%d_k32\", \"TFLOPs\": %.1f, \"MAC_per_clk_per_sm\": %.0f}\n",
                n, 2 * macs / (ms * 1e-3) / 1e12, macs / (ms * 1e-3) / (ghz * 1e9) / grid);
  }
  return 0;
}
