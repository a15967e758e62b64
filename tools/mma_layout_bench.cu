// Microbenchmark for the halo-reuse implicit-GEMM idea: can a kind::tf32 MMA read its A
// operand from a no-swizzle K-major "halo" (rows 16 B apart, so a tap's row shift is a
// start-address offset), and what does an MMA cost per layout / N, alone and with a
// concurrent bulk-copy stream writing shared memory (the TMA producer's traffic)?
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/mlb tools/mma_layout_bench.cu -lcuda
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "../paper_1511_06051_b200/csrc/tc_gemm.cuh"

using namespace psg::tc;

constexpr int kHR = 288;               // halo rows
constexpr int kK = 32;                 // K floats per block
constexpr int kLBO = kHR * 16;         // no-swizzle: K-adjacent core matrices
constexpr int kABytes = kHR * kK * 4;  // 36 KB (both layouts fit)
constexpr int kBBytes = 256 * kK * 4;  // 32 KB
constexpr int kScratch = 64 * 1024;    // bulk-copy landing zone

struct Cfg {
  int a_layout;  // 0 = SW128 K-major (128 rows), 1 = no-swizzle halo
  int n;
  int shift;
  int iters;
  int copy;      // 1 = a second warp streams bulk copies into smem during the MMAs
  int swap_lbo;  // descriptor experiment: swap LBO / SBO for the no-swizzle layout
  int commit_every = 0;  // pair bench: tcgen05.commit after every this many K=32 blocks
};

__device__ __forceinline__ uint32_t sw128_off(int r, int k) {
  return (r / 8) * 1024 + (r % 8) * 128 + ((((k / 4) ^ (r % 8)) & 7) * 16) + (k % 4) * 4;
}

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes,
                                         uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}

__global__ void __launch_bounds__(128) k_bench(Cfg c, const float* A, const float* B, float* D,
                                               long long* cyc, unsigned long long* copied,
                                               const float* big) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~1023ull);
  __shared__ uint32_t tmem_sh;
  __shared__ __align__(8) uint64_t bar_done, bar_copy;
  __shared__ volatile int stop;
  const int tid = threadIdx.x, warp = tid / 32;
  uint8_t* sa = smem;
  uint8_t* sb = smem + kABytes;
  uint8_t* sc = sb + kBBytes;
  // fill A
  for (int i = tid; i < kHR * kK; i += blockDim.x) {
    const int r = i / kK, k = i % kK;
    const float v = A[i];
    if (c.a_layout == 0) {
      const int rr = r - c.shift;
      if (rr >= 0 && rr < 128) *reinterpret_cast<float*>(sa + sw128_off(rr, k)) = v;
    } else {
      *reinterpret_cast<float*>(sa + (k / 4) * kLBO + r * 16 + (k % 4) * 4) = v;
    }
  }
  for (int i = tid; i < 256 * kK; i += blockDim.x)
    *reinterpret_cast<float*>(sb + sw128_off(i / kK, i % kK)) = B[i];
  if (warp == 0) tmem_alloc(smem_u32(&tmem_sh), 256);
  if (tid == 0) {
    mbar_init(smem_u32(&bar_done), 1);
    mbar_init(smem_u32(&bar_copy), 1);
    stop = 0;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  fence_barrier_init();
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tmem = tmem_sh;
  if (warp == 1 && c.copy) {
    if (elect_one()) {
      unsigned long long bytes = 0;
      uint32_t ph = 0;
      const uint32_t b = smem_u32(&bar_copy);
      int i = 0;
      while (!stop) {
        mbar_arrive_expect_tx(b, kScratch);
        for (int q = 0; q < kScratch / 16384; ++q)
          bulk_g2s(smem_u32(sc) + q * 16384, big + ((i * 4 + q) % 4096) * 4096, 16384, b);
        mbar_wait(b, ph);
        ph ^= 1;
        bytes += kScratch;
        ++i;
      }
      copied[blockIdx.x] = bytes;
    }
  } else if (warp == 0) {
    const uint32_t idesc = idesc_tf32(128, c.n, false, false);
    uint64_t ad;
    uint32_t astep;
    if (c.a_layout == 0) {
      ad = smem_desc(smem_u32(sa), 16, 1024, kSw128);
      astep = 32 >> 4;
    } else {
      ad = c.swap_lbo ? smem_desc(smem_u32(sa) + c.shift * 16, 128, kLBO, kSwNone)
                      : smem_desc(smem_u32(sa) + c.shift * 16, kLBO, 128, kSwNone);
      astep = (2 * kLBO) >> 4;
    }
    const uint64_t bd = smem_desc(smem_u32(sb), 16, 1024, kSw128);
    __syncwarp();
    long long t0 = clock64();
    if (elect_one()) {
      for (int it = 0; it < c.iters; ++it) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          mma_tf32(tmem, ad + j * astep, bd + j * 2, idesc, (it | j) != 0 ? 1u : 0u);
      }
      mma_commit(smem_u32(&bar_done));
    }
    __syncwarp();
    mbar_wait(smem_u32(&bar_done), 0);
    long long t1 = clock64();
    if (tid == 0) {
      cyc[blockIdx.x] = t1 - t0;
      stop = 1;
    }
  }
  __syncthreads();
  fence_after_sync();
  if (blockIdx.x == 0) {
    for (int c0 = 0; c0 < c.n; c0 += 32) {
      uint32_t r[32];
      tmem_ld32_async(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c0, r);
      tmem_wait_ld();
      const int row = warp * 32 + (tid % 32);
      for (int j = 0; j < 32 && c0 + j < c.n; ++j) D[row * c.n + c0 + j] = __uint_as_float(r[j]);
    }
  }
  fence_before_sync();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 256);
}

// cta_group::2 pairs: each CTA holds its 128 A rows and half of B's N rows; the leader
// issues M = 256 MMAs.  Timing only (the numerics of the pair path are covered by the
// library's own parity tests).
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256)
    k_bench_pair(Cfg c, const float* A, const float* B, long long* cyc,
                 const __grid_constant__ CUtensorMap cmap, long long crow, int issuers,
                 int tmem_readers, unsigned long long* copied) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~1023ull);
  __shared__ uint32_t tmem_sh;
  __shared__ __align__(8) uint64_t bar_done;
  const int tid = threadIdx.x, warp = tid / 32;
  const uint32_t rank = cluster_rank();
  uint8_t* sa = smem;
  uint8_t* sb = smem + kABytes;
  for (int i = tid; i < kHR * kK; i += blockDim.x) {
    const int r = i / kK, k = i % kK;
    if (c.a_layout == 0) {
      if (r < 128) *reinterpret_cast<float*>(sa + sw128_off(r, k)) = A[i];
    } else {
      *reinterpret_cast<float*>(sa + (k / 4) * kLBO + r * 16 + (k % 4) * 4) = A[i];
    }
  }
  for (int i = tid; i < 128 * kK; i += blockDim.x)
    *reinterpret_cast<float*>(sb + sw128_off(i / kK, i % kK)) = B[i];
  __shared__ __align__(8) uint64_t cbars[4][2];
  __shared__ volatile int stop;
  if (warp == 0) tmem_alloc_pair(smem_u32(&tmem_sh), 512);
  if (tid == 0) {
    mbar_init(smem_u32(&bar_done), 1);
    for (int w = 0; w < 4; ++w)
      for (int i = 0; i < 2; ++i) mbar_init(smem_u32(&cbars[w][i]), 1);
    stop = 0;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  fence_barrier_init();
  fence_before_sync();
  cluster_sync();
  fence_after_sync();
  const uint32_t tmem = tmem_sh;
  if (warp == 0 && rank == 0) {
    const uint32_t idesc = idesc_tf32(256, c.n, false, false);
    uint64_t ad;
    uint32_t astep;
    if (c.a_layout == 0) {
      ad = smem_desc(smem_u32(sa), 16, 1024, kSw128);
      astep = 32 >> 4;
    } else {
      ad = smem_desc(smem_u32(sa) + c.shift * 16, kLBO, 128, kSwNone);
      astep = (2 * kLBO) >> 4;
    }
    const uint64_t bd = smem_desc(smem_u32(sb), 16, 1024, kSw128);
    __syncwarp();
    long long t0 = clock64();
    if (elect_one()) {
      for (int it = 0; it < c.iters; ++it) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          mma_tf32_pair(tmem, ad + j * astep, bd + j * 2, idesc, (it | j) != 0 ? 1u : 0u);
        if (c.commit_every && (it + 1) % c.commit_every == 0)
          mma_commit_pair(smem_u32(&cbars[3][1]), 1);
      }
      mma_commit_pair(smem_u32(&bar_done), 1);
    }
    __syncwarp();
    mbar_wait(smem_u32(&bar_done), 0);
    long long t1 = clock64();
    if (tid == 0) cyc[blockIdx.x / 2] = t1 - t0;
  }
  __syncwarp();
  if (warp == 0 && tid == 0 && rank == 0) {
    // tell both CTAs' helpers to stop (the peer polls its own flag)
    stop = 1;
    uint32_t peer = mapa(smem_u32(const_cast<int*>(&stop)), 1);
    asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(peer), "r"(1) : "memory");
  }
  if (warp >= 1 && warp <= 4 && warp - 1 < issuers && (tid % 32) == 0) {
    // TMA producer stand-in: 2 x 16 KB SW128 tiles in flight per issuer
    const int w = warp - 1;
    const uint32_t base = smem_u32(smem) + kABytes + kBBytes + w * 32768;
    unsigned long long bytes = 0;
    for (int i = 0;; ++i) {
      const int sl = i & 1;
      const uint32_t b = smem_u32(&cbars[w][sl]);
      if (i >= 2) mbar_wait(b, ((i >> 1) - 1) & 1);
      if (stop) {
        if (i >= 1) mbar_wait(smem_u32(&cbars[w][(i - 1) & 1]), ((i - 1) >> 1) & 1);
        break;
      }
      const long long ch = (static_cast<long long>(blockIdx.x) * 7919 + w * 131 + i * 1184LL) % crow;
      mbar_arrive_expect_tx(b, 16384);
      tma_load_2d(base + sl * 16384, &cmap, b, 0, static_cast<int>(ch * 128));
      bytes += 16384;
    }
    copied[blockIdx.x * 4 + w] = bytes;
  }
  __syncwarp();
  if (warp >= 4 && warp < 4 + tmem_readers) {
    // epilogue stand-in: read the other accumulator (columns 256..511) in a loop
    const uint32_t lane_base = static_cast<uint32_t>((warp % 4) * 32) << 16;
    uint32_t r[32], acc = 0;
    while (!stop) {
      for (int c0 = 256; c0 < 512; c0 += 32) {
        tmem_ld32_async(tmem + lane_base + c0, r);
        tmem_wait_ld();
        acc += r[0] + r[31];
      }
    }
    if (acc == 0x12345678) cyc[4096 - 1] = acc;
  }
  __syncwarp();
  fence_before_sync();
  __syncthreads();
  cluster_sync();
  fence_after_sync();
  if (warp == 0) tmem_dealloc_pair(tmem, 512);
}

// L2 / HBM -> shared memory inbound ceiling: every CTA keeps `depth` 16 KB bulk copies in
// flight over a source region of `region` floats (L2-resident or HBM-streaming).
__global__ void __launch_bounds__(32) k_copy(const float* big, long long region, int iters,
                                             int depth, long long* cyc, int same_src) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t bars[16];
  const uint32_t base = smem_u32(smem_raw);
  if (threadIdx.x == 0) {
    for (int i = 0; i < depth; ++i) mbar_init(smem_u32(&bars[i]), 1);
    fence_barrier_init();
  }
  __syncwarp();
  if (threadIdx.x != 0) return;
  const long long chunks = region / 4096;
  long long t0 = clock64();
  for (int i = 0; i < iters + depth; ++i) {
    const int s = i % depth;
    if (i >= depth) mbar_wait(smem_u32(&bars[s]), ((i / depth) - 1) & 1);
    if (i < iters) {
      const long long ch = same_src ? (i % chunks)
                                    : (static_cast<long long>(blockIdx.x) * 7919 + i * 148LL) % chunks;
      mbar_arrive_expect_tx(smem_u32(&bars[s]), 16384);
      bulk_g2s(base + s * 16384, big + ch * 4096, 16384, smem_u32(&bars[s]));
    }
  }
  cyc[blockIdx.x] = clock64() - t0;
}

// Multiple issuers per CTA: warps 0..nw-1 each keep `depth` loads of 16 KB in flight in their
// own ring; mode 0 = bulk copies, 1 = tiled 2D TMA (32 floats x 128 rows, SW128), 2 = the
// same tiled loads as 4 boxes of 32 rows (4 KB).
__global__ void __launch_bounds__(256) k_copy_multi(const __grid_constant__ CUtensorMap map,
                                                   const float* big, long long rows, int iters,
                                                   int depth, int nw, int mode, long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~1023ull);
  __shared__ __align__(8) uint64_t bars[8][8];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int w = 0; w < nw; ++w)
      for (int i = 0; i < depth; ++i) mbar_init(smem_u32(&bars[w][i]), 1);
    fence_barrier_init();
  }
  __syncthreads();
  // mode >= 10: the issuers are lanes 0..nw-1 of warp 0 (mode - 10 = box mode)
  const bool lanes = mode >= 10;
  const int who = lanes ? lane : warp;
  if (lanes ? (warp != 0 || lane >= nw) : (warp >= nw || lane != 0)) return;
  if (lanes) mode -= 10;
  const uint32_t base = smem_u32(smem) + who * depth * 16384;
  const long long chunks = rows / 128;
  long long t0 = clock64();
  for (int i = 0; i < iters + depth; ++i) {
    const int s = i % depth;
    const uint32_t b = smem_u32(&bars[who][s]);
    if (i >= depth) mbar_wait(b, ((i / depth) - 1) & 1);
    if (i < iters) {
      const long long ch =
          (static_cast<long long>(blockIdx.x) * 7919 + who * 131 + i * 1184LL) % chunks;
      mbar_arrive_expect_tx(b, 16384);
      if (mode == 0) {
        bulk_g2s(base + s * 16384, big + ch * 4096, 16384, b);
      } else if (mode == 1) {
        tma_load_2d(base + s * 16384, &map, b, 0, static_cast<int>(ch * 128));
      } else if (mode == 2) {
        for (int q = 0; q < 4; ++q)
          tma_load_2d(base + s * 16384 + q * 4096, &map, b, 0, static_cast<int>(ch * 128 + q * 32));
      } else {  // 64-byte rows: two 16-float x 128-row boxes (SW64)
        for (int q = 0; q < 2; ++q)
          tma_load_2d(base + s * 16384 + q * 8192, &map, b, q * 16, static_cast<int>(ch * 128));
      }
    }
  }
  if (who == 0) cyc[blockIdx.x] = clock64() - t0;
}

// Multicast bandwidth without a consumer protocol: per round every CTA expects 512 KB on
// one barrier; its 4 issuer warps fire 8 boxes each (mc = 0: all 32 boxes loaded locally;
// mc = 1: box b is read once by CTA b % CS and multicast to the whole cluster).  Slots are
// overwritten freely (nobody reads the data); a CTA's own round ends when its 512 KB landed.
template <int CS>
__global__ void __launch_bounds__(128) k_copy_mc2(const __grid_constant__ CUtensorMap map,
                                                   long long chunks, int rounds, int mc,
                                                   long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~1023ull);
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = cluster_rank();
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar), 1);
    fence_barrier_init();
  }
  cluster_sync();
  const long long cl = blockIdx.x / CS;
  long long t0 = clock64();
  for (int r = 0; r < rounds; ++r) {
    if (threadIdx.x == 0) mbar_arrive_expect_tx(smem_u32(&bar), 32 * 16384);
    __syncthreads();
    if (lane == 0) {
      for (int q = 0; q < 8; ++q) {
        const int b = warp * 8 + q;
        const long long ch = (cl * 7919 + (r * 32 + b) * 1184LL + (mc ? 0 : rank * 77)) % chunks;
        const uint32_t dst = smem_u32(smem) + (b % 4) * 16384;
        if (mc) {
          if (b % CS == static_cast<int>(rank)) {
            const uint16_t mask = static_cast<uint16_t>((1u << CS) - 1);
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
                " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst),
                "l"(reinterpret_cast<uint64_t>(&map)), "r"(0), "r"(static_cast<int>(ch * 128)),
                "r"(smem_u32(&bar)), "h"(mask)
                : "memory");
          }
        } else {
          tma_load_2d(dst, &map, smem_u32(&bar), 0, static_cast<int>(ch * 128));
        }
      }
    }
    if (threadIdx.x == 0) mbar_wait(smem_u32(&bar), r & 1);
    __syncthreads();
  }
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
  cluster_sync();
}

int main(int argc, char** argv) {
  setvbuf(stdout, nullptr, _IONBF, 0);
  const bool only_mc2 = argc > 1 && std::string(argv[1]) == "mc2";
  int dev_sms = 0;
  cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, 0);
  std::vector<float> hA(kHR * kK), hB(256 * kK);
  srand(1);
  for (auto& v : hA) v = static_cast<float>(rand() % 5 - 2);
  for (auto& v : hB) v = static_cast<float>(rand() % 5 - 2);
  float *dA, *dB, *dD, *big;
  long long* dc;
  unsigned long long* dcp;
  cudaMalloc(&dA, hA.size() * 4);
  cudaMalloc(&dB, hB.size() * 4);
  cudaMalloc(&dD, 128 * 256 * 4);
  cudaMalloc(&big, 4096ull * 4096 * 4 + 65536);
  cudaMemset(big, 0, 4096ull * 4096 * 4 + 65536);
  cudaMalloc(&dc, 4096 * 8);
  cudaMalloc(&dcp, dev_sms * 8);
  cudaMemcpy(dA, hA.data(), hA.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB.data(), hB.size() * 4, cudaMemcpyHostToDevice);
  const int smem = kABytes + kBBytes + kScratch + 1024;
  cudaFuncSetAttribute(k_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);

  auto run = [&](Cfg c, int grid, double* cyc_per_mma, double* copy_bpc) {
    cudaMemset(dD, 0xff, 128 * 256 * 4);
    cudaMemset(dcp, 0, dev_sms * 8);
    k_bench<<<grid, 128, smem>>>(c, dA, dB, dD, dc, dcp, big);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("error %s\n", cudaGetErrorString(e));
      exit(1);
    }
    std::vector<long long> hc(grid);
    std::vector<unsigned long long> hcp(grid);
    cudaMemcpy(hc.data(), dc, grid * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(hcp.data(), dcp, grid * 8, cudaMemcpyDeviceToHost);
    double s = 0, b = 0;
    for (int i = 0; i < grid; ++i) {
      s += hc[i];
      b += static_cast<double>(hcp[i]) / hc[i];
    }
    *cyc_per_mma = s / grid / (c.iters * 4.0);
    *copy_bpc = b / grid;
    std::vector<float> hD(128 * c.n);
    cudaMemcpy(hD.data(), dD, hD.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < c.n; ++n) {
        double ref = 0;
        for (int k = 0; k < kK; ++k) ref += hA[(m + c.shift) * kK + k] * hB[n * kK + k];
        ref *= c.iters;
        if (hD[m * c.n + n] != static_cast<float>(ref)) ++bad;
      }
    return bad;
  };
  double cpm, bpc;
  if (!only_mc2) {
  printf("# correctness (iters=1)\n");
  for (int lay = 0; lay < 2; ++lay)
    for (int sw = 0; sw < (lay ? 2 : 1); ++sw)
      for (int sh : {0, 1, 5, 37, 159})
        for (int n : {48, 128}) {
          Cfg c{lay, n, sh, 1, 0, sw};
          int bad = run(c, 1, &cpm, &bpc);
          printf("layout=%d swap=%d shift=%3d n=%3d bad=%d\n", lay, sw, sh, n, bad);
        }
  printf("# throughput: cycles per MMA (M=128, K=8), %d CTAs\n", dev_sms);
  for (int copy = 0; copy < 2; ++copy)
    for (int lay = 0; lay < 2; ++lay)
      for (int n : {32, 48, 64, 96, 128, 192, 256}) {
        Cfg c{lay, n, lay ? 7 : 0, 4096, copy, 0};
        int bad = run(c, dev_sms, &cpm, &bpc);
        const double ideal = 128.0 * n * 8 * 2 / 4096.0;
        printf("copy=%d layout=%d n=%3d cyc/mma=%7.1f ideal=%6.1f frac=%.3f smem_rd_B/clk=%.1f "
               "copy_B/clk=%.1f bad=%d\n",
               copy, lay, n, cpm, ideal, ideal / cpm, (4096.0 + n * 32.0) / cpm, bpc, bad);
      }
  }
  {
    printf("# multi-issuer inbound ceiling, 148 CTAs, L2-resident 16 MB source\n");
    float* src;
    const long long rows = (1ll << 22) / 32;  // 16 MB
    cudaMalloc(&src, rows * 128);
    cudaMemset(src, 0, rows * 128);
    CUtensorMap map;
    cuuint64_t dims[2] = {32, static_cast<cuuint64_t>(rows)};
    cuuint64_t strides[1] = {128};
    cuuint32_t box[2] = {32, 128}, box4[2] = {32, 32}, es[2] = {1, 1};
    CUtensorMap map4;
    cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, src, dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cuTensorMapEncodeTiled(&map4, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, src, dims, strides, box4, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    CUtensorMap map16;
    cuuint32_t box16[2] = {16, 128};
    cuTensorMapEncodeTiled(&map16, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, src, dims, strides, box16, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaFuncSetAttribute(k_copy_multi, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (!only_mc2)
    for (int grid : {37, 148})
    for (int mode : {1, 3, 11, 13})
      for (int nw : {1, 2, 4})
        for (int depth : {2}) {
          if (nw * depth * 16384 + 1024 > 200 * 1024) continue;
          const int iters = 1000;
          const CUtensorMap& m = (mode % 10) == 2 ? map4 : (mode % 10) == 3 ? map16 : map;
          cudaEvent_t e0, e1;
          cudaEventCreate(&e0);
          cudaEventCreate(&e1);
          k_copy_multi<<<grid, 256, nw * depth * 16384 + 1024>>>(m, src, rows, 100, depth, nw, mode, dc);
          cudaEventRecord(e0);
          k_copy_multi<<<grid, 256, nw * depth * 16384 + 1024>>>(m, src, rows, iters, depth, nw, mode, dc);
          cudaEventRecord(e1);
          if (cudaDeviceSynchronize() != cudaSuccess) { printf("multi launch failed\n"); return 1; }
          float ms;
          cudaEventElapsedTime(&ms, e0, e1);
          const double bytes = static_cast<double>(grid) * nw * iters * 16384.0;
          printf("grid=%d mode=%d issuers=%d depth=%d aggregate=%.0f GB/s per-SM=%.1f B/clk@1.9GHz\n", grid, mode, nw,
                 depth, bytes / (ms * 1e6), bytes / (ms * 1e-3) / grid / 1.9e9);
        }
    printf("# multicast2: delivered bytes per SM (512 KB per CTA per round)\n");
    for (int cs : {1, 2})  // (4-CTA clusters with multicast hung in this harness)
      for (int mc : {0, 1}) {
        if (cs == 1 && mc) continue;
        const int rounds = 200;
        const size_t sm = 4 * 16384 + 1024;
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        const int g = dev_sms / 4 * 4;
        auto launch = [&](int rr) {
          cudaLaunchConfig_t cfg = {};
          cfg.gridDim = dim3(g); cfg.blockDim = dim3(128); cfg.dynamicSmemBytes = sm;
          cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
          at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
          cfg.attrs = at; cfg.numAttrs = 1;
          if (cs == 1) { cudaFuncSetAttribute(k_copy_mc2<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            cudaLaunchKernelEx(&cfg, k_copy_mc2<1>, map, rows / 128, rr, mc, dc); }
          if (cs == 2) { cudaFuncSetAttribute(k_copy_mc2<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            cudaLaunchKernelEx(&cfg, k_copy_mc2<2>, map, rows / 128, rr, mc, dc); }
        };
        launch(10);
        cudaEventRecord(e0);
        launch(rounds);
        cudaEventRecord(e1);
        cudaError_t err = cudaDeviceSynchronize();
        if (err != cudaSuccess) { printf("mc2 launch failed: %s\n", cudaGetErrorString(err)); return 1; }
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double bytes = static_cast<double>(g) * rounds * 32 * 16384.0;
        printf("cluster=%d multicast=%d delivered=%.0f GB/s per-SM=%.1f B/clk@1.9GHz  L2 reads=%.0f GB/s\n", cs, mc,
               bytes / (ms * 1e6), bytes / (ms * 1e-3) / g / 1.9e9, bytes / (ms * 1e6) / (mc ? cs : 1));
      }
    printf("# pairs + TMA writers / TMEM readers: cycles per M=256 MMA (K=8)\n");
    cudaFuncSetAttribute(k_bench_pair, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kABytes + kBBytes + 4 * 32768 + 1024);
    unsigned long long* dcopied;
    cudaMalloc(&dcopied, 4096 * 8);
    for (int ce : {1, 2, 4, 0})
      for (int n : {48, 128, 192, 256}) {
        Cfg c{0, n, 0, 4096, 0, 0, ce};
        k_bench_pair<<<dev_sms, 256, kABytes + kBBytes + 4 * 32768 + 1024>>>(
            c, dA, dB, dc, map, rows / 128, 0, 0, reinterpret_cast<unsigned long long*>(dc + 2048));
        if (cudaDeviceSynchronize() != cudaSuccess) { printf("pair launch failed\n"); return 1; }
        std::vector<long long> hc(dev_sms / 2);
        cudaMemcpy(hc.data(), dc, hc.size() * 8, cudaMemcpyDeviceToHost);
        double s = 0;
        for (auto v : hc) s += v;
        s /= hc.size() * (c.iters * 4.0);
        printf("commit every %d K-blocks: n=%3d cyc/mma=%7.1f frac=%.3f\n", ce, n, s,
               128.0 * n * 16 / 4096.0 / s);
      }
    for (int readers : {0})
      for (int iss : {0, 4})
        for (int n : {48, 192}) {
          Cfg c{0, n, 0, 4096, 0, 0};
          cudaMemset(dcopied, 0, 4096 * 8);
          k_bench_pair<<<dev_sms, 256, kABytes + kBBytes + 4 * 32768 + 1024>>>(
              c, dA, dB, dc, map, rows / 128, iss, readers, dcopied);
          if (cudaDeviceSynchronize() != cudaSuccess) { printf("pair launch failed\n"); return 1; }
          std::vector<long long> hc(dev_sms / 2);
          std::vector<unsigned long long> hb(dev_sms * 4);
          cudaMemcpy(hc.data(), dc, hc.size() * 8, cudaMemcpyDeviceToHost);
          cudaMemcpy(hb.data(), dcopied, hb.size() * 8, cudaMemcpyDeviceToHost);
          double s = 0, b = 0;
          for (auto v : hc) s += v;
          for (auto v : hb) b += v;
          const double cyc_total = s / hc.size();
          s = cyc_total / (c.iters * 4.0);
          const double ideal = 128.0 * n * 8 * 2 / 4096.0;
          printf("tmem_readers=%d tma_issuers=%d n=%3d cyc/mma=%7.1f frac=%.3f tma_B/clk/SM=%.1f\n",
                 readers, iss, n, s, ideal / s, b / dev_sms / cyc_total);
        }
  }
  printf("# inbound bulk-copy ceiling, %d CTAs x depth x 16 KB\n", dev_sms);
  float* huge;
  const long long huge_f = 1ll << 28;  // 1 GiB
  cudaMalloc(&huge, huge_f * 4);
  cudaMemset(huge, 0, huge_f * 4);
  cudaFuncSetAttribute(k_copy, cudaFuncAttributeMaxDynamicSharedMemorySize, 12 * 16384);
  for (int same : {0, 1})
    for (long long region : {1ll << 22, huge_f})
      for (int grid : {8, 37, 74, 148, 296})
        for (int depth : {4, 8}) {
          const int iters = 2000;
          cudaEvent_t e0, e1;
          cudaEventCreate(&e0);
          cudaEventCreate(&e1);
          k_copy<<<grid, 32, depth * 16384>>>(huge, region, 200, depth, dc, same);
          cudaEventRecord(e0);
          k_copy<<<grid, 32, depth * 16384>>>(huge, region, iters, depth, dc, same);
          cudaEventRecord(e1);
          if (cudaDeviceSynchronize() != cudaSuccess) { printf("launch failed\n"); return 1; }
          float ms;
          cudaEventElapsedTime(&ms, e0, e1);
          std::vector<long long> hc(grid);
          cudaMemcpy(hc.data(), dc, grid * 8, cudaMemcpyDeviceToHost);
          double s = 0;
          for (auto v : hc) s += v;
          s /= grid;
          printf("same=%d region=%5lld MB grid=%3d depth=%2d B/clk/CTA=%.1f aggregate=%.0f GB/s\n",
                 same, region * 4 >> 20, grid, depth, iters * 16384.0 / s,
                 grid * iters * 16384.0 / (ms * 1e6));
        }
  return 0;
}
