// TF32 tensor-core (tcgen05) implicit GEMM for conv fprop / dgrad / wgrad and the
// linear layers, NHWC.  One warp-specialised kernel:
//   warp 0      : TMA producer (one lane) — operand tiles land in a multi-stage SMEM ring
//                 straight from the NHWC activations / weights (no im2col buffer: a conv
//                 tap is a shifted 4-D box whose out-of-bounds cells TMA fills with 0)
//   warp 1      : MMA issuer (one lane) — tcgen05.mma.kind::tf32, fp32 accumulator in TMEM
//   warp 2      : TMEM allocator
//   warps 4..7  : epilogue — tcgen05.ld TMEM -> registers -> bias/ReLU -> HBM
//                 (or fixed-order split-K partials)
// Operand modes (all SWIZZLE_128B unless K-major with 16-float K blocks -> SWIZZLE_64B):
//   A_RECT_K   conv fprop/dgrad A: pixel rectangle x channel block (K-major)
//   A_2D_K     linear fprop/dgrad A: [rows][K] (K-major)
//   A_RECT_MN  conv wgrad A = dY: filters (M, contiguous) x pixel rectangle (K)
//   A_2D_MN    linear wgrad A = dY: [K rows][M] (MN-major)
//   B_2D_K     weights [N rows][K] (K-major)
//   B_WT_MN    conv dgrad B = W^T: channels (N, contiguous) x (tap, filter block) (K)
//   B_RECT_MN  conv wgrad B = X shifted by the CTA's tap (N = channels, K = pixels)
//   B_2D_MN    [K rows][N] (MN-major): linear dgrad W, linear wgrad X
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstring>
#include <mutex>

#include "psg_internal.h"
#include "tc_gemm.cuh"

namespace psg {
namespace {

enum AMode { A_RECT_K = 0, A_2D_K = 1, A_RECT_MN = 2, A_2D_MN = 3 };
enum BMode { B_2D_K = 0, B_WT_MN = 1, B_RECT_MN = 2, B_2D_MN = 3 };
enum RowMap { ROW_RECT = 0, ROW_LINEAR = 1 };

constexpr int kThreads = 256;
constexpr int kTileM = 128;

struct TcArgs {
  int a_mode, b_mode, row_map;
  int n_tile;             // UMMA N (multiple of 16, <= 256)
  int stage_bytes, a_bytes, stages;
  int m_tiles, n_tiles;   // per (group, tap)
  int G, taps;            // blockIdx.y = g * taps + tap
  int kblocks, kb_per_split;
  // coordinate helpers
  int a_c_g;              // A channel / M offset per group
  int b_r_g;              // B row (K or N) offset per group
  int b_n_g;              // B N offset per group (rect MN)
  int cb;                 // K blocks per tap (rect-K A, W^T B)
  int kw, ph, pw, sign;   // tap shift: coord = origin + sign * (u - p)
  // M rectangles (ROW_RECT)
  int rm, wm, th, tw;
  int out_h, out_w;
  // K rectangles (A/B_RECT_MN)
  int rk, wk, kth, ktw;
  // epilogue
  float* out;
  float* ws;
  long long ws_stride;
  const float* bias;
  int relu, accumulate;
  int ldo;
  int m_valid;            // rows valid in M (per group), ROW_LINEAR
  int n_valid;            // columns valid in N (per group)
  int col_g, col_tap, row_g;
};

template <int KBLK>
__global__ void __launch_bounds__(kThreads, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap map_a,
                   const __grid_constant__ CUtensorMap map_b, const TcArgs p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  __shared__ __align__(8) uint64_t full_bar[8], empty_bar[8], tmem_full_bar;
  __shared__ uint32_t tmem_base_sh;

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int tile_m = blockIdx.x / p.n_tiles, tile_n = blockIdx.x % p.n_tiles;
  const int g = blockIdx.y / p.taps, tap = blockIdx.y % p.taps;
  const int split = blockIdx.z;
  const int kb0 = split * p.kb_per_split;
  const int nkb = min(p.kblocks, kb0 + p.kb_per_split) - kb0;

  if (warp == 0 && lane == 0) {
    tc::tma_prefetch(&map_a);
    tc::tma_prefetch(&map_b);
    for (int s = 0; s < p.stages; ++s) {
      tc::mbar_init(tc::smem_u32(&full_bar[s]), 1);
      tc::mbar_init(tc::smem_u32(&empty_bar[s]), 1);
    }
    tc::mbar_init(tc::smem_u32(&tmem_full_bar), 1);
    tc::fence_barrier_init();
  }
  if (warp == 2) tc::tmem_alloc(tc::smem_u32(&tmem_base_sh), 256);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = tmem_base_sh;

  // M-tile origin for pixel rectangles
  int rb = 0, r_oh0 = 0, r_ow0 = 0;
  if (p.row_map == ROW_RECT) {
    rb = tile_m / (p.th * p.tw);
    const int r = tile_m % (p.th * p.tw);
    r_oh0 = (r / p.tw) * p.rm;
    r_ow0 = (r % p.tw) * p.wm;
  }

  if (warp == 0 && lane == 0) {
    // ------------------------------------------------------------ producer
    const int u = tap / p.kw, v = tap % p.kw;
    for (int i = 0; i < nkb; ++i) {
      const int s = i % p.stages;
      tc::mbar_wait(tc::smem_u32(&empty_bar[s]), ((i / p.stages) & 1) ^ 1);
      const uint32_t bar = tc::smem_u32(&full_bar[s]);
      tc::mbar_arrive_expect_tx(bar, p.stage_bytes);
      const uint32_t sa = tc::smem_u32(smem + static_cast<size_t>(s) * p.stage_bytes);
      const uint32_t sb = sa + p.a_bytes;
      const int kb = kb0 + i;
      // K rectangle (pixels) for MN-major rect operands
      int kbi = 0, koh = 0, kow = 0;
      if (p.a_mode == A_RECT_MN || p.b_mode == B_RECT_MN) {
        kbi = kb / (p.kth * p.ktw);
        const int r = kb % (p.kth * p.ktw);
        koh = (r / p.ktw) * p.rk;
        kow = (r % p.ktw) * p.wk;
      }
      switch (p.a_mode) {
        case A_RECT_K: {
          const int t = kb / p.cb, cb = kb % p.cb;
          const int tu = t / p.kw, tv = t % p.kw;
          tc::tma_load_4d(sa, &map_a, bar, p.a_c_g * g + cb * KBLK,
                          r_ow0 + p.sign * (tv - p.pw), r_oh0 + p.sign * (tu - p.ph), rb);
          break;
        }
        case A_2D_K:
          tc::tma_load_2d(sa, &map_a, bar, kb * KBLK, tile_m * kTileM);
          break;
        case A_RECT_MN:
          for (int j = 0; j < kTileM / 32; ++j)
            tc::tma_load_4d(sa + j * KBLK * 128, &map_a, bar,
                            p.a_c_g * g + tile_m * kTileM + 32 * j, kow, koh, kbi);
          break;
        case A_2D_MN:
          for (int j = 0; j < kTileM / 32; ++j)
            tc::tma_load_2d(sa + j * KBLK * 128, &map_a, bar, tile_m * kTileM + 32 * j,
                            kb * KBLK);
          break;
      }
      const int nch = (p.n_tile + 31) / 32;
      switch (p.b_mode) {
        case B_2D_K:
          tc::tma_load_2d(sb, &map_b, bar, kb * KBLK, p.b_r_g * g + tile_n * p.n_tile);
          break;
        case B_WT_MN: {
          const int t = kb / p.cb, fb = kb % p.cb;
          for (int j = 0; j < nch; ++j)
            tc::tma_load_3d(sb + j * KBLK * 128, &map_b, bar, tile_n * p.n_tile + 32 * j, t,
                            p.b_r_g * g + fb * KBLK);
          break;
        }
        case B_RECT_MN:
          for (int j = 0; j < nch; ++j)
            tc::tma_load_4d(sb + j * KBLK * 128, &map_b, bar,
                            p.b_n_g * g + tile_n * p.n_tile + 32 * j, kow + v - p.pw,
                            koh + u - p.ph, kbi);
          break;
        case B_2D_MN:
          for (int j = 0; j < nch; ++j)
            tc::tma_load_2d(sb + j * KBLK * 128, &map_b, bar, tile_n * p.n_tile + 32 * j,
                            kb * KBLK);
          break;
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ------------------------------------------------------------ MMA issue
    const bool a_mn = p.a_mode == A_RECT_MN || p.a_mode == A_2D_MN;
    const bool b_mn = p.b_mode != B_2D_K;
    const uint32_t idesc = tc::idesc_tf32(kTileM, p.n_tile, a_mn, b_mn);
    const uint32_t k_sw = KBLK == 32 ? tc::kSw128 : tc::kSw64;
    const uint32_t k_sbo = 8 * KBLK * 4;  // 8 rows of KBLK floats
    for (int i = 0; i < nkb; ++i) {
      const int s = i % p.stages;
      tc::mbar_wait(tc::smem_u32(&full_bar[s]), (i / p.stages) & 1);
      tc::fence_after_sync();
      const uint32_t sa = tc::smem_u32(smem + static_cast<size_t>(s) * p.stage_bytes);
      const uint32_t sb = sa + p.a_bytes;
#pragma unroll
      for (int j = 0; j < KBLK / 8; ++j) {
        const uint64_t ad = a_mn ? tc::smem_desc(sa + j * 1024, KBLK * 128, 512, tc::kSw128Base32)
                                 : tc::smem_desc(sa + j * 32, 16, k_sbo, k_sw);
        const uint64_t bd = b_mn ? tc::smem_desc(sb + j * 1024, KBLK * 128, 512, tc::kSw128Base32)
                                 : tc::smem_desc(sb + j * 32, 16, k_sbo, k_sw);
        tc::mma_tf32(tmem, ad, bd, idesc, (i | j) != 0 ? 1u : 0u);
      }
      tc::mma_commit(tc::smem_u32(&empty_bar[s]));
    }
    tc::mma_commit(tc::smem_u32(&tmem_full_bar));
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue
    const int ew = warp - 4;
    const int m = ew * 32 + lane;
    bool row_ok;
    long long out_row;
    if (p.row_map == ROW_RECT) {
      const int oh = r_oh0 + m / p.wm, ow = r_ow0 + m % p.wm;
      row_ok = oh < p.out_h && ow < p.out_w;
      out_row = (static_cast<long long>(rb) * p.out_h + oh) * p.out_w + ow;
    } else {
      const int mm = tile_m * kTileM + m;
      row_ok = mm < p.m_valid;
      out_row = static_cast<long long>(p.row_g) * g + mm;
    }
    const int col0 = p.col_g * g + p.col_tap * tap + tile_n * p.n_tile;
    const int nvalid = min(p.n_tile, p.n_valid - tile_n * p.n_tile);
    tc::mbar_wait(tc::smem_u32(&tmem_full_bar), 0);
    tc::fence_after_sync();
    for (int c0 = 0; c0 < p.n_tile; c0 += 16) {
      float vals[16];
      tc::tmem_ld16(tmem + (static_cast<uint32_t>(ew * 32) << 16) + c0, vals);
      if (!row_ok) continue;
      const long long base = out_row * p.ldo + col0 + c0;
      if (p.ws) {
        float* dst = p.ws + split * p.ws_stride + base;
#pragma unroll
        for (int q = 0; q < 16; ++q)
          if (c0 + q < nvalid) dst[q] = vals[q];
      } else {
        float* dst = p.out + base;
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          if (c0 + q >= nvalid) continue;
          float y = vals[q];
          if (p.bias) {
            y += p.bias[col0 + c0 + q];
            if (p.relu) y = y > 0.f ? y : 0.f;
          }
          if (p.accumulate) y += dst[q];
          dst[q] = y;
        }
      }
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 2) {
    tc::fence_after_sync();
    tc::tmem_dealloc(tmem, 256);
  }
}

// Fixed-order second stage: out[i] (+)= sum_z ws[z][i] (+ bias[i % ldo], relu).
__global__ void tc_split_reduce(const float* __restrict__ ws, int splits, long long stride,
                                long long total, const float* __restrict__ bias, int ldo,
                                int relu, int accumulate, float* __restrict__ out) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    float s = 0.f;
    for (int z = 0; z < splits; ++z) s += ws[z * stride + i];
    if (bias) {
      s += bias[i % ldo];
      if (relu) s = s > 0.f ? s : 0.f;
    }
    out[i] = accumulate ? out[i] + s : s;
  }
}

// db[c] = sum over rows of dy[r][c] in a fixed order: row chunks per block, then chunks.
__global__ void bias_grad_partial(const float* __restrict__ dy, long long rows, int cols,
                                  long long rows_per_chunk, float* __restrict__ part) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const long long r0 = blockIdx.y * rows_per_chunk;
  if (c >= cols) return;
  const long long r1 = min(rows, r0 + rows_per_chunk);
  float s = 0.f;
  for (long long r = r0; r < r1; ++r) s += dy[r * cols + c];
  part[static_cast<long long>(blockIdx.y) * cols + c] = s;
}

__global__ void bias_grad_final(const float* __restrict__ part, int chunks, int cols,
                                float* __restrict__ db) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cols) return;
  float s = 0.f;
  for (int z = 0; z < chunks; ++z) s += part[static_cast<long long>(z) * cols + c];
  db[c] = s;
}

// ---------------------------------------------------------------- host side
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  if (!fn) throw CudaError("cuTensorMapEncodeTiled unavailable");
  return fn;
}

// dims / box innermost first; strides in bytes for dims 1..rank-1.
CUtensorMap make_map(const void* base, int rank, const uint64_t* dims, const uint64_t* strides,
                     const uint32_t* box, CUtensorMapSwizzle sw) {
  CUtensorMap m;
  uint32_t estr[5] = {1, 1, 1, 1, 1};
  const CUresult r = encode_fn()(
      &m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, const_cast<void*>(base), dims, strides, box,
      estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
  return m;
}

CUtensorMap map_nhwc(const float* base, int n, int h, int w, int c, int box_c, int box_w,
                     int box_h, CUtensorMapSwizzle sw) {
  const uint64_t dims[4] = {static_cast<uint64_t>(c), static_cast<uint64_t>(w),
                            static_cast<uint64_t>(h), static_cast<uint64_t>(n)};
  const uint64_t str[3] = {static_cast<uint64_t>(c) * 4, static_cast<uint64_t>(w) * c * 4,
                           static_cast<uint64_t>(h) * w * c * 4};
  const uint32_t box[4] = {static_cast<uint32_t>(box_c), static_cast<uint32_t>(box_w),
                           static_cast<uint32_t>(box_h), 1};
  return make_map(base, 4, dims, str, box, sw);
}

CUtensorMap map_2d(const float* base, long long rows, long long cols, int box_c, int box_r,
                   CUtensorMapSwizzle sw) {
  const uint64_t dims[2] = {static_cast<uint64_t>(cols), static_cast<uint64_t>(rows)};
  const uint64_t str[1] = {static_cast<uint64_t>(cols) * 4};
  const uint32_t box[2] = {static_cast<uint32_t>(box_c), static_cast<uint32_t>(box_r)};
  return make_map(base, 2, dims, str, box, sw);
}

int pow2_at_least(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}

// Rectangle of `area` pixels (power of two) over an OH x OW grid: box width >= OW
// when possible.
void rect_shape(int out_w, int area, int& rows, int& width) {
  width = std::min(area, pow2_at_least(out_w));
  rows = area / width;
}

int pick_n_tile(int N) {
  const int tiles = (N + 255) / 256;
  const int per = (N + tiles - 1) / tiles;
  return (per + 15) / 16 * 16;
}

void finish_args(TcArgs& a, int kblk, int sms) {
  const bool b_mn = a.b_mode != B_2D_K;
  const int nb = b_mn ? (a.n_tile + 31) / 32 * 32 : a.n_tile;
  a.a_bytes = kTileM * kblk * 4;
  a.stage_bytes = a.a_bytes + nb * kblk * 4;
  a.stages = std::min(8, (220 * 1024) / a.stage_bytes);
  const long long tiles = static_cast<long long>(a.m_tiles) * a.n_tiles * a.G * a.taps;
  int splits = 1;
  if (tiles < sms) splits = static_cast<int>(std::min<long long>((sms + tiles - 1) / tiles,
                                                                 std::max(1, a.kblocks / 4)));
  a.kb_per_split = (a.kblocks + splits - 1) / splits;
}

int splits_of(const TcArgs& a) { return (a.kblocks + a.kb_per_split - 1) / a.kb_per_split; }

void launch(const TcArgs& a0, const CUtensorMap& ma, const CUtensorMap& mb, int kblk,
            long long out_elems, float* ws, size_t ws_elems, cudaStream_t s) {
  TcArgs a = a0;
  const int splits = splits_of(a);
  if (splits > 1) {
    if (ws_elems < static_cast<size_t>(splits) * out_elems)
      throw std::logic_error("tc: split-K workspace too small");
    a.ws = ws;
    a.ws_stride = out_elems;
  }
  const dim3 grid(a.m_tiles * a.n_tiles, a.G * a.taps, splits);
  const size_t smem = static_cast<size_t>(a.stages) * a.stage_bytes + 1024;
  if (kblk == 32) {
    PSG_CUDA(cudaFuncSetAttribute(tc_gemm_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    tc_gemm_kernel<32><<<grid, kThreads, smem, s>>>(ma, mb, a);
  } else {
    PSG_CUDA(cudaFuncSetAttribute(tc_gemm_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    tc_gemm_kernel<16><<<grid, kThreads, smem, s>>>(ma, mb, a);
  }
  PSG_CUDA(cudaGetLastError());
  if (splits > 1) {
    const int blocks = static_cast<int>(std::min<long long>((out_elems + 255) / 256, 148 * 8));
    tc_split_reduce<<<blocks, 256, 0, s>>>(ws, splits, out_elems, out_elems, a0.bias, a0.ldo,
                                           a0.relu, a0.accumulate, a0.out);
    PSG_CUDA(cudaGetLastError());
  }
}

bool is_linear(const ConvGeom& g) {
  return g.H == 1 && g.W == 1 && g.OH == 1 && g.OW == 1 && g.kh == 1 && g.kw == 1;
}

int kblk_for(int channels) { return channels % 32 == 0 ? 32 : (channels % 16 == 0 ? 16 : 0); }

// --- planners: fill TcArgs (out/bias/flags are set by the caller) -------------
bool plan_fprop(const ConvGeom& g, TcArgs& a, int& kblk) {
  std::memset(&a, 0, sizeof a);
  if (is_linear(g)) {
    const int D = g.cs_in, O = g.F;
    if (D % 4) return false;
    kblk = 32;
    a.a_mode = A_2D_K;
    a.b_mode = B_2D_K;
    a.row_map = ROW_LINEAR;
    a.n_tile = pick_n_tile(O);
    a.m_tiles = (g.n + kTileM - 1) / kTileM;
    a.n_tiles = (O + a.n_tile - 1) / a.n_tile;
    a.G = a.taps = 1;
    a.kblocks = (D + kblk - 1) / kblk;
    a.m_valid = g.n;
    a.n_valid = O;
    a.ldo = O;
    return true;
  }
  if (g.sh != 1 || g.sw != 1) return false;
  kblk = kblk_for(g.Cgs());
  if (!kblk || g.Fg() % 16) return false;
  a.a_mode = A_RECT_K;
  a.b_mode = B_2D_K;
  a.row_map = ROW_RECT;
  rect_shape(g.OW, kTileM, a.rm, a.wm);
  a.th = (g.OH + a.rm - 1) / a.rm;
  a.tw = (g.OW + a.wm - 1) / a.wm;
  a.out_h = g.OH;
  a.out_w = g.OW;
  a.n_tile = pick_n_tile(g.Fg());
  a.m_tiles = g.n * a.th * a.tw;
  a.n_tiles = (g.Fg() + a.n_tile - 1) / a.n_tile;
  a.G = g.G;
  a.taps = 1;
  a.cb = g.Cgs() / kblk;
  a.kblocks = g.kh * g.kw * a.cb;
  a.a_c_g = g.Cgs();
  a.b_r_g = g.Fg();
  a.kw = g.kw;
  a.ph = g.ph;
  a.pw = g.pw;
  a.sign = 1;
  a.n_valid = g.Fg();
  a.col_g = g.Fg();
  a.ldo = g.F;
  return true;
}

bool plan_dgrad(const ConvGeom& g, TcArgs& a, int& kblk) {
  std::memset(&a, 0, sizeof a);
  if (is_linear(g)) {
    const int D = g.cs_in, O = g.F;
    if (O % 4 || D % 4) return false;
    kblk = 32;
    a.a_mode = A_2D_K;   // dY [n][O]
    a.b_mode = B_2D_MN;  // W [O][D]
    a.row_map = ROW_LINEAR;
    a.n_tile = pick_n_tile(D);
    a.m_tiles = (g.n + kTileM - 1) / kTileM;
    a.n_tiles = (D + a.n_tile - 1) / a.n_tile;
    a.G = a.taps = 1;
    a.kblocks = (O + kblk - 1) / kblk;
    a.m_valid = g.n;
    a.n_valid = D;
    a.ldo = D;
    return true;
  }
  if (g.sh != 1 || g.sw != 1) return false;
  kblk = kblk_for(g.Fg());
  if (!kblk || g.Cgs() % 16) return false;
  a.a_mode = A_RECT_K;   // dY rectangles, taps reversed
  a.b_mode = B_WT_MN;    // W^T
  a.row_map = ROW_RECT;
  rect_shape(g.W, kTileM, a.rm, a.wm);
  a.th = (g.H + a.rm - 1) / a.rm;
  a.tw = (g.W + a.wm - 1) / a.wm;
  a.out_h = g.H;
  a.out_w = g.W;
  a.n_tile = pick_n_tile(g.Cgs());
  a.m_tiles = g.n * a.th * a.tw;
  a.n_tiles = (g.Cgs() + a.n_tile - 1) / a.n_tile;
  a.G = g.G;
  a.taps = 1;
  a.cb = g.Fg() / kblk;
  a.kblocks = g.kh * g.kw * a.cb;
  a.a_c_g = g.Fg();
  a.b_r_g = g.Fg();
  a.kw = g.kw;
  a.ph = g.ph;
  a.pw = g.pw;
  a.sign = -1;
  a.n_valid = g.Cgs();
  a.col_g = g.Cgs();
  a.ldo = g.cs_in;
  return true;
}

bool plan_wgrad(const ConvGeom& g, TcArgs& a, int& kblk) {
  std::memset(&a, 0, sizeof a);
  kblk = 32;
  if (is_linear(g)) {
    const int D = g.cs_in, O = g.F;
    if (O % 4 || D % 4) return false;
    a.a_mode = A_2D_MN;  // dY [n][O]
    a.b_mode = B_2D_MN;  // X [n][D]
    a.row_map = ROW_LINEAR;
    a.n_tile = pick_n_tile(D);
    a.m_tiles = (O + kTileM - 1) / kTileM;
    a.n_tiles = (D + a.n_tile - 1) / a.n_tile;
    a.G = a.taps = 1;
    a.kblocks = (g.n + kblk - 1) / kblk;
    a.m_valid = O;
    a.n_valid = D;
    a.ldo = D;
    return true;
  }
  if (g.sh != 1 || g.sw != 1 || g.Cgs() % 16 || g.Fg() % 4) return false;
  a.a_mode = A_RECT_MN;  // dY: filters x pixels
  a.b_mode = B_RECT_MN;  // X shifted by the tap: channels x pixels
  a.row_map = ROW_LINEAR;
  rect_shape(g.OW, kblk, a.rk, a.wk);
  a.kth = (g.OH + a.rk - 1) / a.rk;
  a.ktw = (g.OW + a.wk - 1) / a.wk;
  a.n_tile = pick_n_tile(g.Cgs());
  a.m_tiles = (g.Fg() + kTileM - 1) / kTileM;
  a.n_tiles = (g.Cgs() + a.n_tile - 1) / a.n_tile;
  a.G = g.G;
  a.taps = g.kh * g.kw;
  a.kblocks = g.n * a.kth * a.ktw;
  a.a_c_g = g.Fg();
  a.b_n_g = g.Cgs();
  a.kw = g.kw;
  a.ph = g.ph;
  a.pw = g.pw;
  a.m_valid = g.Fg();
  a.n_valid = g.Cgs();
  a.row_g = g.Fg();
  a.col_tap = g.Cgs();
  a.ldo = g.Kf();
  return true;
}

int sm_count() {
  static int sms = [] {
    int dev = 0, v = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return sms;
}

// MN-major tf32 operands: 128B rows swizzled in 32B chunks (UMMA SWIZZLE_128B_BASE32B).
constexpr CUtensorMapSwizzle kMnSwizzle = CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B;

CUtensorMapSwizzle k_swizzle(int kblk) {
  return kblk == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
}

// dW split partials followed by the bias-gradient partials (64 row chunks max).
size_t tc_wgrad_ws_elems(const ConvGeom& g) {
  TcArgs a;
  int kblk;
  if (!plan_wgrad(g, a, kblk)) return 0;
  finish_args(a, kblk, sm_count());
  const int splits = splits_of(a);
  return (splits > 1 ? static_cast<size_t>(splits) * g.F * g.Kf() : 0) +
         64 * static_cast<size_t>(g.F);
}

}  // namespace

bool tc_supported(const ConvGeom& g, int which) {
  TcArgs a;
  int kblk;
  switch (which) {
    case 0:
      return plan_fprop(g, a, kblk);
    case 1:
      return plan_dgrad(g, a, kblk);
    default:
      return plan_wgrad(g, a, kblk);
  }
}

size_t tc_workspace_elems(const ConvGeom& g) {
  size_t e = 0;
  TcArgs a;
  int kblk;
  if (plan_fprop(g, a, kblk)) {
    finish_args(a, kblk, sm_count());
    if (splits_of(a) > 1)
      e = std::max(e, static_cast<size_t>(splits_of(a)) * g.n * g.OH * g.OW * g.F);
  }
  if (plan_dgrad(g, a, kblk)) {
    finish_args(a, kblk, sm_count());
    if (splits_of(a) > 1)
      e = std::max(e, static_cast<size_t>(splits_of(a)) * g.n * g.H * g.W * g.cs_in);
  }
  if (plan_wgrad(g, a, kblk)) {
    finish_args(a, kblk, sm_count());
    e = std::max(e, tc_wgrad_ws_elems(g));
  }
  return e;
}

int tc_launches(const ConvGeom& g, int which) {
  TcArgs a;
  int kblk;
  const bool ok = which == 0 ? plan_fprop(g, a, kblk)
                             : which == 1 ? plan_dgrad(g, a, kblk) : plan_wgrad(g, a, kblk);
  if (!ok) return -1;
  finish_args(a, kblk, sm_count());
  return (splits_of(a) > 1 ? 2 : 1) + (which == 2 ? 2 : 0);
}

void tc_fprop(const ConvGeom& g, const float* x, const float* w, const float* bias, float* y,
              bool relu, const Workspace& ws, cudaStream_t s) {
  TcArgs a;
  int kblk;
  if (!plan_fprop(g, a, kblk)) throw std::logic_error("tc_fprop: unsupported geometry");
  finish_args(a, kblk, sm_count());
  a.out = y;
  a.bias = bias;
  a.relu = relu;
  CUtensorMap ma, mb;
  if (a.a_mode == A_2D_K) {
    ma = map_2d(x, g.n, g.cs_in, kblk, kTileM, k_swizzle(kblk));
    mb = map_2d(w, g.F, g.cs_in, kblk, a.n_tile, k_swizzle(kblk));
  } else {
    ma = map_nhwc(x, g.n, g.H, g.W, g.cs_in, kblk, a.wm, a.rm, k_swizzle(kblk));
    mb = map_2d(w, g.F, g.Kf(), kblk, a.n_tile, k_swizzle(kblk));
  }
  launch(a, ma, mb, kblk, static_cast<long long>(g.n) * g.OH * g.OW * g.F, ws.ptr, ws.elems, s);
}

void tc_dgrad(const ConvGeom& g, const float* dy, const float* w, float* dx, bool accumulate,
              const Workspace& ws, cudaStream_t s) {
  TcArgs a;
  int kblk;
  if (!plan_dgrad(g, a, kblk)) throw std::logic_error("tc_dgrad: unsupported geometry");
  finish_args(a, kblk, sm_count());
  a.out = dx;
  a.accumulate = accumulate;
  CUtensorMap ma, mb;
  if (a.a_mode == A_2D_K) {
    ma = map_2d(dy, g.n, g.F, kblk, kTileM, k_swizzle(kblk));
    mb = map_2d(w, g.F, g.cs_in, 32, kblk, kMnSwizzle);
  } else {
    ma = map_nhwc(dy, g.n, g.OH, g.OW, g.F, kblk, a.wm, a.rm, k_swizzle(kblk));
    const uint64_t dims[3] = {static_cast<uint64_t>(g.Cgs()),
                              static_cast<uint64_t>(g.kh) * g.kw, static_cast<uint64_t>(g.F)};
    const uint64_t str[2] = {static_cast<uint64_t>(g.Cgs()) * 4,
                             static_cast<uint64_t>(g.Kf()) * 4};
    const uint32_t box[3] = {32, 1, static_cast<uint32_t>(kblk)};
    mb = make_map(w, 3, dims, str, box, kMnSwizzle);
  }
  launch(a, ma, mb, kblk, static_cast<long long>(g.n) * g.H * g.W * g.cs_in, ws.ptr, ws.elems,
         s);
}

void tc_wgrad(const ConvGeom& g, const float* x, const float* dy, float* dw, float* db,
              const Workspace& ws, cudaStream_t s) {
  TcArgs a;
  int kblk;
  if (!plan_wgrad(g, a, kblk)) throw std::logic_error("tc_wgrad: unsupported geometry");
  finish_args(a, kblk, sm_count());
  a.out = dw;
  CUtensorMap ma, mb;
  if (a.a_mode == A_2D_MN) {
    ma = map_2d(dy, g.n, g.F, 32, kblk, kMnSwizzle);
    mb = map_2d(x, g.n, g.cs_in, 32, kblk, kMnSwizzle);
  } else {
    ma = map_nhwc(dy, g.n, g.OH, g.OW, g.F, 32, a.wk, a.rk, kMnSwizzle);
    mb = map_nhwc(x, g.n, g.H, g.W, g.cs_in, 32, a.wk, a.rk, kMnSwizzle);
  }
  const long long dw_elems = static_cast<long long>(g.F) * g.Kf();
  // the split-K workspace holds dW partials; bias partials go after them
  const int splits = splits_of(a);
  float* part = ws.ptr + (splits > 1 ? splits * dw_elems : 0);
  launch(a, ma, mb, kblk, dw_elems, ws.ptr, ws.elems, s);
  // db[f] = sum over output pixels of dY[pix][f]
  const long long rows = static_cast<long long>(g.n) * g.OH * g.OW;
  const int chunks = static_cast<int>(std::min<long long>(64, (rows + 255) / 256));
  const long long per = (rows + chunks - 1) / chunks;
  const dim3 grid((g.F + 127) / 128, chunks);
  bias_grad_partial<<<grid, 128, 0, s>>>(dy, rows, g.F, per, part);
  PSG_CUDA(cudaGetLastError());
  bias_grad_final<<<(g.F + 127) / 128, 128, 0, s>>>(part, chunks, g.F, db);
  PSG_CUDA(cudaGetLastError());
}

}  // namespace psg
