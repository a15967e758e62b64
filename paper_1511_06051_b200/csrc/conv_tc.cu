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
//   B_3D_K     conv fprop weights as [F][taps][C/G] (K-major, channel tail zero-filled)
//   B_RECT_MN  conv wgrad B = X shifted by the CTA's tap (N = channels, K = pixels)
//   B_2D_MN    [K rows][N] (MN-major): linear dgrad W, linear wgrad X
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <set>

#include "psg_internal.h"
#include "tc_gemm.cuh"
#include "tc_kernel.cuh"

namespace psg {
namespace {

using namespace tck;

// Fixed-order second stage: out[i] (+)= sum_z ws[z][i] (+ bias[i % ldo], relu); columns
// i % ldo >= valid_cols (row padding the GEMM never writes) are set to 0.
// Fused wgrad bias (TcArgs::bias_chunk): db[f] = sum_z db_part[z][f] in the same pass.
__global__ void tc_split_reduce(const float* __restrict__ ws, int splits, long long stride,
                                long long total, const float* __restrict__ bias, int ldo,
                                int valid_cols, int relu, int accumulate,
                                const float* __restrict__ mask, float* __restrict__ out,
                                const float* __restrict__ db_part, int nb,
                                float* __restrict__ db) {
  pdl_enter();
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
       i < total + nb; i += static_cast<long long>(gridDim.x) * blockDim.x) {
    if (i >= total) {
      const int f = static_cast<int>(i - total);
      float s = 0.f;
      for (int z = 0; z < splits; ++z) s += db_part[static_cast<long long>(z) * nb + f];
      db[f] = s;
      continue;
    }
    if (valid_cols < ldo && i % ldo >= valid_cols) {
      out[i] = 0.f;
      continue;
    }
    float s = 0.f;
    for (int z = 0; z < splits; ++z) s += ws[z * stride + i];
    if (bias) {
      s += bias[i % ldo];
      if (relu) s = s > 0.f ? s : 0.f;
    }
    if (mask && !(mask[i] > 0.f)) s = 0.f;  // folded ReLU backward (dgrad)
    out[i] = accumulate ? out[i] + s : s;
  }
}

// The same per element, four consecutive elements of one row per thread (ldo, valid_cols
// and the pointers 16-byte aligned): identical arithmetic and order, a quarter of the
// instructions and 16-byte accesses.
__global__ void tc_split_reduce4(const float4* __restrict__ ws, int splits, long long stride4,
                                 long long total4, const float* __restrict__ bias, int ldo,
                                 int valid_cols, int relu, int accumulate,
                                 const float4* __restrict__ mask, float4* __restrict__ out,
                                 const float* __restrict__ db_part, int nb,
                                 float* __restrict__ db) {
  pdl_enter();
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
       i < total4 + nb; i += static_cast<long long>(gridDim.x) * blockDim.x) {
    if (i >= total4) {
      const int f = static_cast<int>(i - total4);
      float s = 0.f;
      for (int z = 0; z < splits; ++z) s += db_part[static_cast<long long>(z) * nb + f];
      db[f] = s;
      continue;
    }
    const int col = static_cast<int>((4 * i) % ldo);
    if (valid_cols < ldo && col >= valid_cols) {
      out[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      continue;
    }
    float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
    for (int z = 0; z < splits; ++z) {
      const float4 v = ws[z * stride4 + i];
      s.x += v.x;
      s.y += v.y;
      s.z += v.z;
      s.w += v.w;
    }
    if (bias) {
      const float4 bb = *reinterpret_cast<const float4*>(bias + col);
      s.x += bb.x;
      s.y += bb.y;
      s.z += bb.z;
      s.w += bb.w;
      if (relu) {
        s.x = s.x > 0.f ? s.x : 0.f;
        s.y = s.y > 0.f ? s.y : 0.f;
        s.z = s.z > 0.f ? s.z : 0.f;
        s.w = s.w > 0.f ? s.w : 0.f;
      }
    }
    if (mask) {  // folded ReLU backward (dgrad)
      const float4 m = mask[i];
      if (!(m.x > 0.f)) s.x = 0.f;
      if (!(m.y > 0.f)) s.y = 0.f;
      if (!(m.z > 0.f)) s.z = 0.f;
      if (!(m.w > 0.f)) s.w = 0.f;
    }
    if (accumulate) {
      const float4 o = out[i];
      s.x = o.x + s.x;
      s.y = o.y + s.y;
      s.z = o.z + s.z;
      s.w = o.w + s.w;
    }
    out[i] = s;
  }
}

// db[c] = sum over rows of dy[r][c] in a fixed order.  Stage 1: block (cb, chunk) owns a
// contiguous row chunk and up to 256 column units (float4 when cols % 4 == 0); thread
// (ty, tx) sums rows r0 + ty, r0 + ty + rpi, ... of unit tx, then row-lanes combine in
// order.  Stage 2: one warp per column sums the chunk partials (lane-strided, then a
// fixed xor tree).  The order depends only on the geometry: deterministic.
constexpr int kBiasChunksMax = 512;

__device__ __forceinline__ float4 add4(float4 a, float4 b) {
  return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}
__device__ __forceinline__ float add4(float a, float b) { return a + b; }
__device__ __forceinline__ float4 zero4(float4) { return make_float4(0.f, 0.f, 0.f, 0.f); }
__device__ __forceinline__ float zero4(float) { return 0.f; }

template <typename V>
__global__ void __launch_bounds__(256) bias_grad_partial(const V* __restrict__ dy, int rows,
                                                         int units, int rows_per_chunk,
                                                         V* __restrict__ part) {
  pdl_enter();
  __shared__ V red[256];
  const int cpr = min(units, 256), rpi = 256 / cpr;
  const int tx = threadIdx.x % cpr, ty = threadIdx.x / cpr;
  const int u = blockIdx.x * cpr + tx;
  const int r0 = blockIdx.y * rows_per_chunk, r1 = min(rows, r0 + rows_per_chunk);
  V acc = zero4(V{});
  if (ty < rpi && u < units) {
#pragma unroll 4
    for (int r = r0 + ty; r < r1; r += rpi) acc = add4(acc, dy[static_cast<size_t>(r) * units + u]);
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  if (ty == 0 && u < units) {
    for (int i = 1; i < rpi; ++i) acc = add4(acc, red[i * cpr + tx]);
    part[static_cast<size_t>(blockIdx.y) * units + u] = acc;
  }
}

__global__ void bias_grad_final(const float* __restrict__ part, int chunks, int cols,
                                float* __restrict__ db) {
  pdl_enter();
  const int c = blockIdx.x * 8 + threadIdx.x / 32, lane = threadIdx.x % 32;
  if (c >= cols) return;
  float s = 0.f;
  for (int z = lane; z < chunks; z += 32) s += part[static_cast<size_t>(z) * cols + c];
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) db[c] = s;
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

// im2col-mode map over NHWC [n][h][w][c]: boxes of `pixels` consecutive traversal
// positions x box_c channels.  The traversal grid is the (w + upper - lower) x
// (h + upper - lower) positions starting at the lower corner (corners: [0] = W, [1] = H).
CUtensorMap map_nhwc_im2col(const float* base, int n, int h, int w, int c, int box_c,
                            int pixels, int lw, int lh, int uw, int uh, CUtensorMapSwizzle sw) {
  using Fn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                          const cuuint64_t*, const int*, const int*, cuuint32_t, cuuint32_t,
                          const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static Fn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<Fn>(p);
  });
  if (!fn) throw CudaError("cuTensorMapEncodeIm2col unavailable");
  const cuuint64_t dims[4] = {static_cast<cuuint64_t>(c), static_cast<cuuint64_t>(w),
                              static_cast<cuuint64_t>(h), static_cast<cuuint64_t>(n)};
  const cuuint64_t str[3] = {static_cast<cuuint64_t>(c) * 4, static_cast<cuuint64_t>(w) * c * 4,
                             static_cast<cuuint64_t>(h) * w * c * 4};
  const int lower[2] = {lw, lh}, upper[2] = {uw, uh};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  CUtensorMap m;
  const CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(base), dims,
                        str, lower, upper, static_cast<cuuint32_t>(box_c),
                        static_cast<cuuint32_t>(pixels), estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw CudaError("cuTensorMapEncodeIm2col failed (" + std::to_string(r) + ")");
  return m;
}

// TMA im2col boxes over linear pixel tiles (no rectangle padding of M in fprop / dgrad,
// of K in wgrad).  PSG_TC_IM2COL bit 0: fprop / dgrad, bit 1: wgrad (default 3; 0 keeps
// the pixel rectangles).
bool use_im2col(int bit = 1) {
  static const int v = [] {
    const char* e = std::getenv("PSG_TC_IM2COL");
    return e ? std::atoi(e) : 3;
  }();
  return (v & bit) != 0;
}

// Switch a rect-K plan (fprop / dgrad) to linear pixel tiles over an out_h x out_w grid.
void to_im2col(TcArgs& a, const ConvGeom& g, int out_h, int out_w, int sign) {
  if (!use_im2col()) return;
  // TMA im2col corners are signed 8-bit for 4-D maps
  const int lw = sign > 0 ? -g.pw : -(g.kw - 1 - g.pw), lh = sign > 0 ? -g.ph : -(g.kh - 1 - g.ph);
  if (lw < -128 || lh < -128 || g.kw > 128 || g.kh > 128) return;
  a.a_mode = A_IM2COL_K;
  a.row_map = ROW_LINEAR;
  a.out_h = out_h;
  a.out_w = out_w;
  a.kh = g.kh;
  a.im_lw = lw;
  a.im_lh = lh;
  a.m_valid = g.n * out_h * out_w;
  a.m_tiles = (a.m_valid + kTileM - 1) / kTileM;
  a.row_g = 0;
}

// MN-major [rows][cols] (cols % 32 == 0) as [cols / 32][rows][32]: one box = `chunks`
// 32-column chunks x box_r rows, landing chunk-major in smem (PSG_TC_ONEBOX=0: per chunk).
bool one_box_enabled() {
  static const bool v = [] {
    const char* e = std::getenv("PSG_TC_ONEBOX");
    return e ? std::atoi(e) != 0 : true;
  }();
  return v;
}

CUtensorMap map_mn_chunks(const float* base, long long rows, long long cols, int box_r,
                          int chunks) {
  const uint64_t dims[3] = {32, static_cast<uint64_t>(rows), static_cast<uint64_t>(cols / 32)};
  const uint64_t str[2] = {static_cast<uint64_t>(cols) * 4, 128};
  const uint32_t box[3] = {32, static_cast<uint32_t>(box_r), static_cast<uint32_t>(chunks)};
  return make_map(base, 3, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
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

// CTA pairs (cta_group::2, M = 256 per MMA): for K-major A (M = pixels / rows) with at
// least two M tiles.  The pair halves each CTA's share of B and doubles the MMA's M, which
// lifts the tensor-pipe ceiling (tools/tma_bench.cu: one CTA's M = 128 MMAs take a fixed
// ~200 cycles each for N <= 256, a pair's M = 256 MMA reaches ~1.1 PFLOP/s at N >= 128).
// MN-major B is loaded in 32-column chunks, so each half must be whole chunks (N % 64).
int sm_count();

bool fuse_wgrad_bias() {  // PSG_TC_WGRAD_BIAS=0: separate bias_grad passes (A/B)
  static const bool v = [] {
    const char* e = std::getenv("PSG_TC_WGRAD_BIAS");
    return e ? std::atoi(e) != 0 : true;
  }();
  return v;
}

bool bias_tile_enabled() {  // PSG_TC_BIAS_TILE=0: no extra N tile for the bias chunk (A/B)
  static const bool v = [] {
    const char* e = std::getenv("PSG_TC_BIAS_TILE");
    return e ? std::atoi(e) != 0 : true;
  }();
  return v;
}

// TMA-store epilogue staging chunks per epilogue warp (PSG_TC_EPI_TMA: 0 = direct row stores
// in every epilogue, 1 or 2 chunks; two let a chunk's smem writes overlap the previous
// chunk's store but take 16 KB more from the stage ring)
int epi_tma_bufs() {
  static const int v = [] {
    const char* e = std::getenv("PSG_TC_EPI_TMA");
    return e ? std::max(0, std::min(2, std::atoi(e))) : 1;
  }();
  return v;
}

bool pair_k16_off() {  // PSG_TC_PAIR_K16=1: pairs for narrow 16-float-K-block GEMMs too (A/B)
  static const bool v = [] {
    const char* e = std::getenv("PSG_TC_PAIR_K16");
    return !e || std::atoi(e) == 0;
  }();
  return v;
}

bool want_pair(const TcArgs& a, int kblk) {
  static const int env = [] {
    const char* e = std::getenv("PSG_TC_PAIR");
    return e ? std::atoi(e) : 1;
  }();
  if (a.pair_policy == PSG_TC_PAIR_NEVER || (!env && a.pair_policy != PSG_TC_PAIR_ALWAYS))
    return false;
  // legality: K-major A (M = pixels / rows) or a one-box MN-major A (wgrad: M = filters),
  // with at least two M tiles
  static const bool pair_mn = [] {  // PSG_TC_PAIR_MN=0: single-CTA MN-major-A GEMMs only
    const char* e = std::getenv("PSG_TC_PAIR_MN");
    return !e || std::atoi(e) != 0;
  }();
  if (a.a_mode != A_RECT_K && a.a_mode != A_2D_K && a.a_mode != A_IM2COL_K &&
      !(a.a_mode == A_2D_MN && pair_mn))
    return false;
  if (a.m_tiles < 2) return false;
  if (a.pair_policy == PSG_TC_PAIR_ALWAYS) return true;  // parity tests of the pair kernels
  static const int min_n = [] {  // narrow tiles: the pair's B half is too thin to pay off
    const char* e = std::getenv("PSG_TC_PAIR_MIN_N");  // (cifar10_quick's N = 32 convs: +1%)
    return e ? std::atoi(e) : 48;
  }();
  if (a.n_tile < min_n) return false;
  // 16-float K blocks and N <= 64 (GoogLeNet's space-to-depth conv1 fprop: x' at 16
  // channels, 64 filters): each stage is too small for the pair to pay, 101 -> 87 us single
  if (kblk == 16 && a.n_tile <= 64 && pair_k16_off()) return false;
  // short K (GoogLeNet's 1x1 convs over 64 / 192 channels: 2 / 6 K blocks): the pair's
  // cluster overhead is not repaid; GoogLeNet +0.4%
  static const int k_kb = [] {  // PSG_TC_PAIR_K_KB: fewest K blocks for a K-major-A pair
    const char* e = std::getenv("PSG_TC_PAIR_K_KB");
    return e ? std::atoi(e) : 8;
  }();
  if (a.a_mode != A_2D_MN && a.kblocks < k_kb) return false;
  // small GEMMs: halving the number of work units costs more in load balance than the
  // pair gains (cifar10_quick); want >= 2 waves of clusters
  const long long units = static_cast<long long>((a.m_tiles + 1) / 2) * a.n_tiles * a.G * a.taps;
  // long-K linear layers (AlexNet fc6 / fc7 at b = 256: two M tiles, split K restores the
  // parallelism): the pair reads each weight tile from L2 once instead of per M tile,
  // fc6 fwd / dgrad -10%
  // (MN-major A — the wgrads over linear pixels — from 512 K blocks: GoogLeNet's 14 x 14
  // wgrads at 196 lose 5-10% as pairs, AlexNet's conv2-5 wgrads at 1352+ gain)
  static const int mn_kb = [] {  // PSG_TC_PAIR_MN_KB: that threshold (A/B)
    const char* e = std::getenv("PSG_TC_PAIR_MN_KB");
    return e ? std::atoi(e) : 512;
  }();
  const bool long_linear = (a.a_mode == A_2D_K && a.kblocks >= 64) ||
                           (a.a_mode == A_2D_MN && a.kblocks >= mn_kb);
  return env > 1 || units >= sm_count() || long_linear;
}

// PSG_TC_SPLIT_CHARGE: K blocks charged for splitting at all.  24 (vs 8): cifar10_quick
// +5% (fewer split-K partials and reduce launches), AlexNet / GoogLeNet neutral.
int split_charge() {
  static const int v = [] {
    const char* e = std::getenv("PSG_TC_SPLIT_CHARGE");
    return e ? std::max(0, std::atoi(e)) : 24;
  }();
  return v;
}

void finish_args(TcArgs& a, int kblk, int sms) {
  const bool b_mn = a.b_mode != B_2D_K && a.b_mode != B_3D_K;
  a.pair = want_pair(a, kblk) ? 1 : 0;
  if (a.pair && b_mn && a.n_tile % 64) {
    a.n_tile = std::min(256, (a.n_tile + 63) / 64 * 64);  // pad: the extra columns read 0
    a.n_tiles = (a.n_valid + a.n_tile - 1) / a.n_tile;
  }
  if (a.bias_chunk && a.n_tiles * (a.n_tile / 32) <= a.bias_chunk) a.bias_chunk = 0;
  a.b_cols = a.pair ? a.n_tile / 2 : a.n_tile;
  a.m_units = a.pair ? (a.m_tiles + 1) / 2 : a.m_tiles;
  const int nb = b_mn ? (a.b_cols + 31) / 32 * 32 : a.b_cols;
  a.a_bytes = kTileM * kblk * 4;
  const bool a_mn = a.a_mode == A_RECT_MN || a.a_mode == A_2D_MN;
  a.a_chunks = a_mn && a.m_tiles == 1 ? std::min(kTileM / 32, (a.m_valid + 31) / 32)
                                      : kTileM / 32;
  a.a_tx = a_mn ? a.a_chunks * 32 * kblk * 4 : a.a_bytes;
  a.stage_bytes = a.a_bytes + nb * kblk * 4;
  // narrow K blocks (small slots) are grouped kps per pipeline stage, ~48 KB per stage:
  // fewer barrier round trips per MMA (PSG_TC_KPS overrides)
  static const int kps_env = [] {
    const char* e = std::getenv("PSG_TC_KPS");
    return e ? std::max(1, std::atoi(e)) : 0;
  }();
  a.kps = kps_env ? kps_env : std::max(1, std::min(4, 48 * 1024 / a.stage_bytes));  // ~48 KB
  // TMA-store epilogue (not the multi-tap wgrad's scattered column map): its staging
  // chunks come out of the stage ring's budget
  a.epi_tma = !a.cpt && a.row_map == ROW_LINEAR ? epi_tma_bufs() : 0;
  const int budget = 225 * 1024 - kEpiBytes - (a.epi_tma ? 4 * a.epi_tma * kOutChunkBytes + 1024 : 0);
  a.stages = std::min(8, budget / (a.kps * a.stage_bytes));
  if (a.stages < 2) {
    a.kps = 1;
    a.stages = std::min(8, budget / a.stage_bytes);
  }
  static const int producers = [] {
    const char* e = std::getenv("PSG_TC_PRODUCERS");
    const int v = e ? std::atoi(e) : kMaxProducers;
    return std::max(1, std::min(kMaxProducers, v));
  }();
  // a producer may only run one ring ahead of the slot it refills (parity waits): <= stages.
  // (Producers sharing every stage's boxes instead measured 2.5x slower: each producer
  // then pays every stage's barrier wait and cursor walk, which cost about as much as a
  // box issue.)
  a.producers = std::min(producers, a.stages);
  // the producers' cursor jump over the other producers' stages, as mixed-radix digits
  {
    const int D = (a.producers - 1) * a.kps;
    a.adv_kb = D;
    if (a.cb) {
      a.adv_c0 = D % a.cb;
      a.adv_tap = D / a.cb;
      a.adv_tv = a.adv_tap % a.kw;
      a.adv_tu = a.adv_tap / a.kw;
    }
    if (a.kth) {
      a.adv_w = D % a.ktw;
      a.adv_h = (D / a.ktw) % a.kth;
      a.adv_b = D / (a.ktw * a.kth);
    }
  }
  const long long tiles = static_cast<long long>(a.m_units) * a.n_tiles * a.G * a.taps;
  if (a.pair) sms /= 2;  // one work unit per cluster
  // Split K so that the persistent grid's waves are full: minimise
  // waves(tiles * s) * ceil(kblocks / s) (+ a small charge per extra split for the partials
  // and the reduce pass); at least 4 K blocks per split.
  int splits = 1;
  if (tiles < 2LL * sms) {
    long long best = -1;
    const int max_s = std::max(1, std::min(a.kblocks / 4, 64));
    for (int sp = 1; sp <= max_s; ++sp) {
      const long long waves = (tiles * sp + sms - 1) / sms;
      // a split adds a reduce launch (~4 us ~ 8 K blocks) and sp partial tiles
      const long long cost =
          waves * ((a.kblocks + sp - 1) / sp) + (sp > 1 ? split_charge() + sp / 4 : 0);
      if (best < 0 || cost < best) {
        best = cost;
        splits = sp;
      }
    }
  }
  a.kb_per_split = (a.kblocks + splits - 1) / splits;
  a.splits = (a.kblocks + a.kb_per_split - 1) / a.kb_per_split;
  a.total_tiles = tiles * a.splits;
}

int splits_of(const TcArgs& a) { return (a.kblocks + a.kb_per_split - 1) / a.kb_per_split; }

int sm_count() {
  static int sms = [] {
    int dev = 0, v = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return sms;
}

constexpr CUtensorMapSwizzle kMnSwizzleOnes = CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B;

// A 32 x 32 matrix of 1.0f on the current device (the fused wgrad bias's B chunk).
const float* ones_matrix() {
  static std::mutex mu;
  static float* per_dev[64] = {};
  int dev = 0;
  PSG_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  if (!per_dev[dev]) {
    float h[32 * 32];
    for (float& v : h) v = 1.f;
    float* d = nullptr;
    PSG_CUDA(cudaMalloc(&d, sizeof h));
    PSG_CUDA(cudaMemcpy(d, h, sizeof h, cudaMemcpyHostToDevice));
    PSG_CUDA(cudaDeviceSynchronize());  // before any stream uses it
    per_dev[dev] = d;
  }
  return per_dev[dev];
}

// PSG_TC_PROF=1: every launch gets its own 8 clock64 counters (TcArgs::prof) and a label;
// psg_debug_tc_prof prints them.  The counter block is allocated with the workspaces,
// outside any stream capture.
struct TcProf {
  std::mutex mu;
  bool on = std::getenv("PSG_TC_PROF") != nullptr;
  unsigned long long* dev = nullptr;
  std::vector<std::string> labels;
};
constexpr int kProfMax = 1024;
TcProf& tc_prof() {
  static TcProf p;
  return p;
}
void tc_prof_alloc() {
  TcProf& pr = tc_prof();
  std::lock_guard<std::mutex> lock(pr.mu);
  if (!pr.on || pr.dev) return;
  PSG_CUDA(cudaMalloc(&pr.dev, kProfMax * 8 * sizeof(unsigned long long)));
  PSG_CUDA(cudaMemset(pr.dev, 0, kProfMax * 8 * sizeof(unsigned long long)));
  PSG_CUDA(cudaDeviceSynchronize());
}

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
  // float4 epilogue stores need 16-byte aligned rows and 4-column-aligned validity bounds
  a.epi_vec = a.ldo % 4 == 0 && a.col_g % 4 == 0 && a.col_tap % 4 == 0 &&
              (a.cpt ? a.cgs % 4 == 0 : a.n_valid % 4 == 0);
  float* dst = splits > 1 ? ws : a.out;
  if (!a.epi_vec || reinterpret_cast<uintptr_t>(dst) % 16) a.epi_tma = 0;
  a.ring_bytes = (a.stages * a.kps * a.stage_bytes + 1023) / 1024 * 1024;
  CUtensorMap mo;
  std::memset(&mo, 0, sizeof mo);
  if (a.bias_chunk) {  // wgrad: the ones matrix of the bias chunk (KBLK rows x 32)
    const uint64_t dims[2] = {32, 32};
    const uint64_t str[1] = {32 * 4};
    const uint32_t box[2] = {32, static_cast<uint32_t>(kblk)};
    mo = make_map(ones_matrix(), 2, dims, str, box, kMnSwizzleOnes);
    if (splits > 1) a.db_part = ws + static_cast<long long>(splits) * out_elems;
  } else if (a.epi_tma) {  // out [rows][ldo] or the workspace [splits][rows][ldo], 32 x 32 boxes
    const uint64_t rows = static_cast<uint64_t>(out_elems / a.ldo);
    const uint64_t dims[3] = {static_cast<uint64_t>(a.ldo), rows, static_cast<uint64_t>(splits)};
    const uint64_t str[2] = {static_cast<uint64_t>(a.ldo) * 4, rows * a.ldo * 4};
    const uint32_t box[3] = {32, 32, 1};
    mo = make_map(dst, splits > 1 ? 3 : 2, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B);
  }
  const size_t smem = static_cast<size_t>(a.ring_bytes) + 4 * a.epi_tma * kOutChunkBytes +
                      1024;  // + alignment of the dynamic base
  const int per = a.pair ? 2 : 1;
  {
    TcProf& pr = tc_prof();
    std::lock_guard<std::mutex> lock(pr.mu);
    if (pr.dev && pr.labels.size() < static_cast<size_t>(kProfMax)) {
      a.prof = pr.dev + pr.labels.size() * 8;
      char buf[160];
      std::snprintf(buf, sizeof buf,
                    "kblk%d a%d b%d pair%d n%dx%d m%d G%d taps%d kb%d splits%d kps%d stages%d",
                    kblk, a.a_mode, a.b_mode, a.pair, a.n_tile, a.n_tiles, a.m_tiles, a.G,
                    a.taps, a.kblocks, splits, a.kps, a.stages);
      pr.labels.push_back(buf);
    }
  }
  static const bool debug = std::getenv("PSG_TC_DEBUG") != nullptr;
  if (debug)
    std::fprintf(stderr,
                 "tc: a%d b%d pair %d m_tiles %d m_units %d n_tile %d x%d G %d taps %d kblocks %d "
                 "splits %d kps %d stages %d producers %d epi_tma %d smem %zu\n",
                 a.a_mode, a.b_mode, a.pair, a.m_tiles, a.m_units, a.n_tile, a.n_tiles, a.G,
                 a.taps, a.kblocks, splits, a.kps, a.stages, a.producers, a.epi_tma, smem);
  const unsigned units =
      static_cast<unsigned>(std::min<long long>(a.total_tiles, sm_count() / per));
  auto go = [&](auto kern) {
    allow_max_dynamic_smem(reinterpret_cast<const void*>(kern));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(units * per);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (pdl_enabled()) {
      attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[na++].val.programmaticStreamSerializationAllowed = 1;
    }
    if (a.pair) {
      attr[na].id = cudaLaunchAttributeClusterDimension;
      attr[na].val.clusterDim.x = per;
      attr[na].val.clusterDim.y = 1;
      attr[na++].val.clusterDim.z = 1;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    PSG_CUDA(cudaLaunchKernelEx(&cfg, kern, ma, mb, mo, a));
  };
  // tc_gemm_kernel's EPI: wgrad (multi-tap column map), dgrad (mask / accumulate), fprop
  const int epi = a.cpt ? 2 : (a.mask || a.accumulate) ? 1 : 0;
  if (a.cpt && (a.mask || a.accumulate)) throw std::logic_error("tc: wgrad epilogue with dgrad operands");
  auto pick = [&](auto k0, auto k1, auto k2) { epi == 0 ? go(k0) : epi == 1 ? go(k1) : go(k2); };
  if (kblk == 32) {
    if (a.pair)
      pick(tc_gemm_kernel<32, true, 0>, tc_gemm_kernel<32, true, 1>, tc_gemm_kernel<32, true, 2>);
    else
      pick(tc_gemm_kernel<32, false, 0>, tc_gemm_kernel<32, false, 1>, tc_gemm_kernel<32, false, 2>);
  } else {
    if (a.pair)
      pick(tc_gemm_kernel<16, true, 0>, tc_gemm_kernel<16, true, 1>, tc_gemm_kernel<16, true, 2>);
    else
      pick(tc_gemm_kernel<16, false, 0>, tc_gemm_kernel<16, false, 1>, tc_gemm_kernel<16, false, 2>);
  }
  PSG_CUDA(cudaGetLastError());
  if (splits > 1) {
    const int nb = a0.bias_chunk ? a0.db_ld : 0;
    const int vcols = a0.valid_cols ? a0.valid_cols : a0.ldo;
    auto al16 = [](const void* q) { return reinterpret_cast<uintptr_t>(q) % 16 == 0; };
    if (a0.ldo % 4 == 0 && vcols % 4 == 0 && out_elems % 4 == 0 && al16(ws) && al16(a0.out) &&
        (!a0.bias || al16(a0.bias)) && (!a0.mask || al16(a0.mask))) {
      const long long total4 = out_elems / 4;
      const int blocks = static_cast<int>(std::min<long long>((total4 + nb + 255) / 256, 148 * 8));
      launch_k(tc_split_reduce4, blocks, 256, 0, s, reinterpret_cast<const float4*>(ws), splits,
               total4, total4, a0.bias, a0.ldo, vcols, a0.relu, a0.accumulate,
               reinterpret_cast<const float4*>(a0.mask), reinterpret_cast<float4*>(a0.out),
               static_cast<const float*>(a.db_part), nb, a0.db);
    } else {
      const int blocks = static_cast<int>(std::min<long long>((out_elems + nb + 255) / 256, 148 * 8));
      launch_k(tc_split_reduce, blocks, 256, 0, s, ws, splits, out_elems, out_elems, a0.bias,
               a0.ldo, vcols, a0.relu, a0.accumulate, a0.mask, a0.out,
               static_cast<const float*>(a.db_part), nb, a0.db);
    }
    PSG_CUDA(cudaGetLastError());
  }
}

bool is_linear(const ConvGeom& g) {
  return g.H == 1 && g.W == 1 && g.OH == 1 && g.OW == 1 && g.kh == 1 && g.kw == 1;
}

int kblk_for(int channels) { return channels % 32 == 0 ? 32 : (channels % 16 == 0 ? 16 : 0); }

// 16-channel K blocks move 64-byte rows, which the TMA engine serves at about half the
// bytes per clock of 128-byte rows (tools/tma_bench.cu): prefer zero-padded 32-blocks.
bool prefer_k32() {
  static const bool v = [] {
    const char* e = std::getenv("PSG_TC_K32");
    return e ? std::atoi(e) != 0 : false;
  }();
  return v;
}

// --- planners: fill TcArgs (out/bias/flags are set by the caller) -------------
bool plan_fprop(const ConvGeom& g, TcArgs& a, int& kblk) {
  std::memset(&a, 0, sizeof a);
  a.pair_policy = g.tc_pair;
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
  if (g.sh != 1 || g.sw != 1 || g.Fg() % 16) return false;
  kblk = kblk_for(g.Cgs());
  if (kblk == 16 && prefer_k32()) kblk = 0;
  // C/G not a multiple of 16: 32-channel blocks per tap, the tail read as 0 (A: the NHWC
  // input's channels past C read OOB, other groups' channels meet B's OOB zeros; B: W
  // viewed as [F][taps][C/G])
  const bool padded = kblk == 0;
  if (padded) {
    if (g.cs_in % 4 || g.Cgs() % 4) return false;
    kblk = 32;
  }
  a.a_mode = A_RECT_K;
  a.b_mode = padded ? B_3D_K : B_2D_K;
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
  a.cb = (g.Cgs() + kblk - 1) / kblk;
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
  to_im2col(a, g, g.OH, g.OW, 1);
  return true;
}

}  // namespace

// dgrad B from a K-major copy of the weights, Wt[g][c][tap][f] (written per step by
// tc_dgrad_wt_transpose): C/G not a multiple of 64 would otherwise pad an MN-major B to
// whole 64-column pair halves (AlexNet conv2: 48 -> 64); K-major B splits 48 = 2 x 24 rows.
bool tc_dgrad_wt(const ConvGeom& g) {
  static const bool env = [] {
    const char* e = std::getenv("PSG_TC_DGRAD_WT");
    return e ? std::atoi(e) != 0 : true;
  }();
  // small layers (GoogLeNet's 28 x 28 and smaller, cifar10_quick): the transpose launch
  // costs more than the MN-major B's padding; PSG_TC_DGRAD_WT_MIN_PX: the pixel threshold
  static const long long min_px = [] {
    const char* e = std::getenv("PSG_TC_DGRAD_WT_MIN_PX");
    return e ? std::atoll(e) : 65536LL;
  }();
  return env && !is_linear(g) && g.sh == 1 && g.sw == 1 && g.Cgs() % 64 != 0 &&
         g.Cgs() % 16 == 0 && g.Fg() % 32 == 0 &&
         static_cast<long long>(g.n) * g.H * g.W >= min_px;
}

namespace {

__global__ void dgrad_wt_k(const float* __restrict__ w, int Fg, int taps, int Cg, int Kp,
                           float* __restrict__ wt, int total) {
  pdl_enter();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  const int f = i % Fg, r = i / Fg, tap = r % taps, gc = r / taps, g = gc / Cg, c = gc % Cg;
  wt[i] = w[static_cast<size_t>(g * Fg + f) * Kp + tap * Cg + c];
}

}  // namespace

void tc_dgrad_wt_transpose(const ConvGeom& g, const float* w, float* wt, cudaStream_t s) {
  const int taps = g.kh * g.kw, total = g.F * taps * g.Cgs();
  launch_k(dgrad_wt_k, (total + 255) / 256, 256, 0, s, w, g.Fg(), taps, g.Cgs(), g.Kp(), wt,
           total);
  PSG_CUDA(cudaGetLastError());
}

namespace {

bool plan_dgrad(const ConvGeom& g, TcArgs& a, int& kblk) {
  std::memset(&a, 0, sizeof a);
  a.pair_policy = g.tc_pair;
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
  if (g.sh != 1 || g.sw != 1 || g.Cgs() % 4 || g.cs_in % 4) return false;
  kblk = kblk_for(g.Fg());
  if (kblk == 16 && prefer_k32()) kblk = 0;
  if (!kblk) {  // F/G not a multiple of 16: 32-filter blocks, the tail read as 0 (B's 4-D view)
    if (g.Fg() % 4 || g.F % 4) return false;
    kblk = 32;
  }
  a.a_mode = A_RECT_K;   // dY rectangles, taps reversed
  a.b_mode = tc_dgrad_wt(g) ? B_3D_K : B_WT_MN;  // Wt (K-major copy) or W^T (MN-major)
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
  a.cb = (g.Fg() + kblk - 1) / kblk;
  a.kblocks = g.kh * g.kw * a.cb;
  a.a_c_g = g.Fg();
  // B rows per group: W^T (B_WT_MN) takes the group as its own coordinate; the K-major copy
  // Wt[g][c][tap][f] (B_3D_K) stacks the groups' C/G channel rows
  a.b_r_g = a.b_mode == B_3D_K ? g.Cgs() : g.Fg();
  a.kw = g.kw;
  a.ph = g.ph;
  a.pw = g.pw;
  a.sign = -1;
  a.n_valid = g.Cgs();
  a.col_g = g.Cgs();
  a.ldo = g.cs_in;
  to_im2col(a, g, g.H, g.W, -1);
  return true;
}

bool plan_wgrad(const ConvGeom& g, TcArgs& a, int& kblk) {
  std::memset(&a, 0, sizeof a);
  a.pair_policy = g.tc_pair;
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
  // Multi-tap tiles: N spans several taps x (C/G rounded up to 32) channels, so one dY
  // block (A) feeds up to 256 output columns; each 32-column chunk of B is X shifted by its
  // own tap (channels past C/G are loaded but never stored).
  if (g.sh != 1 || g.sw != 1 || g.cs_in % 4 || g.Cgs() < 16 || g.F % 4) return false;
  a.a_mode = A_RECT_MN;  // dY: filters x pixel rectangle
  a.b_mode = B_TAPS_MN;  // X shifted per chunk: (tap, channel) x pixel rectangle
  a.row_map = ROW_LINEAR;
  rect_shape(g.OW, kblk, a.rk, a.wk);
  a.kth = (g.OH + a.rk - 1) / a.rk;
  a.ktw = (g.OW + a.wk - 1) / a.wk;
  a.ntaps = g.kh * g.kw;
  a.cpt = (g.Cgs() + 31) / 32 * 32;
  a.cgs = g.Cgs();
  const int chunks = a.ntaps * a.cpt / 32;
  a.n_tiles = (chunks + 7) / 8;
  a.n_tile = 32 * ((chunks + a.n_tiles - 1) / a.n_tiles);
  a.m_tiles = (g.Fg() + kTileM - 1) / kTileM;
  a.G = g.G;
  a.taps = 1;
  a.kblocks = g.n * a.kth * a.ktw;
  a.a_c_g = g.Fg();
  a.b_n_g = g.Cgs();
  a.kw = g.kw;
  a.ph = g.ph;
  a.pw = g.pw;
  a.m_valid = g.Fg();
  a.n_valid = a.ntaps * a.cpt;
  a.row_g = g.Fg();
  a.ldo = g.Kp();
  a.valid_cols = g.Kf();
  if (use_im2col(2) && g.pw <= 128 && g.ph <= 128 && g.kw <= 128 && g.kh <= 128) {
    // K = linear output pixels (no rectangle padding): dY as a plain [pixels][F] matrix,
    // X chunks as TMA im2col boxes shifted by each chunk's tap
    a.a_mode = A_2D_MN;
    a.b_mode = B_TAPS_IM2COL;
    a.kth = a.ktw = 0;
    a.out_h = g.OH;
    a.out_w = g.OW;
    a.im_lw = -g.pw;
    a.im_lh = -g.ph;
    a.kh = g.kh;
    a.kblocks = (g.n * g.OH * g.OW + kblk - 1) / kblk;
    // a spare chunk in the last N tile (the tiles' chunks exceed the taps' chunks) carries
    // the bias gradient (TcArgs::bias_chunk) instead of a harmless reload
    // (or one more chunk per tile when that costs <= ~10% more MMA operand bytes: AlexNet
    // conv1's 18 chunks in 3 x 6 -> 3 x 7; the separate pass re-reads all of dY)
    if (fuse_wgrad_bias()) {
      const int wider = 32 * ((chunks + 1 + a.n_tiles - 1) / a.n_tiles);
      if (a.n_tiles * (a.n_tile / 32) <= chunks && wider <= 256 &&
          10 * (128 + wider) <= 11 * (128 + a.n_tile))
        a.n_tile = wider;
      // (or, one filter tile, one more N tile: the bias pass's dY re-read and its two
      // launches traded for a second read of the dY tiles — GoogLeNet's 1x1 wgrads over 256
      // / 512 channels)
      if (a.n_tiles * (a.n_tile / 32) <= chunks && a.m_tiles == 1 && bias_tile_enabled()) {
        const int nt = a.n_tiles + 1, w = 32 * ((chunks + 1 + nt - 1) / nt);
        if (w <= 256) {
          a.n_tiles = nt;
          a.n_tile = w;
        }
      }
      if (a.n_tiles * (a.n_tile / 32) > chunks) a.bias_chunk = chunks;
    }
  }
  return true;
}


// MN-major tf32 operands: 128B rows swizzled in 32B chunks (UMMA SWIZZLE_128B_BASE32B).
constexpr CUtensorMapSwizzle kMnSwizzle = CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B;

CUtensorMapSwizzle k_swizzle(int kblk) {
  return kblk == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
}

bool plan_wgrad_col(const ConvGeom& g, TcArgs& a) {
  std::memset(&a, 0, sizeof a);
  a.pair_policy = g.tc_pair;
  if (g.F % 4 || g.Fg() % 4 || g.Kp() % 4) return false;
  a.a_mode = A_2D_MN;   // dY [pixels][F]
  a.b_mode = B_COL_MN;  // col [G][pixels][Kp]
  a.row_map = ROW_LINEAR;
  a.n_tile = pick_n_tile(g.Kf());
  a.m_tiles = (g.Fg() + kTileM - 1) / kTileM;
  a.n_tiles = (g.Kf() + a.n_tile - 1) / a.n_tile;
  a.G = g.G;
  a.taps = 1;
  a.kblocks = static_cast<int>((static_cast<long long>(g.n) * g.OH * g.OW + 31) / 32);
  a.a_c_g = g.Fg();
  a.m_valid = g.Fg();
  a.n_valid = g.Kf();
  a.row_g = g.Fg();
  a.ldo = g.Kp();
  a.valid_cols = g.Kf();  // dW's padding columns Kf..Kp: zero
  return true;
}

// db[f] = sum over rows of dY[row][f], fixed order (row chunks, then chunks).
void bias_grad(const float* dy, long long rows, int F, float* part, float* db, cudaStream_t s) {
  if (rows >= (1LL << 31) || rows * F >= (1LL << 40)) throw std::invalid_argument("bias_grad: too large");
  const bool vec = F % 4 == 0;
  const int units = vec ? F / 4 : F;
  const int cpr = std::min(units, 256), rpi = 256 / cpr;
  const int cblocks = (units + cpr - 1) / cpr;
  const long long want = std::max<long long>(1, std::min<long long>(
      (rows + rpi * 8 - 1) / (rpi * 8), 4 * sm_count() / cblocks));
  const int chunks = static_cast<int>(std::min<long long>(kBiasChunksMax, want));
  const int per = static_cast<int>((rows + chunks - 1) / chunks);
  const dim3 grid(cblocks, chunks);
  if (vec)
    launch_k(bias_grad_partial<float4>, grid, 256, 0, s, reinterpret_cast<const float4*>(dy),
                                                   static_cast<int>(rows), units, per,
                                                   reinterpret_cast<float4*>(part));
  else
    launch_k(bias_grad_partial<float>, grid, 256, 0, s, dy, static_cast<int>(rows), units, per, part);
  PSG_CUDA(cudaGetLastError());
  launch_k(bias_grad_final, (F + 7) / 8, 256, 0, s, part, chunks, F, db);
  PSG_CUDA(cudaGetLastError());
}

// dW split partials followed by the bias-gradient partials (kBiasChunksMax row chunks max).
size_t tc_wgrad_ws_elems(const ConvGeom& g) {
  TcArgs a;
  int kblk;
  if (!plan_wgrad(g, a, kblk)) return 0;
  finish_args(a, kblk, sm_count());
  const int splits = splits_of(a);
  return (splits > 1 ? static_cast<size_t>(splits) * g.F * g.Kp() : 0) +
         kBiasChunksMax * static_cast<size_t>(g.F);
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
  ones_matrix();  // allocated here, outside any stream capture (the nets size workspaces first)
  tc_prof_alloc();
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
  return (splits_of(a) > 1 ? 2 : 1) + (which == 2 && !a.bias_chunk ? 2 : 0);
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
    mb = map_2d(w, g.F, g.cs_in, kblk, a.b_cols, k_swizzle(kblk));
  } else {
    if (a.a_mode == A_IM2COL_K)  // traversal grid OH x OW: upper = pad - (k - 1)
      ma = map_nhwc_im2col(x, g.n, g.H, g.W, g.cs_in, kblk, kTileM, a.im_lw, a.im_lh,
                           g.pw - (g.kw - 1), g.ph - (g.kh - 1), k_swizzle(kblk));
    else
      ma = map_nhwc(x, g.n, g.H, g.W, g.cs_in, kblk, a.wm, a.rm, k_swizzle(kblk));
    if (a.b_mode == B_3D_K) {
      const uint64_t dims[3] = {static_cast<uint64_t>(g.Cgs()),
                                static_cast<uint64_t>(g.kh) * g.kw, static_cast<uint64_t>(g.F)};
      const uint64_t str[2] = {static_cast<uint64_t>(g.Cgs()) * 4,
                               static_cast<uint64_t>(g.Kp()) * 4};
      const uint32_t box[3] = {static_cast<uint32_t>(kblk), 1, static_cast<uint32_t>(a.b_cols)};
      mb = make_map(w, 3, dims, str, box, k_swizzle(kblk));
    } else {
      mb = map_2d(w, g.F, g.Kp(), kblk, a.b_cols, k_swizzle(kblk));
    }
  }
  launch(a, ma, mb, kblk, static_cast<long long>(g.n) * g.OH * g.OW * g.F, ws.ptr, ws.elems, s);
}

void tc_dgrad(const ConvGeom& g, const float* dy, const float* w, float* dx, bool accumulate,
              const Workspace& ws, cudaStream_t s, const float* relu_mask, const float* wt) {
  TcArgs a;
  int kblk;
  if (!plan_dgrad(g, a, kblk)) throw std::logic_error("tc_dgrad: unsupported geometry");
  finish_args(a, kblk, sm_count());
  a.out = dx;
  a.accumulate = accumulate;
  a.mask = relu_mask;
  CUtensorMap ma, mb;
  if (a.a_mode == A_2D_K) {
    ma = map_2d(dy, g.n, g.F, kblk, kTileM, k_swizzle(kblk));
    a.b_one = one_box_enabled() && g.cs_in % 32 == 0 && a.n_tile % 32 == 0 && a.b_cols % 32 == 0;
    mb = a.b_one ? map_mn_chunks(w, g.F, g.cs_in, kblk, (a.b_cols + 31) / 32)
                 : map_2d(w, g.F, g.cs_in, 32, kblk, kMnSwizzle);
  } else {
    if (a.a_mode == A_IM2COL_K)  // traversal grid H x W over dY: lower = -(k-1-p), upper = -p
      ma = map_nhwc_im2col(dy, g.n, g.OH, g.OW, g.F, kblk, kTileM, a.im_lw, a.im_lh, -g.pw,
                           -g.ph, k_swizzle(kblk));
    else
      ma = map_nhwc(dy, g.n, g.OH, g.OW, g.F, kblk, a.wm, a.rm, k_swizzle(kblk));
    if (a.b_mode == B_3D_K) {  // Wt viewed as [G * C/G][taps][F/G], K-major boxes
      if (!wt) throw std::logic_error("tc_dgrad: transposed weights missing");
      const uint64_t taps = static_cast<uint64_t>(g.kh) * g.kw;
      const uint64_t dims[3] = {static_cast<uint64_t>(g.Fg()), taps,
                                static_cast<uint64_t>(g.G) * g.Cgs()};
      const uint64_t str[2] = {static_cast<uint64_t>(g.Fg()) * 4, taps * g.Fg() * 4};
      const uint32_t box[3] = {static_cast<uint32_t>(kblk), 1, static_cast<uint32_t>(a.b_cols)};
      mb = make_map(wt, 3, dims, str, box, k_swizzle(kblk));
    } else if (one_box_enabled() && g.Cgs() % 32 == 0 && a.n_tile % 32 == 0 &&
               a.b_cols % 32 == 0) {  // W as [G][taps][C/G / 32][F/G][32]
      a.b_one = 1;
      const uint64_t taps = static_cast<uint64_t>(g.kh) * g.kw;
      const uint64_t dims[5] = {32, static_cast<uint64_t>(g.Fg()),
                                static_cast<uint64_t>(g.Cgs() / 32), taps,
                                static_cast<uint64_t>(g.G)};
      const uint64_t str[4] = {static_cast<uint64_t>(g.Kp()) * 4, 128,
                               static_cast<uint64_t>(g.Cgs()) * 4,
                               static_cast<uint64_t>(g.Fg()) * g.Kp() * 4};
      const uint32_t box[5] = {32, static_cast<uint32_t>(kblk),
                               static_cast<uint32_t>((a.b_cols + 31) / 32), 1, 1};
      mb = make_map(w, 5, dims, str, box, kMnSwizzle);
    } else {
      const uint64_t dims[4] = {static_cast<uint64_t>(g.Cgs()),
                                static_cast<uint64_t>(g.kh) * g.kw, static_cast<uint64_t>(g.Fg()),
                                static_cast<uint64_t>(g.G)};
      const uint64_t str[3] = {static_cast<uint64_t>(g.Cgs()) * 4,
                               static_cast<uint64_t>(g.Kp()) * 4,
                               static_cast<uint64_t>(g.Fg()) * g.Kp() * 4};
      const uint32_t box[4] = {32, 1, static_cast<uint32_t>(kblk), 1};
      mb = make_map(w, 4, dims, str, box, kMnSwizzle);
    }
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
  const bool a_one = one_box_enabled() && a.a_mode == A_2D_MN && g.F % 32 == 0 &&
                     a.a_c_g % 32 == 0;
  a.a_one = a_one;
  if (a.b_mode == B_TAPS_IM2COL) {
    const long long pixels = static_cast<long long>(g.n) * g.OH * g.OW;
    ma = a_one ? map_mn_chunks(dy, pixels, g.F, kblk, a.a_chunks)
               : map_2d(dy, pixels, g.F, 32, kblk, kMnSwizzle);
    mb = map_nhwc_im2col(x, g.n, g.H, g.W, g.cs_in, 32, kblk, a.im_lw, a.im_lh,
                         g.pw - (g.kw - 1), g.ph - (g.kh - 1), kMnSwizzle);
  } else if (a.a_mode == A_2D_MN) {
    ma = a_one ? map_mn_chunks(dy, g.n, g.F, kblk, a.a_chunks)
               : map_2d(dy, g.n, g.F, 32, kblk, kMnSwizzle);
    a.b_one = one_box_enabled() && g.cs_in % 32 == 0 && a.n_tile % 32 == 0 && a.b_cols % 32 == 0;
    mb = a.b_one ? map_mn_chunks(x, g.n, g.cs_in, kblk, (a.b_cols + 31) / 32)
                 : map_2d(x, g.n, g.cs_in, 32, kblk, kMnSwizzle);
  } else {
    ma = map_nhwc(dy, g.n, g.OH, g.OW, g.F, 32, a.wk, a.rk, kMnSwizzle);
    mb = map_nhwc(x, g.n, g.H, g.W, g.cs_in, 32, a.wk, a.rk, kMnSwizzle);
  }
  const long long dw_elems = static_cast<long long>(g.F) * g.Kp();
  // the split-K workspace holds dW partials; bias partials go after them
  const int splits = splits_of(a);
  float* part = ws.ptr + (splits > 1 ? splits * dw_elems : 0);
  if (a.bias_chunk) {  // dbias from the ones chunk of the same GEMM (+ the split reduce)
    a.db = db;
    a.db_ld = g.F;
  }
  launch(a, ma, mb, kblk, dw_elems, ws.ptr, ws.elems, s);
  if (!a.bias_chunk) bias_grad(dy, static_cast<long long>(g.n) * g.OH * g.OW, g.F, part, db, s);
}

// ---- wgrad of narrow layers against an im2col matrix col[G][n*OH*OW][Kp] ----
// D_g[f][(u,v,c)] = sum_pix dY[pix][g*Fg + f] * col[g][pix][(u,v,c)]: M = Fg, N = Kf
// (wide), K = pixels.  Used when the per-tap rectangles would give tiny tiles
// (F/G < 128, C/G not a multiple of 32) or the layer takes the im2col route anyway.
bool tc_wgrad_col_supported(const ConvGeom& g) {
  TcArgs a;
  return plan_wgrad_col(g, a);
}

size_t tc_wgrad_col_ws_elems(const ConvGeom& g) {
  TcArgs a;
  if (!plan_wgrad_col(g, a)) return 0;
  finish_args(a, 32, sm_count());
  const int splits = splits_of(a);
  return (splits > 1 ? static_cast<size_t>(splits) * g.F * g.Kp() : 0) +
         kBiasChunksMax * static_cast<size_t>(g.F);
}

int tc_wgrad_col_launches(const ConvGeom& g) {
  TcArgs a;
  if (!plan_wgrad_col(g, a)) return -1;
  finish_args(a, 32, sm_count());
  return (splits_of(a) > 1 ? 2 : 1) + 2;
}

void tc_wgrad_col(const ConvGeom& g, const float* col, const float* dy, float* dw, float* db,
                  const Workspace& ws, cudaStream_t s) {
  TcArgs a;
  if (!plan_wgrad_col(g, a)) throw std::logic_error("tc_wgrad_col: unsupported geometry");
  finish_args(a, 32, sm_count());
  a.out = dw;
  const long long pixels = static_cast<long long>(g.n) * g.OH * g.OW;
  const CUtensorMap ma = map_2d(dy, pixels, g.F, 32, 32, kMnSwizzle);
  const uint64_t dims[3] = {static_cast<uint64_t>(g.Kp()), static_cast<uint64_t>(pixels),
                            static_cast<uint64_t>(g.G)};
  const uint64_t str[2] = {static_cast<uint64_t>(g.Kp()) * 4,
                           static_cast<uint64_t>(pixels) * g.Kp() * 4};
  const uint32_t box[3] = {32, 32, 1};
  const CUtensorMap mb = make_map(col, 3, dims, str, box, kMnSwizzle);
  const long long dw_elems = static_cast<long long>(g.F) * g.Kp();
  const int splits = splits_of(a);
  float* part = ws.ptr + (splits > 1 ? splits * dw_elems : 0);
  launch(a, ma, mb, 32, dw_elems, ws.ptr, ws.elems, s);
  bias_grad(dy, pixels, g.F, part, db, s);
}


// Labels and counters of the PSG_TC_PROF launches, one line each (see TcArgs::prof).
std::string tc_prof_report(bool reset) {
  TcProf& pr = tc_prof();
  std::lock_guard<std::mutex> lock(pr.mu);
  std::string out;
  if (!pr.dev) return out;
  std::vector<unsigned long long> h(pr.labels.size() * 8);
  if (!h.empty())
    PSG_CUDA(cudaMemcpy(h.data(), pr.dev, h.size() * sizeof(unsigned long long),
                        cudaMemcpyDeviceToHost));
  for (size_t i = 0; i < pr.labels.size(); ++i) {
    char buf[320];
    std::snprintf(buf, sizeof buf, "%zu|%s|%llu %llu %llu %llu %llu %llu %llu %llu\n", i,
                  pr.labels[i].c_str(), h[i * 8], h[i * 8 + 1], h[i * 8 + 2], h[i * 8 + 3],
                  h[i * 8 + 4], h[i * 8 + 5], h[i * 8 + 6], h[i * 8 + 7]);
    out += buf;
  }
  if (reset) PSG_CUDA(cudaMemset(pr.dev, 0, kProfMax * 8 * sizeof(unsigned long long)));
  return out;
}

}  // namespace psg
