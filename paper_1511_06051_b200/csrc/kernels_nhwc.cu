// NHWC bandwidth kernels with 32-bit index decoding (64-bit integer division is
// emulated on the GPU and was the bottleneck of the first versions): pooling, LRN,
// dropout, batch gather / host-batch staging.  Host wrappers check that every tensor
// fits 32-bit indexing.
#include <algorithm>

#include "psg_internal.h"

namespace psg {
namespace {

inline int grid_for(size_t n, int block = 256, int max_blocks = 148 * 16) {
  const size_t b = (n + block - 1) / block;
  return static_cast<int>(std::max<size_t>(1, std::min<size_t>(b, max_blocks)));
}

inline uint32_t checked32(size_t n, const char* what) {
  if (n >= (1ULL << 31)) throw std::invalid_argument(std::string(what) + ": tensor too large");
  return static_cast<uint32_t>(n);
}

#define GRID_STRIDE32(i, n)                                                 \
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < (n); \
       i += gridDim.x * blockDim.x)

__device__ __forceinline__ uint64_t mix64(uint64_t x) {  // rng.hpp:11-16
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

// ------------------------------------------------------------------ pool ---
// model.hpp:369-406 (max, strict '>' so the first maximum in (u, v) scan order
// wins) with Caffe padding / ceil windows; AVE divides by the window clipped to
// the padded extent.  route = (u * kw + v) relative to the unclipped window.
__global__ void pool_fwd_k(PoolGeom g, const float* __restrict__ x, float* __restrict__ y,
                           uint8_t* __restrict__ route, uint32_t total) {
  GRID_STRIDE32(i, total) {
    const uint32_t c = i % g.C, pix = i / g.C;
    const int ow = static_cast<int>(pix % g.OW), t = static_cast<int>(pix / g.OW);
    const int oh = t % g.OH, b = t / g.OH;
    const int hs0 = oh * g.sh - g.ph, ws0 = ow * g.sw - g.pw;
    const int he0 = hs0 + g.kh, we0 = ws0 + g.kw;
    const int hs = max(hs0, 0), ws = max(ws0, 0), he = min(he0, g.H), we = min(we0, g.W);
    const float* xb = x + (static_cast<size_t>(b) * g.H * g.W) * g.C + c;
    if (g.method == PSG_POOL_AVE) {
      const int size = (min(he0, g.H + g.ph) - hs0) * (min(we0, g.W + g.pw) - ws0);
      float acc = 0.f;
      for (int r = hs; r < he; ++r)
        for (int s = ws; s < we; ++s) acc += xb[(r * g.W + s) * g.C];
      y[i] = acc / static_cast<float>(size);
    } else {
      float best = xb[(hs * g.W + ws) * g.C];
      int arg = (hs - hs0) * g.kw + (ws - ws0);
      for (int r = hs; r < he; ++r) {
        for (int s = ws; s < we; ++s) {
          const float v = xb[(r * g.W + s) * g.C];
          if (v > best) {
            best = v;
            arg = (r - hs0) * g.kw + (s - ws0);
          }
        }
      }
      y[i] = best;
      route[i] = static_cast<uint8_t>(arg);
    }
  }
}

// model.hpp:492-498 as a deterministic gather: each input sums, in ascending
// output order, the dy of the covering windows that routed to it.
__global__ void pool_bwd_k(PoolGeom g, const float* __restrict__ dy,
                           const uint8_t* __restrict__ route, float* __restrict__ dx,
                           int accumulate, uint32_t total) {
  GRID_STRIDE32(i, total) {
    const uint32_t c = i % g.C, pix = i / g.C;
    const int w = static_cast<int>(pix % g.W), t = static_cast<int>(pix / g.W);
    const int h = t % g.H, b = t / g.H;
    // windows with oh*sh - ph <= h < oh*sh - ph + kh
    const int ohl = max(0, (h + g.ph - g.kh + g.sh) / g.sh);
    const int ohh = min(g.OH - 1, (h + g.ph) / g.sh);
    const int owl = max(0, (w + g.pw - g.kw + g.sw) / g.sw);
    const int owh = min(g.OW - 1, (w + g.pw) / g.sw);
    const uint32_t obase = static_cast<uint32_t>(b) * g.OH * g.OW;
    float acc = 0.f;
    for (int oh = ohl; oh <= ohh; ++oh) {
      const int hs0 = oh * g.sh - g.ph;
      if (h < hs0 || h >= hs0 + g.kh) continue;
      for (int ow = owl; ow <= owh; ++ow) {
        const int ws0 = ow * g.sw - g.pw;
        if (w < ws0 || w >= ws0 + g.kw) continue;
        const uint32_t o = (obase + oh * g.OW + ow) * g.C + c;
        if (g.method == PSG_POOL_AVE) {
          const int size =
              (min(hs0 + g.kh, g.H + g.ph) - hs0) * (min(ws0 + g.kw, g.W + g.pw) - ws0);
          acc += dy[o] / static_cast<float>(size);
        } else if (route[o] == (h - hs0) * g.kw + (w - ws0)) {
          acc += dy[o];
        }
      }
    }
    dx[i] = accumulate ? dx[i] + acc : acc;
  }
}

// ------------------------------------------------------------------- lrn ---
// Caffe LRN ACROSS_CHANNELS.  One warp per pixel: the pixel's C channels are staged
// in shared memory, window sums read them from there (each value read once from HBM).
// The scale is recomputed in backward instead of being stored.
constexpr int kLrnWarps = 8;

__global__ void lrn_fwd_k(LrnGeom g, const float* __restrict__ x, float* __restrict__ y) {
  extern __shared__ float sm[];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  float* sx = sm + warp * g.C;
  const int pre = (g.size - 1) / 2, post = g.size - pre - 1;
  const float a = g.alpha / g.size;
  for (uint32_t p = blockIdx.x * kLrnWarps + warp; p < static_cast<uint32_t>(g.pixels);
       p += gridDim.x * kLrnWarps) {
    const float* xp = x + static_cast<size_t>(p) * g.C;
    for (int c = lane; c < g.C; c += 32) {
      const float v = xp[c];
      sx[c] = v * v;
    }
    __syncwarp();
    for (int c = lane; c < g.C; c += 32) {
      const int lo = max(0, c - pre), hi = min(g.C - 1, c + post);
      float acc = 0.f;
      for (int q = lo; q <= hi; ++q) acc += sx[q];
      const float s = g.k + a * acc;
      y[static_cast<size_t>(p) * g.C + c] = xp[c] * powf(s, -g.beta);
    }
    __syncwarp();
  }
}

__global__ void lrn_bwd_k(LrnGeom g, const float* __restrict__ x, const float* __restrict__ dy,
                          float* __restrict__ dx, int accumulate) {
  extern __shared__ float sm[];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  float* sx = sm + warp * 3 * g.C;  // x^2
  float* st = sx + g.C;             // dy * y / scale
  float* ssp = st + g.C;            // scale^-beta
  const int pre = (g.size - 1) / 2, post = g.size - pre - 1;
  const float a = g.alpha / g.size, ratio = 2.f * g.alpha * g.beta / g.size;
  for (uint32_t p = blockIdx.x * kLrnWarps + warp; p < static_cast<uint32_t>(g.pixels);
       p += gridDim.x * kLrnWarps) {
    const size_t base = static_cast<size_t>(p) * g.C;
    for (int c = lane; c < g.C; c += 32) {
      const float v = x[base + c];
      sx[c] = v * v;
    }
    __syncwarp();
    for (int c = lane; c < g.C; c += 32) {
      const int lo = max(0, c - pre), hi = min(g.C - 1, c + post);
      float acc = 0.f;
      for (int q = lo; q <= hi; ++q) acc += sx[q];
      const float s = g.k + a * acc;
      const float sp = powf(s, -g.beta);
      ssp[c] = sp;
      st[c] = dy[base + c] * x[base + c] * sp / s;
    }
    __syncwarp();
    for (int c = lane; c < g.C; c += 32) {
      // channels q whose window contains c: q in [c - post, c + pre]
      const int lo = max(0, c - post), hi = min(g.C - 1, c + pre);
      float acc = 0.f;
      for (int q = lo; q <= hi; ++q) acc += st[q];
      const float v = dy[base + c] * ssp[c] - ratio * x[base + c] * acc;
      dx[base + c] = accumulate ? dx[base + c] + v : v;
    }
    __syncwarp();
  }
}

// --------------------------------------------------------------- dropout ---
// Keep-mask = splitmix64(mix(base ^ step) + nchw_index) >> 40 >= ratio * 2^24.
__device__ __forceinline__ float drop_mask(const DropGeom& g, uint64_t base, uint32_t i,
                                           uint32_t thresh, float keep) {
  const uint32_t c = i % g.C, t = i / g.C;
  const uint32_t w = t % g.W, t2 = t / g.W;
  const uint32_t h = t2 % g.H, b = t2 / g.H;
  const uint64_t nchw = ((static_cast<uint64_t>(b) * g.C + c) * g.H + h) * g.W + w;
  const uint32_t u = static_cast<uint32_t>(mix64(base + nchw) >> 40);
  return u >= thresh ? keep : 0.f;
}

__global__ void dropout_fwd_k(DropGeom g, const float* __restrict__ x, float* __restrict__ y,
                              const uint64_t* __restrict__ d_step, int train, uint32_t total) {
  if (!train) {
    GRID_STRIDE32(i, total) y[i] = x[i];
    return;
  }
  const uint64_t base = mix64(g.base_seed ^ *d_step);
  const uint32_t thresh = static_cast<uint32_t>(static_cast<double>(g.ratio) * 16777216.0);
  const float keep = static_cast<float>(1.0 / (1.0 - static_cast<double>(g.ratio)));
  GRID_STRIDE32(i, total) y[i] = x[i] * drop_mask(g, base, i, thresh, keep);
}

__global__ void dropout_bwd_k(DropGeom g, const float* __restrict__ dy, float* __restrict__ dx,
                              const uint64_t* __restrict__ d_step, int accumulate,
                              uint32_t total) {
  const uint64_t base = mix64(g.base_seed ^ *d_step);
  const uint32_t thresh = static_cast<uint32_t>(static_cast<double>(g.ratio) * 16777216.0);
  const float keep = static_cast<float>(1.0 / (1.0 - static_cast<double>(g.ratio)));
  GRID_STRIDE32(i, total) {
    const float v = dy[i] * drop_mask(g, base, i, thresh, keep);
    dx[i] = accumulate ? dx[i] + v : v;
  }
}

// ---------------------------------------------------------------- gather ---
// data.hpp:292-304 gather_batch from the HBM-resident shard (NHWC rows).
__global__ void gather_k(const float* __restrict__ ds, const int32_t* __restrict__ ds_labels,
                         const uint32_t* __restrict__ idx, const int* __restrict__ cursor, int b,
                         int pixels, int C, int cs, float* __restrict__ out,
                         int32_t* __restrict__ labels) {
  const int i = blockIdx.y;
  const uint32_t row = idx[static_cast<size_t>(cursor ? *cursor : 0) * b + i];
  const float* src = ds + static_cast<size_t>(row) * pixels * C;
  float* dst = out + static_cast<size_t>(i) * pixels * cs;
  if (blockIdx.x == 0 && threadIdx.x == 0) labels[i] = ds_labels[row];
  const uint32_t stride = gridDim.x * blockDim.x;
  if (cs == C) {
    const uint32_t n = static_cast<uint32_t>(pixels) * C;
    if ((n % 4) == 0) {
      const float4* s4 = reinterpret_cast<const float4*>(src);
      float4* d4 = reinterpret_cast<float4*>(dst);
      for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n / 4; j += stride)
        d4[j] = __ldg(s4 + j);
    } else {
      for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride)
        dst[j] = __ldg(src + j);
    }
  } else {
    const uint32_t n = static_cast<uint32_t>(pixels) * cs;
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride) {
      const uint32_t c = j % cs, p = j / cs;
      dst[j] = c < static_cast<uint32_t>(C) ? __ldg(src + p * C + c) : 0.f;
    }
  }
}

// Host-fed batch (reference NCHW layout) -> data layer NHWC with channel stride cs.
__global__ void stage_nchw_k(const float* __restrict__ src, int C, int H, int W, int cs,
                             float* __restrict__ dst, uint32_t total) {
  GRID_STRIDE32(i, total) {
    const uint32_t c = i % cs, t = i / cs;
    const uint32_t w = t % W, t2 = t / W;
    const uint32_t h = t2 % H, b = t2 / H;
    dst[i] = c < static_cast<uint32_t>(C) ? src[((static_cast<size_t>(b) * C + c) * H + h) * W + w]
                                          : 0.f;
  }
}

}  // namespace

void pool_fwd(const PoolGeom& g, const float* x, float* y, uint8_t* route, cudaStream_t s) {
  const uint32_t n = checked32(static_cast<size_t>(g.n) * g.OH * g.OW * g.C, "pool");
  checked32(static_cast<size_t>(g.n) * g.H * g.W * g.C, "pool");
  pool_fwd_k<<<grid_for(n), 256, 0, s>>>(g, x, y, route, n);
  PSG_CUDA(cudaGetLastError());
}

void pool_bwd(const PoolGeom& g, const float* dy, const uint8_t* route, float* dx,
              bool accumulate, cudaStream_t s) {
  const uint32_t n = checked32(static_cast<size_t>(g.n) * g.H * g.W * g.C, "pool");
  pool_bwd_k<<<grid_for(n), 256, 0, s>>>(g, dy, route, dx, accumulate, n);
  PSG_CUDA(cudaGetLastError());
}

void lrn_fwd(const LrnGeom& g, const float* x, float* y, cudaStream_t s) {
  checked32(static_cast<size_t>(g.pixels) * g.C, "lrn");
  const int blocks = static_cast<int>(std::min<long>((g.pixels + kLrnWarps - 1) / kLrnWarps,
                                                     148L * 8));
  lrn_fwd_k<<<blocks, 32 * kLrnWarps, kLrnWarps * g.C * sizeof(float), s>>>(g, x, y);
  PSG_CUDA(cudaGetLastError());
}

void lrn_bwd(const LrnGeom& g, const float* x, const float* dy, float* dx, bool accumulate,
             cudaStream_t s) {
  checked32(static_cast<size_t>(g.pixels) * g.C, "lrn");
  const int blocks = static_cast<int>(std::min<long>((g.pixels + kLrnWarps - 1) / kLrnWarps,
                                                     148L * 8));
  lrn_bwd_k<<<blocks, 32 * kLrnWarps, 3 * kLrnWarps * g.C * sizeof(float), s>>>(g, x, dy, dx,
                                                                               accumulate);
  PSG_CUDA(cudaGetLastError());
}

void dropout_fwd(const DropGeom& g, const float* x, float* y, const uint64_t* d_step, bool train,
                 cudaStream_t s) {
  const uint32_t n = checked32(static_cast<size_t>(g.n) * g.C * g.H * g.W, "dropout");
  dropout_fwd_k<<<grid_for(n), 256, 0, s>>>(g, x, y, d_step, train, n);
  PSG_CUDA(cudaGetLastError());
}

void dropout_bwd(const DropGeom& g, const float* dy, float* dx, const uint64_t* d_step,
                 bool accumulate, cudaStream_t s) {
  const uint32_t n = checked32(static_cast<size_t>(g.n) * g.C * g.H * g.W, "dropout");
  dropout_bwd_k<<<grid_for(n), 256, 0, s>>>(g, dy, dx, d_step, accumulate, n);
  PSG_CUDA(cudaGetLastError());
}

void gather_batch(const float* ds_images, const int32_t* ds_labels, const uint32_t* idx,
                  const int* cursor, int b, int pixels, int C, int cs, float* out,
                  int32_t* labels, cudaStream_t s) {
  const size_t per_row = checked32(static_cast<size_t>(pixels) * cs, "gather");
  const int bx = static_cast<int>(std::max<size_t>(1, std::min<size_t>((per_row / 4 + 255) / 256, 64)));
  gather_k<<<dim3(bx, b), 256, 0, s>>>(ds_images, ds_labels, idx, cursor, b, pixels, C, cs, out,
                                       labels);
  PSG_CUDA(cudaGetLastError());
}

void stage_batch_nchw(const float* src, int n, int C, int H, int W, int cs, float* dst,
                      cudaStream_t s) {
  const uint32_t total = checked32(static_cast<size_t>(n) * H * W * cs, "stage");
  stage_nchw_k<<<grid_for(total), 256, 0, s>>>(src, C, H, W, cs, dst, total);
  PSG_CUDA(cudaGetLastError());
}

}  // namespace psg
