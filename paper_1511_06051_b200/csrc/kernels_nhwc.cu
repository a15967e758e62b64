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
// V = float4 (4 channels per thread, C % 4 == 0) or float; index math per V.
__device__ __forceinline__ float comp(const float4& v, int j) {
  return j == 0 ? v.x : j == 1 ? v.y : j == 2 ? v.z : v.w;
}
__device__ __forceinline__ float& comp(float4& v, int j) {
  return j == 0 ? v.x : j == 1 ? v.y : j == 2 ? v.z : v.w;
}
__device__ __forceinline__ float comp(const float& v, int) { return v; }
__device__ __forceinline__ float& comp(float& v, int) { return v; }
template <typename V> struct RouteOf;
template <> struct RouteOf<float4> { using T = uchar4; static constexpr int n = 4; };
template <> struct RouteOf<float> { using T = uint8_t; static constexpr int n = 1; };
__device__ __forceinline__ uint8_t rcomp(const uchar4& r, int j) {
  return j == 0 ? r.x : j == 1 ? r.y : j == 2 ? r.z : r.w;
}
__device__ __forceinline__ uint8_t& rcomp(uchar4& r, int j) {
  return j == 0 ? r.x : j == 1 ? r.y : j == 2 ? r.z : r.w;
}
__device__ __forceinline__ uint8_t rcomp(const uint8_t& r, int) { return r; }
__device__ __forceinline__ uint8_t& rcomp(uint8_t& r, int) { return r; }

// One block per output row (b, oh) in forward / input row (b, h) in backward: the row's
// window ranges are decoded once per block; threads walk (column, channel-vector) pairs
// with incremental indices (no per-element division).
template <typename V, int K>
__global__ void __launch_bounds__(256) pool_fwd_k(PoolGeom g, const V* __restrict__ x,
                                                  V* __restrict__ y,
                                                  typename RouteOf<V>::T* __restrict__ route,
                                                  int cv) {
  pdl_enter();
  constexpr int L = RouteOf<V>::n;
  const int oh = blockIdx.x % g.OH, b = blockIdx.x / g.OH;
  const int hs0 = oh * g.sh - g.ph, he0 = hs0 + g.kh;
  const int hs = max(hs0, 0), he = min(he0, g.H);
  const V* xb = x + static_cast<size_t>(b) * g.H * g.W * cv;
  const size_t ybase = static_cast<size_t>(blockIdx.x) * g.OW * cv;
  const int total = g.OW * cv, step_c = blockDim.x % cv, step_w = blockDim.x / cv;
  int c = threadIdx.x % cv, ow = threadIdx.x / cv;
  for (int j = threadIdx.x; j < total; j += blockDim.x) {
    const int ws0 = ow * g.sw - g.pw, we0 = ws0 + g.kw;
    const int ws = max(ws0, 0), we = min(we0, g.W);
    if constexpr (K > 0) {
      // K x K window (kh = kw = K): all taps loaded first (predicated), then reduced in
      // (u, v) scan order — the same arithmetic as the runtime-bound loops below
      V v[K > 0 ? K * K : 1];
#pragma unroll
      for (int u = 0; u < K; ++u)
#pragma unroll
        for (int q = 0; q < K; ++q) {
          const int r = hs0 + u, t = ws0 + q;
          if (r >= hs && r < he && t >= ws && t < we) v[u * K + q] = __ldg(xb + (r * g.W + t) * cv + c);
        }
      if (g.method == PSG_POOL_AVE) {
        const float size = static_cast<float>((min(he0, g.H + g.ph) - hs0) *
                                              (min(we0, g.W + g.pw) - ws0));
        V acc;
#pragma unroll
        for (int q = 0; q < L; ++q) comp(acc, q) = 0.f;
#pragma unroll
        for (int u = 0; u < K; ++u)
#pragma unroll
          for (int q = 0; q < K; ++q) {
            const int r = hs0 + u, t = ws0 + q;
            if (r >= hs && r < he && t >= ws && t < we)
#pragma unroll
              for (int e = 0; e < L; ++e) comp(acc, e) += comp(v[u * K + q], e);
          }
#pragma unroll
        for (int q = 0; q < L; ++q) comp(acc, q) = comp(acc, q) / size;
        y[ybase + j] = acc;
      } else {
        V best;  // the first valid tap, then strict '>' in scan order
        typename RouteOf<V>::T arg;
        bool have = false;
#pragma unroll
        for (int u = 0; u < K; ++u)
#pragma unroll
          for (int q = 0; q < K; ++q) {
            const int r = hs0 + u, t = ws0 + q;
            if (r >= hs && r < he && t >= ws && t < we) {
              if (!have) {
                best = v[u * K + q];
#pragma unroll
                for (int e = 0; e < L; ++e) rcomp(arg, e) = static_cast<uint8_t>(u * K + q);
                have = true;
                continue;
              }
#pragma unroll
              for (int e = 0; e < L; ++e)
                if (comp(v[u * K + q], e) > comp(best, e)) {
                  comp(best, e) = comp(v[u * K + q], e);
                  rcomp(arg, e) = static_cast<uint8_t>(u * K + q);
                }
            }
          }
        y[ybase + j] = best;
        route[ybase + j] = arg;
      }
    } else if (g.method == PSG_POOL_AVE) {
      const float size = static_cast<float>((min(he0, g.H + g.ph) - hs0) *
                                            (min(we0, g.W + g.pw) - ws0));
      V acc;
#pragma unroll
      for (int q = 0; q < L; ++q) comp(acc, q) = 0.f;
      for (int r = hs; r < he; ++r)
        for (int t = ws; t < we; ++t) {
          const V v = __ldg(xb + (r * g.W + t) * cv + c);
#pragma unroll
          for (int q = 0; q < L; ++q) comp(acc, q) += comp(v, q);
        }
#pragma unroll
      for (int q = 0; q < L; ++q) comp(acc, q) = comp(acc, q) / size;
      y[ybase + j] = acc;
    } else {
      V best = __ldg(xb + (hs * g.W + ws) * cv + c);
      typename RouteOf<V>::T arg;
      const uint8_t a0 = static_cast<uint8_t>((hs - hs0) * g.kw + (ws - ws0));
#pragma unroll
      for (int q = 0; q < L; ++q) rcomp(arg, q) = a0;
      for (int r = hs; r < he; ++r) {
        for (int t = ws; t < we; ++t) {
          const V v = __ldg(xb + (r * g.W + t) * cv + c);
          const uint8_t a = static_cast<uint8_t>((r - hs0) * g.kw + (t - ws0));
#pragma unroll
          for (int q = 0; q < L; ++q)
            if (comp(v, q) > comp(best, q)) {
              comp(best, q) = comp(v, q);
              rcomp(arg, q) = a;
            }
        }
      }
      y[ybase + j] = best;
      route[ybase + j] = arg;
    }
    c += step_c;
    ow += step_w;
    if (c >= cv) {
      c -= cv;
      ++ow;
    }
  }
}

// model.hpp:492-498 as a deterministic gather: each input sums, in ascending
// output order, the dy of the covering windows that routed to it.
// KS > 0: kh = kw = KS and sh = sw = SS at compile time (the window / stride divisions and
// bounds checks become constants; same arithmetic, same summation order).
template <typename V, int KS, int SS>
__global__ void __launch_bounds__(256) pool_bwd_k(PoolGeom g, const V* __restrict__ dy,
                                                  const typename RouteOf<V>::T* __restrict__ route,
                                                  V* __restrict__ dx, int accumulate, int cv,
                                                  const V* __restrict__ mask, int loads_first) {
  pdl_enter();
  constexpr int L = RouteOf<V>::n;
  const int kh = KS > 0 ? KS : g.kh, kw = KS > 0 ? KS : g.kw;
  const int sh = KS > 0 ? SS : g.sh, sw = KS > 0 ? SS : g.sw;
  const int h = blockIdx.x % g.H, b = blockIdx.x / g.H;
  // windows with oh*sh - ph <= h < oh*sh - ph + kh
  const int ohl = max(0, (h + g.ph - kh + sh) / sh);
  const int ohh = min(g.OH - 1, (h + g.ph) / sh);
  const uint32_t obase = static_cast<uint32_t>(b) * g.OH * g.OW;
  const size_t xbase = static_cast<size_t>(blockIdx.x) * g.W * cv;
  const int total = g.W * cv, step_c = blockDim.x % cv, step_w = blockDim.x / cv;
  int c = threadIdx.x % cv, w = threadIdx.x / cv;
  if constexpr (KS > 0) {
    if (g.method == PSG_POOL_MAX && loads_first) {
      // every covering window's dy and route loaded before any is used (NW x NW candidates,
      // predicated), then summed in the same ascending (oh, ow) order as the loop below
      constexpr int NW = (KS + SS - 1) / SS;
      using RT = typename RouteOf<V>::T;
      for (int j = threadIdx.x; j < total; j += blockDim.x) {
        const int owl = max(0, (w + g.pw - kw + sw) / sw);
        const int owh = min(g.OW - 1, (w + g.pw) / sw);
        V dd[NW][NW];
        RT rr[NW][NW];
        bool ok[NW][NW];
#pragma unroll
        for (int i = 0; i < NW; ++i)
#pragma unroll
          for (int q = 0; q < NW; ++q) {
            const int oh = ohl + i, ow = owl + q;
            const int hs0 = oh * sh - g.ph, ws0 = ow * sw - g.pw;
            ok[i][q] = oh <= ohh && ow <= owh && h >= hs0 && h < hs0 + kh && w >= ws0 &&
                       w < ws0 + kw;
            if (ok[i][q]) {
              const uint32_t o = (obase + oh * g.OW + ow) * cv + c;
              dd[i][q] = __ldg(dy + o);
              rr[i][q] = __ldg(route + o);
            }
          }
        V m, o;
        if (mask) m = __ldg(mask + xbase + j);
        if (accumulate) o = dx[xbase + j];
        V acc;
#pragma unroll
        for (int e = 0; e < L; ++e) comp(acc, e) = 0.f;
#pragma unroll
        for (int i = 0; i < NW; ++i)
#pragma unroll
          for (int q = 0; q < NW; ++q) {
            const int hs0 = (ohl + i) * sh - g.ph, ws0 = (owl + q) * sw - g.pw;
            const uint8_t want = static_cast<uint8_t>((h - hs0) * kw + (w - ws0));
            if (!ok[i][q]) continue;
#pragma unroll
            for (int e = 0; e < L; ++e)
              if (rcomp(rr[i][q], e) == want) comp(acc, e) += comp(dd[i][q], e);
          }
        if (mask) {
#pragma unroll
          for (int e = 0; e < L; ++e)
            if (!(comp(m, e) > 0.f)) comp(acc, e) = 0.f;
        }
        if (accumulate) {
#pragma unroll
          for (int e = 0; e < L; ++e) comp(acc, e) += comp(o, e);
        }
        dx[xbase + j] = acc;
        c += step_c;
        w += step_w;
        if (c >= cv) {
          c -= cv;
          ++w;
        }
      }
      return;
    }
  }
  for (int j = threadIdx.x; j < total; j += blockDim.x) {
    const int owl = max(0, (w + g.pw - kw + sw) / sw);
    const int owh = min(g.OW - 1, (w + g.pw) / sw);
    V acc;
#pragma unroll
    for (int q = 0; q < L; ++q) comp(acc, q) = 0.f;
    for (int oh = ohl; oh <= ohh; ++oh) {
      const int hs0 = oh * sh - g.ph;
      if (h < hs0 || h >= hs0 + kh) continue;
      for (int ow = owl; ow <= owh; ++ow) {
        const int ws0 = ow * sw - g.pw;
        if (w < ws0 || w >= ws0 + kw) continue;
        const uint32_t o = (obase + oh * g.OW + ow) * cv + c;
        const V d = __ldg(dy + o);
        if (g.method == PSG_POOL_AVE) {
          const float size = static_cast<float>((min(hs0 + kh, g.H + g.ph) - hs0) *
                                                (min(ws0 + kw, g.W + g.pw) - ws0));
#pragma unroll
          for (int q = 0; q < L; ++q) comp(acc, q) += comp(d, q) / size;
        } else {
          const typename RouteOf<V>::T r = __ldg(route + o);
          const uint8_t want = static_cast<uint8_t>((h - hs0) * kw + (w - ws0));
#pragma unroll
          for (int q = 0; q < L; ++q)
            if (rcomp(r, q) == want) comp(acc, q) += comp(d, q);
        }
      }
    }
    if (mask) {
      const V m = __ldg(mask + xbase + j);
#pragma unroll
      for (int q = 0; q < L; ++q)
        if (!(comp(m, q) > 0.f)) comp(acc, q) = 0.f;
    }
    if (accumulate) {
      const V o = dx[xbase + j];
#pragma unroll
      for (int q = 0; q < L; ++q) comp(acc, q) += comp(o, q);
    }
    dx[xbase + j] = acc;
    c += step_c;
    w += step_w;
    if (c >= cv) {
      c -= cv;
      ++w;
    }
  }
}

// ------------------------------------------------------------------- lrn ---
// Caffe LRN ACROSS_CHANNELS over NHWC.  A block stages a tile of whole pixels (a
// contiguous run of tp*C floats) in shared memory with independent coalesced loads, then
// every window sum reads shared memory; thread e's channel advances incrementally
// (c += 256 % C) so there is no per-element division.  The window (SIZE taps, a template
// parameter for the common size 5) is unrolled with predicated taps, summed in ascending
// channel order; s^-beta uses the SFU exp2/log2 (relative error ~1e-6, inside the 1e-5
// strict bar).  The scale is recomputed in backward instead of being stored.
constexpr int kLrnThreads = 256;
constexpr int kLrnTileElems = 2048;

__device__ __forceinline__ float lrn_pow(float s, float beta) {  // s^-beta, s >= k > 0
  float l, r;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l) : "f"(s));
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(__fmul_rn(-beta, l)));
  return r;
}

// sum over q in [lo_off, hi_off] of f(row[c + q]) for taps inside [0, C), ascending q.
template <int SIZE, bool SQUARE>
__device__ __forceinline__ float lrn_window(const float* row, int c, int C, int lo_off, int n) {
  float acc = 0.f;
  if (SIZE > 0) {
#pragma unroll
    for (int q = 0; q < SIZE; ++q) {
      const int ch = c + lo_off + q;
      if (ch >= 0 && ch < C) {
        const float v = row[ch];
        acc += SQUARE ? v * v : v;
      }
    }
  } else {
    for (int q = 0; q < n; ++q) {
      const int ch = c + lo_off + q;
      if (ch >= 0 && ch < C) {
        const float v = row[ch];
        acc += SQUARE ? v * v : v;
      }
    }
  }
  return acc;
}

template <int SIZE>
__global__ void __launch_bounds__(kLrnThreads) lrn_fwd_k(LrnGeom g, const float* __restrict__ x,
                                                         float* __restrict__ y, int tp) {
  pdl_enter();
  extern __shared__ float sm[];
  float* sx = sm;
  const int pre = (g.size - 1) / 2, C = g.C;
  const float a = g.alpha / g.size;
  const int ntiles = (g.pixels + tp - 1) / tp, step = kLrnThreads % C;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const size_t e0 = static_cast<size_t>(tile) * tp * C;
    const int ne = min(tp, g.pixels - tile * tp) * C;
#pragma unroll 8
    for (int e = threadIdx.x; e < ne; e += kLrnThreads) sx[e] = __ldg(x + e0 + e);
    __syncthreads();
    int c = threadIdx.x % C;
    for (int e = threadIdx.x; e < ne; e += kLrnThreads) {
      const float acc = lrn_window<SIZE, true>(sx + (e - c), c, C, -pre, g.size);
      y[e0 + e] = sx[e] * lrn_pow(g.k + a * acc, g.beta);
      c += step;
      if (c >= C) c -= C;
    }
    __syncthreads();
  }
}

template <int SIZE>
__global__ void __launch_bounds__(kLrnThreads) lrn_bwd_k(LrnGeom g, const float* __restrict__ x,
                                                         const float* __restrict__ dy,
                                                         float* __restrict__ dx, int accumulate,
                                                         int relu_mask, int tp) {
  pdl_enter();
  extern __shared__ float sm[];
  const int C = g.C, tile_elems = tp * C;
  float* sx = sm;                   // x
  float* sd = sx + tile_elems;      // dy
  float* st = sd + tile_elems;      // dy * y / scale
  float* ssp = st + tile_elems;     // scale^-beta
  const int pre = (g.size - 1) / 2, post = g.size - pre - 1;
  const float a = g.alpha / g.size, ratio = 2.f * g.alpha * g.beta / g.size;
  const int ntiles = (g.pixels + tp - 1) / tp, step = kLrnThreads % C;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const size_t e0 = static_cast<size_t>(tile) * tp * C;
    const int ne = min(tp, g.pixels - tile * tp) * C;
#pragma unroll 8
    for (int e = threadIdx.x; e < ne; e += kLrnThreads) {
      sx[e] = __ldg(x + e0 + e);
      sd[e] = __ldg(dy + e0 + e);
    }
    __syncthreads();
    int c = threadIdx.x % C;
    for (int e = threadIdx.x; e < ne; e += kLrnThreads) {
      const float s = g.k + a * lrn_window<SIZE, true>(sx + (e - c), c, C, -pre, g.size);
      const float sp = lrn_pow(s, g.beta);
      ssp[e] = sp;
      st[e] = sd[e] * sx[e] * sp * __frcp_rn(s);
      c += step;
      if (c >= C) c -= C;
    }
    __syncthreads();
    c = threadIdx.x % C;
    for (int e = threadIdx.x; e < ne; e += kLrnThreads) {
      // channels q whose window contains c: q in [c - post, c + pre]
      const float acc = lrn_window<SIZE, false>(st + (e - c), c, C, -post, g.size);
      float v = sd[e] * ssp[e] - ratio * sx[e] * acc;
      if (relu_mask && !(sx[e] > 0.f)) v = 0.f;
      dx[e0 + e] = accumulate ? dx[e0 + e] + v : v;
      c += step;
      if (c >= C) c -= C;
    }
    __syncthreads();
  }
}

// Streaming LRN for size 5 and C % 8 == 0 (AlexNet / GoogLeNet): thread = 8 consecutive
// channels of one pixel, no shared memory and no barriers — each thread loads its run plus
// the neighbouring channels it needs (float4, the neighbours mostly L1 hits) and keeps the
// window sums in registers (same ascending 5-term sums as the tile kernels).  Channels
// outside [0, C) read as zero.
// The streaming LRN kernels (standalone and fused with the max pool) evaluate every
// channel through these helpers with explicitly rounded operations (no compiler FMA
// contraction choices), so the fused and unfused paths agree bit for bit.
__device__ __forceinline__ float lrn_sq5(const float* w) {  // sum of 5 squares, ascending
  float acc = 0.f;
#pragma unroll
  for (int q = 0; q < 5; ++q) acc = __fmaf_rn(w[q], w[q], acc);
  return acc;
}
__device__ __forceinline__ float lrn_sum5(const float* w) {
  float acc = 0.f;
#pragma unroll
  for (int q = 0; q < 5; ++q) acc = __fadd_rn(acc, w[q]);
  return acc;
}
__device__ __forceinline__ float lrn_scale(float k, float a, float sq) { return __fmaf_rn(a, sq, k); }
// dy * x * s^-beta / s (the term each channel contributes to its neighbours' gradients)
__device__ __forceinline__ float lrn_st(float d, float x, float sp, float sc) {
  return __fmul_rn(__fmul_rn(__fmul_rn(d, x), sp), __frcp_rn(sc));
}
__device__ __forceinline__ float lrn_dx(float d, float sp, float ratio, float x, float sum_st) {
  return __fsub_rn(__fmul_rn(d, sp), __fmul_rn(__fmul_rn(ratio, x), sum_st));
}

constexpr int kLrnRun = 8;

__device__ __forceinline__ float4 lrn_ld4(const float* p, int c, int C) {
  return (c >= 0 && c < C) ? __ldg(reinterpret_cast<const float4*>(p + c))
                           : make_float4(0.f, 0.f, 0.f, 0.f);
}
__device__ __forceinline__ void lrn_put4(float* v, float4 q) {
  v[0] = q.x;
  v[1] = q.y;
  v[2] = q.z;
  v[3] = q.w;
}

__global__ void __launch_bounds__(256) lrn_fwd_run_k(LrnGeom g, const float* __restrict__ x,
                                                     float* __restrict__ y, uint32_t total_runs) {
  pdl_enter();
  const int C = g.C, runs = C / kLrnRun;
  const float a = g.alpha / g.size;
  GRID_STRIDE32(r, total_runs) {
    const uint32_t pix = r / runs;
    const int c0 = static_cast<int>(r % runs) * kLrnRun;
    const float* xp = x + static_cast<size_t>(pix) * C;
    float v[16];  // channels c0-4 .. c0+11
    lrn_put4(v, lrn_ld4(xp, c0 - 4, C));
    lrn_put4(v + 4, lrn_ld4(xp, c0, C));
    lrn_put4(v + 8, lrn_ld4(xp, c0 + 4, C));
    lrn_put4(v + 12, lrn_ld4(xp, c0 + 8, C));
    float out[kLrnRun];
#pragma unroll
    for (int i = 0; i < kLrnRun; ++i) {  // channel c0 + i = v[i + 4]; window v[i+2 .. i+6]
      out[i] = __fmul_rn(v[i + 4], lrn_pow(lrn_scale(g.k, a, lrn_sq5(v + i + 2)), g.beta));
    }
    float4* dst = reinterpret_cast<float4*>(y + static_cast<size_t>(pix) * C + c0);
    dst[0] = make_float4(out[0], out[1], out[2], out[3]);
    dst[1] = make_float4(out[4], out[5], out[6], out[7]);
  }
}

__global__ void __launch_bounds__(256) lrn_bwd_run_k(LrnGeom g, const float* __restrict__ x,
                                                     const float* __restrict__ dy,
                                                     float* __restrict__ dx, int accumulate,
                                                     int relu_mask, uint32_t total_runs) {
  pdl_enter();
  const int C = g.C, runs = C / kLrnRun;
  const float a = g.alpha / g.size, ratio = 2.f * g.alpha * g.beta / g.size;
  GRID_STRIDE32(r, total_runs) {
    const uint32_t pix = r / runs;
    const int c0 = static_cast<int>(r % runs) * kLrnRun;
    const size_t base = static_cast<size_t>(pix) * C;
    float v[16], d[16];  // channels c0-4 .. c0+11
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      lrn_put4(v + 4 * k, lrn_ld4(x + base, c0 - 4 + 4 * k, C));
      lrn_put4(d + 4 * k, lrn_ld4(dy + base, c0 - 4 + 4 * k, C));
    }
    // st = dy * x * s^-beta / s and s^-beta for channels c0-2 .. c0+9 (index j = ch - c0 + 2)
    float st[12], sp[12];
#pragma unroll
    for (int j = 0; j < 12; ++j) {
      const float sc = lrn_scale(g.k, a, lrn_sq5(v + j));  // window of channel j + c0 - 2
      sp[j] = lrn_pow(sc, g.beta);
      st[j] = lrn_st(d[j + 2], v[j + 2], sp[j], sc);  // zero outside [0, C): x = 0
    }
    float out[kLrnRun];
#pragma unroll
    for (int i = 0; i < kLrnRun; ++i) {  // channels q whose window holds c: [c-2, c+2]
      out[i] = lrn_dx(d[i + 4], sp[i + 2], ratio, v[i + 4], lrn_sum5(st + i));
      if (relu_mask && !(v[i + 4] > 0.f)) out[i] = 0.f;
    }
    float4* dst = reinterpret_cast<float4*>(dx + base + c0);
    if (accumulate) {
      const float4 o0 = dst[0], o1 = dst[1];
      out[0] += o0.x; out[1] += o0.y; out[2] += o0.z; out[3] += o0.w;
      out[4] += o1.x; out[5] += o1.y; out[6] += o1.z; out[7] += o1.w;
    }
    dst[0] = make_float4(out[0], out[1], out[2], out[3]);
    dst[1] = make_float4(out[4], out[5], out[6], out[7]);
  }
}

// ------------------------------------------------------- LRN -> max pool ---
// An LRN (size 5, C % 8 == 0) whose only consumer is a 3x3 max pool: the LRN output is
// never stored.  Thread = (pool output pixel, 8-channel run); each valid window tap
// recomputes the LRN of its 8 channels from x (the same ascending 5-term sums and lrn_pow
// as lrn_fwd_run_k) and feeds the max / route scan of pool_fwd_k — bitwise the unfused
// pair (each LRN value is recomputed by the <= 4 windows that hold it).
__device__ __forceinline__ void lrn_run8(const float* xp, int c0, int C, float a, const LrnGeom& g,
                                         float* out) {
  float v[16];  // channels c0-4 .. c0+11
  lrn_put4(v, lrn_ld4(xp, c0 - 4, C));
  lrn_put4(v + 4, lrn_ld4(xp, c0, C));
  lrn_put4(v + 8, lrn_ld4(xp, c0 + 4, C));
  lrn_put4(v + 12, lrn_ld4(xp, c0 + 8, C));
#pragma unroll
  for (int i = 0; i < kLrnRun; ++i) {
    out[i] = __fmul_rn(v[i + 4], lrn_pow(lrn_scale(g.k, a, lrn_sq5(v + i + 2)), g.beta));
  }
}

__global__ void __launch_bounds__(256) lrn_maxpool_fwd_k(LrnGeom lg, PoolGeom g,
                                                         const float* __restrict__ x,
                                                         float* __restrict__ y,
                                                         uint8_t* __restrict__ route,
                                                         uint32_t total_runs) {
  pdl_enter();
  constexpr int K = 3;
  const int C = g.C, runs = C / kLrnRun;
  const float a = lg.alpha / lg.size;
  GRID_STRIDE32(r, total_runs) {
    const uint32_t opix = r / runs;
    const int c0 = static_cast<int>(r % runs) * kLrnRun;
    const int ow = static_cast<int>(opix % g.OW);
    const uint32_t t = opix / g.OW;
    const int oh = static_cast<int>(t % g.OH), b = static_cast<int>(t / g.OH);
    const int hs0 = oh * g.sh - g.ph, ws0 = ow * g.sw - g.pw;
    const int hs = max(hs0, 0), he = min(hs0 + K, g.H), ws = max(ws0, 0), we = min(ws0 + K, g.W);
    const float* xb = x + static_cast<size_t>(b) * g.H * g.W * C;
    float best[kLrnRun];
    uint8_t arg[kLrnRun];
    bool have = false;
#pragma unroll
    for (int u = 0; u < K; ++u)
#pragma unroll
      for (int q = 0; q < K; ++q) {
        const int rr = hs0 + u, tt = ws0 + q;
        if (rr < hs || rr >= he || tt < ws || tt >= we) continue;
        float o[kLrnRun];
        lrn_run8(xb + static_cast<size_t>(rr * g.W + tt) * C, c0, C, a, lg, o);
#pragma unroll
        for (int e = 0; e < kLrnRun; ++e)
          if (!have || o[e] > best[e]) {
            best[e] = o[e];
            arg[e] = static_cast<uint8_t>(u * K + q);
          }
        have = true;
      }
    const size_t ob = static_cast<size_t>(opix) * C + c0;
    float4* dst = reinterpret_cast<float4*>(y + ob);
    dst[0] = make_float4(best[0], best[1], best[2], best[3]);
    dst[1] = make_float4(best[4], best[5], best[6], best[7]);
    uchar4* rd = reinterpret_cast<uchar4*>(route + ob);
    rd[0] = make_uchar4(arg[0], arg[1], arg[2], arg[3]);
    rd[1] = make_uchar4(arg[4], arg[5], arg[6], arg[7]);
  }
}

// Backward of the fused pair: thread = (LRN input pixel, RUN-channel run, RUN = 8 or 6)
// with the runs of a pixel on consecutive lanes of one warp (lp = runs rounded up to a
// power of two lanes per pixel), so the LRN window halos (x at c0-4 .. c0-1 /
// c0+RUN .. c0+RUN+3, and the st terms of c0-2, c0-1, c0+RUN, c0+RUN+1) come from the
// neighbouring lanes by shuffles;
// each lane gathers the pool gradient of its own 8 channels only, from the covering
// windows in ascending (oh, ow) order (pool_bwd_k's sum), and evaluates lrn_bwd_run_k's
// arithmetic unchanged — bitwise the unfused pool backward + LRN backward.
template <int RUN>  // RUN consecutive channels at p (RUN = 8: float4 x 2, 6: float2 x 3)
__device__ __forceinline__ void ld_run(const float* p, float* v) {
  if constexpr (RUN == 8) {
    lrn_put4(v, __ldg(reinterpret_cast<const float4*>(p)));
    lrn_put4(v + 4, __ldg(reinterpret_cast<const float4*>(p + 4)));
  } else {
#pragma unroll
    for (int k = 0; k < RUN / 2; ++k) {
      const float2 q = __ldg(reinterpret_cast<const float2*>(p) + k);
      v[2 * k] = q.x;
      v[2 * k + 1] = q.y;
    }
  }
}
// n / d and n % d for a fixed divisor from a host-computed magic multiplier (n < 2^31)
// (mul = ceil(2^(32+s) / d) < 2^33 with s = ceil(log2 d): n * mul < 2^64, and the rounding
// error n * (mul * d - 2^(32+s)) / (d * 2^(32+s)) < 1 / (2d) never crosses an integer)
struct FastDiv {
  uint64_t mul = 0;
  uint32_t d = 1, shift = 0;
  FastDiv() = default;
  explicit FastDiv(uint32_t div) : d(div) {
    while ((1ull << shift) < d) ++shift;
    mul = ((1ull << (32 + shift)) + d - 1) / d;
  }
  __device__ __forceinline__ uint32_t div(uint32_t n) const {
    return static_cast<uint32_t>((static_cast<uint64_t>(n) * mul) >> (32 + shift));
  }
};

// S > 0: the specialised case (3x3 windows, stride S, no padding, compile time): the
// covering windows of a pixel come from shifts, their bounds checks are implied by the
// range, and the route bytes of 4 channels compare in one SIMD op.  S = 0: any geometry.
template <int NW, int RUN, int S>
__global__ void __launch_bounds__(256) lrn_maxpool_bwd_k(LrnGeom lg, PoolGeom g,
                                                         const float* __restrict__ x,
                                                         const float* __restrict__ dpool,
                                                         const uint8_t* __restrict__ route,
                                                         float* __restrict__ dx, int accumulate,
                                                         int relu_mask, int lp, uint32_t pixels,
                                                         FastDiv fw, FastDiv fh) {
  pdl_enter();
  const int C = g.C, runs = C / RUN, ppw = 32 / lp;
  const float a = lg.alpha / lg.size, ratio = 2.f * lg.alpha * lg.beta / lg.size;
  const int lane = threadIdx.x & 31, grp = lane / lp, run = lane % lp, c0 = run * RUN;
  const uint32_t warps = gridDim.x * (blockDim.x / 32);
  for (uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) / 32; w * ppw < pixels; w += warps) {
    const uint32_t pix = w * ppw + grp;  // warp-uniform loop: every lane reaches the shuffles
    const bool act = run < runs && pix < pixels;
    float v[RUN], d[RUN];
#pragma unroll
    for (int i = 0; i < RUN; ++i) v[i] = d[i] = 0.f;
    size_t base = 0;
    if constexpr (S > 0) {
     if (act) {
      base = static_cast<size_t>(pix) * C + c0;
      ld_run<RUN>(x + base, v);
      const uint32_t t = fw.div(pix), bq = fh.div(t);
      const int wq = static_cast<int>(pix - t * g.W), h = static_cast<int>(t - bq * g.H);
      const int ohl = max(0, (h - 3 + S) / S), ohh = min(g.OH - 1, h / S);
      const int owl = max(0, (wq - 3 + S) / S), owh = min(g.OW - 1, wq / S);
#pragma unroll
      for (int i = 0; i < NW; ++i) {
        const int oh = ohl + i;
        if (oh > ohh) break;
        const size_t orow = (static_cast<size_t>(bq) * g.OH + oh) * g.OW;
        const uint32_t u3 = static_cast<uint32_t>(h - oh * S) * 3u;
#pragma unroll
        for (int q = 0; q < NW; ++q) {
          const int ow = owl + q;
          if (ow > owh) break;
          const uint32_t want = (u3 + static_cast<uint32_t>(wq - ow * S)) * 0x01010101u;
          const size_t ob = (orow + ow) * C + c0;
          float dd[RUN];
          ld_run<RUN>(dpool + ob, dd);
          uint32_t rr[2];
          if constexpr (RUN == 8) {
            const uint2 q2 = __ldg(reinterpret_cast<const uint2*>(route + ob));
            rr[0] = q2.x;
            rr[1] = q2.y;
          } else {
            const uint16_t* r16 = reinterpret_cast<const uint16_t*>(route + ob);
            rr[0] = __ldg(r16) | (static_cast<uint32_t>(__ldg(r16 + 1)) << 16);
            rr[1] = __ldg(r16 + 2);
          }
          const uint32_t m0 = __vcmpeq4(rr[0], want), m1 = __vcmpeq4(rr[1], want);
#pragma unroll
          for (int e = 0; e < RUN; ++e)  // select, not "+ 0": same values as the generic path
            d[e] = ((e < 4 ? m0 : m1) >> (8 * (e & 3))) & 1u ? d[e] + dd[e] : d[e];
        }
      }
     }
    } else if (act) {
      base = static_cast<size_t>(pix) * C + c0;
      ld_run<RUN>(x + base, v);
      const int wq = static_cast<int>(pix % g.W);
      const uint32_t t = pix / g.W;
      const int h = static_cast<int>(t % g.H), b = static_cast<int>(t / g.H);
      const int ohl = max(0, (h + g.ph - g.kh + g.sh) / g.sh);
      const int ohh = min(g.OH - 1, (h + g.ph) / g.sh);
      const int owl = max(0, (wq + g.pw - g.kw + g.sw) / g.sw);
      const int owh = min(g.OW - 1, (wq + g.pw) / g.sw);
#pragma unroll
      for (int i = 0; i < NW; ++i)
#pragma unroll
        for (int q = 0; q < NW; ++q) {
          const int oh = ohl + i, ow = owl + q;
          const int hs0 = oh * g.sh - g.ph, ws0 = ow * g.sw - g.pw;
          if (oh > ohh || ow > owh || h < hs0 || h >= hs0 + g.kh || wq < ws0 || wq >= ws0 + g.kw)
            continue;
          const uint32_t want = static_cast<uint32_t>((h - hs0) * g.kw + (wq - ws0));
          const size_t ob = (static_cast<size_t>(b * g.OH + oh) * g.OW + ow) * C + c0;
          float dd[RUN];
          ld_run<RUN>(dpool + ob, dd);
          uint32_t rr[2];  // RUN route bytes (RUN = 8: 8-byte aligned, 6: 2-byte aligned)
          if constexpr (RUN == 8) {
            const uint2 q2 = __ldg(reinterpret_cast<const uint2*>(route + ob));
            rr[0] = q2.x;
            rr[1] = q2.y;
          } else {
            const uint16_t* r16 = reinterpret_cast<const uint16_t*>(route + ob);
            rr[0] = __ldg(r16) | (static_cast<uint32_t>(__ldg(r16 + 1)) << 16);
            rr[1] = __ldg(r16 + 2);
          }
#pragma unroll
          for (int e = 0; e < RUN; ++e)
            if (((rr[e / 4] >> (8 * (e & 3))) & 0xffu) == want) d[e] += dd[e];
        }
    }
    // x at channels c0-4 .. c0+RUN+3 (neighbour lanes; zero outside [0, C))
    float xw[RUN + 8];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float l = __shfl_up_sync(0xffffffffu, v[RUN - 4 + k], 1);
      const float r = __shfl_down_sync(0xffffffffu, v[k], 1);
      xw[k] = run > 0 ? l : 0.f;
      xw[RUN + 4 + k] = run + 1 < runs ? r : 0.f;
    }
#pragma unroll
    for (int i = 0; i < RUN; ++i) xw[4 + i] = v[i];
    float st[RUN], sp[RUN];
#pragma unroll
    for (int i = 0; i < RUN; ++i) {  // channel c0 + i = xw[i + 4]; window xw[i+2 .. i+6]
      const float sc = lrn_scale(lg.k, a, lrn_sq5(xw + i + 2));
      sp[i] = lrn_pow(sc, lg.beta);
      st[i] = lrn_st(d[i], v[i], sp[i], sc);
    }
    // st at channels c0-2 .. c0+RUN+1
    float sw[RUN + 4];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const float l = __shfl_up_sync(0xffffffffu, st[RUN - 2 + k], 1);
      const float r = __shfl_down_sync(0xffffffffu, st[k], 1);
      sw[k] = run > 0 ? l : 0.f;
      sw[RUN + 2 + k] = run + 1 < runs ? r : 0.f;
    }
#pragma unroll
    for (int i = 0; i < RUN; ++i) sw[2 + i] = st[i];
    if (!act) continue;
    float out[RUN];
#pragma unroll
    for (int i = 0; i < RUN; ++i) {  // channels whose window holds c0 + i: sw[i .. i+4]
      out[i] = lrn_dx(d[i], sp[i], ratio, v[i], lrn_sum5(sw + i));
      if (relu_mask && !(v[i] > 0.f)) out[i] = 0.f;
    }
    float* dst = dx + base;
#pragma unroll
    for (int k = 0; k < RUN / 2; ++k) {
      float2 o = make_float2(out[2 * k], out[2 * k + 1]);
      float2* p2 = reinterpret_cast<float2*>(dst) + k;
      if (accumulate) {
        const float2 q = *p2;
        o.x += q.x;
        o.y += q.y;
      }
      *p2 = o;
    }
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
  pdl_enter();
  if (!train) {
    GRID_STRIDE32(i, total) y[i] = x[i];
    return;
  }
  const uint64_t base = mix64(g.base_seed ^ *d_step);
  const uint32_t thresh = static_cast<uint32_t>(static_cast<double>(g.ratio) * 16777216.0);
  const float keep = static_cast<float>(1.0 / (1.0 - static_cast<double>(g.ratio)));
  GRID_STRIDE32(i, total) y[i] = x[i] * drop_mask(g, base, i, thresh, keep);
}

// relu_mask: the backward of a ReLU whose only consumer is this dropout, folded in
// (dx = relu_mask > 0 ? dy * mask : 0, written to the ReLU's input gradient).
__global__ void dropout_bwd_k(DropGeom g, const float* __restrict__ dy, float* __restrict__ dx,
                              const uint64_t* __restrict__ d_step, int accumulate,
                              const float* __restrict__ relu_mask, uint32_t total) {
  pdl_enter();
  const uint64_t base = mix64(g.base_seed ^ *d_step);
  const uint32_t thresh = static_cast<uint32_t>(static_cast<double>(g.ratio) * 16777216.0);
  const float keep = static_cast<float>(1.0 / (1.0 - static_cast<double>(g.ratio)));
  GRID_STRIDE32(i, total) {
    float v = dy[i] * drop_mask(g, base, i, thresh, keep);
    if (relu_mask && !(relu_mask[i] > 0.f)) v = 0.f;
    dx[i] = accumulate ? dx[i] + v : v;
  }
}

// ---------------------------------------------------------------- gather ---
// data.hpp:292-304 gather_batch from the HBM-resident shard (NHWC rows).
__global__ void gather_k(const float* __restrict__ ds, const int32_t* __restrict__ ds_labels,
                         const uint32_t* __restrict__ idx, const int* __restrict__ cursor, int b,
                         int pixels, int C, int cs, float* __restrict__ out,
                         int32_t* __restrict__ labels) {
  pdl_enter();
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
  pdl_enter();
  GRID_STRIDE32(i, total) {
    const uint32_t c = i % cs, t = i / cs;
    const uint32_t w = t % W, t2 = t / W;
    const uint32_t h = t2 % H, b = t2 / H;
    dst[i] = c < static_cast<uint32_t>(C) ? src[((static_cast<size_t>(b) * C + c) * H + h) * W + w]
                                          : 0.f;
  }
}

}  // namespace

namespace {
// compile-time window for the common square 3x3 / 2x2 pools (loads issued together)
int pool_k(const PoolGeom& g) {
  if (g.kh == g.kw && (g.kh == 2 || g.kh == 3)) return g.kh;
  return 0;
}
}  // namespace

void pool_fwd(const PoolGeom& g, const float* x, float* y, uint8_t* route, cudaStream_t s) {
  checked32(static_cast<size_t>(g.n) * g.OH * g.OW * g.C, "pool");
  checked32(static_cast<size_t>(g.n) * g.H * g.W * g.C, "pool");
  const unsigned rows = static_cast<unsigned>(g.n) * g.OH;
  const int k = pool_k(g);
  if (g.C % 4 == 0) {
    auto kern = k == 3 ? pool_fwd_k<float4, 3> : k == 2 ? pool_fwd_k<float4, 2> : pool_fwd_k<float4, 0>;
    launch_k(kern, rows, 256, 0, s, g, reinterpret_cast<const float4*>(x),
             reinterpret_cast<float4*>(y), reinterpret_cast<uchar4*>(route), g.C / 4);
  } else {
    auto kern = k == 3 ? pool_fwd_k<float, 3> : k == 2 ? pool_fwd_k<float, 2> : pool_fwd_k<float, 0>;
    launch_k(kern, rows, 256, 0, s, g, x, y, route, g.C);
  }
  PSG_CUDA(cudaGetLastError());
}

void pool_bwd(const PoolGeom& g, const float* dy, const uint8_t* route, float* dx,
              bool accumulate, cudaStream_t s, const float* relu_mask) {
  // PSG_POOL_BWD_LOADS_FIRST=0: the window loop for the compile-time 3x3 windows too (A/B)
  static const int loads_first = [] {
    const char* e = std::getenv("PSG_POOL_BWD_LOADS_FIRST");
    return e ? (std::atoi(e) != 0 ? 1 : 0) : 1;
  }();
  checked32(static_cast<size_t>(g.n) * g.H * g.W * g.C, "pool");
  const unsigned rows = static_cast<unsigned>(g.n) * g.H;
  const bool k3 = g.kh == 3 && g.kw == 3 && g.sh == g.sw && (g.sh == 1 || g.sh == 2);
  if (g.C % 4 == 0) {
    auto kern = !k3 ? pool_bwd_k<float4, 0, 0>
                    : g.sh == 2 ? pool_bwd_k<float4, 3, 2> : pool_bwd_k<float4, 3, 1>;
    launch_k(kern, rows, 256, 0, s, g, reinterpret_cast<const float4*>(dy),
             reinterpret_cast<const uchar4*>(route), reinterpret_cast<float4*>(dx), accumulate,
             g.C / 4, reinterpret_cast<const float4*>(relu_mask), loads_first);
  } else {
    auto kern = !k3 ? pool_bwd_k<float, 0, 0>
                    : g.sh == 2 ? pool_bwd_k<float, 3, 2> : pool_bwd_k<float, 3, 1>;
    launch_k(kern, rows, 256, 0, s, g, dy, route, dx, accumulate, g.C, relu_mask, loads_first);
  }
  PSG_CUDA(cudaGetLastError());
}

namespace {
int lrn_tile_pixels(const LrnGeom& g) { return std::max(1, kLrnTileElems / g.C); }
int lrn_blocks(const LrnGeom& g, int tp) {
  return static_cast<int>(std::min<long>((g.pixels + tp - 1) / tp, 148L * 16));
}
}  // namespace

template <class K>
void lrn_launch(K kernel, size_t smem) {
  if (smem > 48 * 1024) allow_max_dynamic_smem(reinterpret_cast<const void*>(kernel));
}

bool lrn_run_ok(const LrnGeom& g) { return g.size == 5 && g.C % kLrnRun == 0; }

void lrn_fwd(const LrnGeom& g, const float* x, float* y, cudaStream_t s) {
  checked32(static_cast<size_t>(g.pixels) * g.C, "lrn");
  if (lrn_run_ok(g)) {
    const uint32_t runs = checked32(static_cast<size_t>(g.pixels) * (g.C / kLrnRun), "lrn");
    launch_k(lrn_fwd_run_k, grid_for(runs), 256, 0, s, g, x, y, runs);
    PSG_CUDA(cudaGetLastError());
    return;
  }
  const int tp = lrn_tile_pixels(g);
  const size_t smem = static_cast<size_t>(tp) * g.C * sizeof(float);
  auto k = g.size == 5 ? lrn_fwd_k<5> : lrn_fwd_k<0>;
  lrn_launch(k, smem);
  launch_k(k, lrn_blocks(g, tp), kLrnThreads, smem, s, g, x, y, tp);
  PSG_CUDA(cudaGetLastError());
}

void lrn_bwd(const LrnGeom& g, const float* x, const float* dy, float* dx, bool accumulate,
             cudaStream_t s, bool relu_mask) {
  checked32(static_cast<size_t>(g.pixels) * g.C, "lrn");
  if (lrn_run_ok(g)) {
    const uint32_t runs = checked32(static_cast<size_t>(g.pixels) * (g.C / kLrnRun), "lrn");
    launch_k(lrn_bwd_run_k, grid_for(runs), 256, 0, s, g, x, dy, dx, accumulate, relu_mask ? 1 : 0,
                                                 runs);
    PSG_CUDA(cudaGetLastError());
    return;
  }
  const int tp = lrn_tile_pixels(g);
  const size_t smem = 4 * static_cast<size_t>(tp) * g.C * sizeof(float);
  auto k = g.size == 5 ? lrn_bwd_k<5> : lrn_bwd_k<0>;
  lrn_launch(k, smem);
  launch_k(k, lrn_blocks(g, tp), kLrnThreads, smem, s, g, x, dy, dx, accumulate, relu_mask ? 1 : 0,
                                                 tp);
  PSG_CUDA(cudaGetLastError());
}

void dropout_fwd(const DropGeom& g, const float* x, float* y, const uint64_t* d_step, bool train,
                 cudaStream_t s) {
  const uint32_t n = checked32(static_cast<size_t>(g.n) * g.C * g.H * g.W, "dropout");
  launch_k(dropout_fwd_k, grid_for(n), 256, 0, s, g, x, y, d_step, train, n);
  PSG_CUDA(cudaGetLastError());
}

void dropout_bwd(const DropGeom& g, const float* dy, float* dx, const uint64_t* d_step,
                 bool accumulate, cudaStream_t s, const float* relu_mask) {
  const uint32_t n = checked32(static_cast<size_t>(g.n) * g.C * g.H * g.W, "dropout");
  launch_k(dropout_bwd_k, grid_for(n), 256, 0, s, g, dy, dx, d_step, accumulate, relu_mask, n);
  PSG_CUDA(cudaGetLastError());
}

void gather_batch(const float* ds_images, const int32_t* ds_labels, const uint32_t* idx,
                  const int* cursor, int b, int pixels, int C, int cs, float* out,
                  int32_t* labels, cudaStream_t s) {
  const size_t per_row = checked32(static_cast<size_t>(pixels) * cs, "gather");
  const int bx = static_cast<int>(std::max<size_t>(1, std::min<size_t>((per_row / 4 + 255) / 256, 64)));
  launch_k(gather_k, dim3(bx, b), 256, 0, s, ds_images, ds_labels, idx, cursor, b, pixels, C, cs, out,
                                       labels);
  PSG_CUDA(cudaGetLastError());
}

void stage_batch_nchw(const float* src, int n, int C, int H, int W, int cs, float* dst,
                      cudaStream_t s) {
  const uint32_t total = checked32(static_cast<size_t>(n) * H * W * cs, "stage");
  launch_k(stage_nchw_k, grid_for(total), 256, 0, s, src, C, H, W, cs, dst, total);
  PSG_CUDA(cudaGetLastError());
}

bool lrn_maxpool_fusable(const LrnGeom& lg, const PoolGeom& pg) {
  return lg.size == 5 && lg.C % kLrnRun == 0 && lg.C <= 256 && pg.C == lg.C &&
         pg.method == PSG_POOL_MAX &&
         pg.kh == 3 && pg.kw == 3 && pg.sh == pg.sw && (pg.sh == 1 || pg.sh == 2) &&
         static_cast<size_t>(pg.n) * pg.H * pg.W * pg.C < (1ULL << 31);
}

void lrn_maxpool_fwd(const LrnGeom& lg, const PoolGeom& g, const float* x, float* y,
                     uint8_t* route, cudaStream_t s) {
  const uint32_t runs =
      checked32(static_cast<size_t>(g.n) * g.OH * g.OW * (g.C / kLrnRun), "lrn_pool");
  launch_k(lrn_maxpool_fwd_k, grid_for(runs, 256, 148 * 8), 256, 0, s, lg, g, x, y, route, runs);
  PSG_CUDA(cudaGetLastError());
}

void lrn_maxpool_bwd(const LrnGeom& lg, const PoolGeom& g, const float* x, const float* dpool,
                     const uint8_t* route, float* dx, bool accumulate, bool relu_mask,
                     cudaStream_t s) {
  // channels per lane: 8, or 6 when that fills the pixel's power-of-two lane group better
  // (C = 96: 16 lanes of 6 instead of 12 of 16 lanes busy; C = 192: 32 instead of 24)
  auto lanes = [](int runs) {
    int lp = 1;
    while (lp < runs) lp <<= 1;
    return lp;
  };
  const int r8 = g.C / 8, l8 = lanes(r8);
  const bool six = g.C % 6 == 0 && lanes(g.C / 6) <= 32 &&
                   static_cast<double>(g.C / 6) / lanes(g.C / 6) > static_cast<double>(r8) / l8;
  const int lp = six ? lanes(g.C / 6) : l8;
  if (lp > 32) throw std::invalid_argument("lrn_pool: more than 256 channels");
  const uint32_t pixels = checked32(static_cast<size_t>(g.n) * g.H * g.W, "lrn_pool");
  checked32(static_cast<size_t>(pixels) * g.C, "lrn_pool");
  const size_t warps = (pixels + 32 / lp - 1) / (32 / lp);
  static const bool spec_env = [] {  // PSG_LRN_BWD_SPEC=0: the generic window path (A/B)
    const char* e = std::getenv("PSG_LRN_BWD_SPEC");
    return e ? std::atoi(e) != 0 : true;
  }();
  const bool spec = spec_env && g.ph == 0 && g.pw == 0;  // fusable: 3x3, stride 1 or 2
  auto kern = spec ? (six ? (g.sh == 1 ? lrn_maxpool_bwd_k<3, 6, 1> : lrn_maxpool_bwd_k<2, 6, 2>)
                          : (g.sh == 1 ? lrn_maxpool_bwd_k<3, 8, 1> : lrn_maxpool_bwd_k<2, 8, 2>))
                   : (six ? (g.sh == 1 ? lrn_maxpool_bwd_k<3, 6, 0> : lrn_maxpool_bwd_k<2, 6, 0>)
                          : (g.sh == 1 ? lrn_maxpool_bwd_k<3, 8, 0> : lrn_maxpool_bwd_k<2, 8, 0>));
  launch_k(kern, grid_for(warps * 32, 256, 148 * 8), 256, 0, s, lg, g, x, dpool, route, dx,
           accumulate ? 1 : 0, relu_mask ? 1 : 0, lp, pixels,
           FastDiv(static_cast<uint32_t>(g.W)), FastDiv(static_cast<uint32_t>(g.H)));
  PSG_CUDA(cudaGetLastError());
}

}  // namespace psg
