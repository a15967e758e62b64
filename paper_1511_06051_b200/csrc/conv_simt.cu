// Strict-mode (fp32 FFMA) implicit-GEMM convolution for NHWC activations.
//
// Replaces the reference's scalar loops model.hpp:334-367 (forward_conv),
// :544-585 (backward_conv), :408-427 / :516-542 (linear = 1x1 conv on a 1x1
// image).  One register-tiled kernel, three operand-gather "problems":
//   fprop : D[pix][f]      = sum_{(u,v,c)} X(pix,u,v,c) * W[f][u][v][c]   (+bias, relu)
//   dgrad : D[pix_in][c]   = sum_{(u,v,f)} dY(pix_in,u,v,f) * W[f][u][v][c]
//   wgrad : D[f][(u,v,c)|1] = sum_{pix} dY[pix][f] * X(pix,u,v,c)  (bias = ones column)
// Reductions are fixed-order (per-thread sequential over a K chunk, then a
// fixed-order sum over chunks) — no atomics, bitwise reproducible.
#include <algorithm>

#include "psg_internal.h"

namespace psg {
namespace {

constexpr int BK = 8;

// ---------------------------------------------------------------- fprop ----
struct FpropProb {
  const float* x;
  const float* w;
  const float* bias;
  float* y;
  int H, W, cs_in, OH, OW, F, kh, kw, sh, sw, ph, pw, Cgs, Fg, G;
  int M, N, K;
  int relu;
  int Kp;     // weight row stride
  float* ws;  // split-K partials [splits][G][M][N], or null for a direct store
  static constexpr bool A_KC = true;  // A contiguous along k (channels)
  static constexpr bool B_KC = true;
  struct ACtx {
    const float* base;
    int ih0, iw0;
  };
  struct AK {
    int off, u, v;
    bool ok;
  };
  struct BCtx {
    const float* row;
  };
  struct BK_ {
    int k;
    bool ok;
  };
  __device__ ACtx actx(int g, int m) const {
    ACtx c{nullptr, 0, 0};
    if (m >= M) return c;
    const int ow = m % OW, t = m / OW, oh = t % OH, b = t / OH;
    c.base = x + static_cast<size_t>(b) * H * W * cs_in + g * Cgs;
    c.ih0 = oh * sh - ph;
    c.iw0 = ow * sw - pw;
    return c;
  }
  __device__ AK akey(int, int k, int ke) const {
    AK a;
    a.ok = k < ke;
    a.off = k % Cgs;
    const int t = k / Cgs;
    a.v = t % kw;
    a.u = t / kw;
    return a;
  }
  __device__ float a(const ACtx& c, const AK& k) const {
    if (!c.base || !k.ok) return 0.f;
    const int ih = c.ih0 + k.u, iw = c.iw0 + k.v;
    if (static_cast<unsigned>(ih) >= static_cast<unsigned>(H) ||
        static_cast<unsigned>(iw) >= static_cast<unsigned>(W))
      return 0.f;
    return __ldg(c.base + (static_cast<size_t>(ih) * W + iw) * cs_in + k.off);
  }
  __device__ BCtx bctx(int g, int n) const {
    return BCtx{n < N ? w + static_cast<size_t>(g * Fg + n) * Kp : nullptr};
  }
  __device__ BK_ bkey(int, int k, int ke) const { return BK_{k, k < ke}; }
  __device__ float b(const BCtx& c, const BK_& k) const {
    return (c.row && k.ok) ? __ldg(c.row + k.k) : 0.f;
  }
  __device__ void store(int g, int z, int m, int n, float v) const {
    if (ws) {
      ws[((static_cast<size_t>(z) * G + g) * M + m) * N + n] = v;
      return;
    }
    const int f = g * Fg + n;
    v += bias[f];
    if (relu) v = v > 0.f ? v : 0.f;
    y[static_cast<size_t>(m) * F + f] = v;
  }
};

// ---------------------------------------------------------------- dgrad ----
struct DgradProb {
  const float* dy;
  const float* w;
  float* dx;
  int H, W, cs_in, OH, OW, F, kh, kw, sh, sw, ph, pw, Cgs, Fg, G;
  int M, N, K;
  int accumulate;
  int Kp;     // weight row stride
  float* ws;  // split-K partials, or null for a direct store
  static constexpr bool A_KC = true;   // dY contiguous along f (fastest part of k)
  static constexpr bool B_KC = false;  // W contiguous along c (= n)
  struct ACtx {
    const float* base;
    int ih, iw;
  };
  struct AK {
    int f, u, v;
    bool ok;
  };
  struct BCtx {
    int c;
  };
  struct BK_ {
    const float* wp;
  };
  __device__ ACtx actx(int g, int m) const {
    ACtx c{nullptr, 0, 0};
    if (m >= M) return c;
    const int iw = m % W, t = m / W, ih = t % H, b = t / H;
    c.base = dy + static_cast<size_t>(b) * OH * OW * F + g * Fg;
    c.ih = ih;
    c.iw = iw;
    return c;
  }
  __device__ AK akey(int, int k, int ke) const {
    AK a;
    a.ok = k < ke;
    a.f = k % Fg;
    const int t = k / Fg;
    a.v = t % kw;
    a.u = t / kw;
    return a;
  }
  __device__ float a(const ACtx& c, const AK& k) const {
    if (!c.base || !k.ok) return 0.f;
    const int ohn = c.ih + ph - k.u, own = c.iw + pw - k.v;
    if (ohn < 0 || own < 0) return 0.f;
    if (ohn % sh || own % sw) return 0.f;
    const int oh = ohn / sh, ow = own / sw;
    if (oh >= OH || ow >= OW) return 0.f;
    return __ldg(c.base + (static_cast<size_t>(oh) * OW + ow) * F + k.f);
  }
  __device__ BCtx bctx(int, int n) const { return BCtx{n < N ? n : -1}; }
  __device__ BK_ bkey(int g, int k, int ke) const {
    if (k >= ke) return BK_{nullptr};
    const int f = k % Fg, t = k / Fg, v = t % kw, u = t / kw;
    return BK_{w + static_cast<size_t>(g * Fg + f) * Kp + static_cast<size_t>(u * kw + v) * Cgs};
  }
  __device__ float b(const BCtx& c, const BK_& k) const {
    return (c.c >= 0 && k.wp) ? __ldg(k.wp + c.c) : 0.f;
  }
  __device__ void store(int g, int z, int m, int n, float v) const {
    if (ws) {
      ws[((static_cast<size_t>(z) * G + g) * M + m) * N + n] = v;
      return;
    }
    float* p = dx + static_cast<size_t>(m) * cs_in + g * Cgs + n;
    *p = accumulate ? *p + v : v;
  }
};

// ---------------------------------------------------------------- wgrad ----
struct WgradProb {
  const float* x;
  const float* dy;
  float* ws;  // split partials [splits][G][M][N] (N = Kf + 1)
  float* dw;
  float* db;
  int H, W, cs_in, OH, OW, F, kh, kw, sh, sw, ph, pw, Cgs, Fg, G;
  int M, N, K;  // M = Fg, N = Kf + 1, K = n*OH*OW
  int Kf;
  int Kp;      // dW row stride
  int direct;  // one split: write dW / db directly
  static constexpr bool A_KC = false;  // dY contiguous along f (= m)
  static constexpr bool B_KC = false;  // X contiguous along c (part of n)
  struct ACtx {
    int f;
  };
  struct AK {
    int pix;
  };
  struct BCtx {
    int u, v, c, kind;  // kind 0 = tap, 1 = bias column, 2 = out of range
  };
  struct BK_ {
    const float* base;
    int ih0, iw0;
  };
  __device__ ACtx actx(int g, int m) const { return ACtx{m < M ? g * Fg + m : -1}; }
  __device__ AK akey(int, int k, int ke) const { return AK{k < ke ? k : -1}; }
  __device__ float a(const ACtx& c, const AK& k) const {
    if (c.f < 0 || k.pix < 0) return 0.f;
    return __ldg(dy + static_cast<size_t>(k.pix) * F + c.f);
  }
  __device__ BCtx bctx(int, int n) const {
    BCtx c{0, 0, 0, 2};
    if (n < Kf) {
      c.c = n % Cgs;
      const int t = n / Cgs;
      c.v = t % kw;
      c.u = t / kw;
      c.kind = 0;
    } else if (n == Kf) {
      c.kind = 1;
    }
    return c;
  }
  __device__ BK_ bkey(int g, int k, int ke) const {
    BK_ r{nullptr, 0, 0};
    if (k >= ke) return r;
    const int ow = k % OW, t = k / OW, oh = t % OH, b = t / OH;
    r.base = x + static_cast<size_t>(b) * H * W * cs_in + g * Cgs;
    r.ih0 = oh * sh - ph;
    r.iw0 = ow * sw - pw;
    return r;
  }
  __device__ float b(const BCtx& c, const BK_& k) const {
    if (!k.base || c.kind == 2) return 0.f;
    if (c.kind == 1) return 1.f;
    const int ih = k.ih0 + c.u, iw = k.iw0 + c.v;
    if (static_cast<unsigned>(ih) >= static_cast<unsigned>(H) ||
        static_cast<unsigned>(iw) >= static_cast<unsigned>(W))
      return 0.f;
    return __ldg(k.base + (static_cast<size_t>(ih) * W + iw) * cs_in + c.c);
  }
  __device__ void store(int g, int z, int m, int n, float v) const {
    if (direct) {
      if (n < Kf)
        dw[static_cast<size_t>(g * Fg + m) * Kp + n] = v;
      else
        db[g * Fg + m] = v;
    } else {
      ws[((static_cast<size_t>(z) * G + g) * M + m) * N + n] = v;
    }
  }
};

template <class P, int BM, int BN, int TM, int TN>
__global__ void __launch_bounds__((BM / TM) * (BN / TN))
    igemm_simt(const P p, int tiles_n, int kchunk) {
  pdl_enter();
  constexpr int NT = (BM / TM) * (BN / TN);
  constexpr int AL = BM * BK / NT, BL = BN * BK / NT;
  static_assert(AL >= 1 && BL >= 1 && NT % BK == 0, "tile config");
  __shared__ __align__(16) float As[2][BK][BM + 4];
  __shared__ __align__(16) float Bs[2][BK][BN + 4];
  const int tid = threadIdx.x;
  const int g = blockIdx.z % p.G, z = blockIdx.z / p.G;
  const int m0 = (blockIdx.x / tiles_n) * BM, n0 = (blockIdx.x % tiles_n) * BN;
  const int kb = z * kchunk, ke = min(p.K, kb + kchunk);

  int a_m[AL], a_k[AL], b_n[BL], b_k[BL];
  typename P::ACtx actx[AL];
  typename P::BCtx bctx[BL];
#pragma unroll
  for (int i = 0; i < AL; ++i) {
    const int e = tid + i * NT;
    a_k[i] = P::A_KC ? e % BK : e / BM;
    a_m[i] = P::A_KC ? e / BK : e % BM;
    actx[i] = p.actx(g, m0 + a_m[i]);
  }
#pragma unroll
  for (int i = 0; i < BL; ++i) {
    const int e = tid + i * NT;
    b_k[i] = P::B_KC ? e % BK : e / BN;
    b_n[i] = P::B_KC ? e / BK : e % BN;
    bctx[i] = p.bctx(g, n0 + b_n[i]);
  }
  float ra[AL], rb[BL];
  auto load = [&](int k0) {
    if constexpr (P::A_KC) {
      const auto key = p.akey(g, k0 + a_k[0], ke);
#pragma unroll
      for (int i = 0; i < AL; ++i) ra[i] = p.a(actx[i], key);
    } else {
#pragma unroll
      for (int i = 0; i < AL; ++i) ra[i] = p.a(actx[i], p.akey(g, k0 + a_k[i], ke));
    }
    if constexpr (P::B_KC) {
      const auto key = p.bkey(g, k0 + b_k[0], ke);
#pragma unroll
      for (int i = 0; i < BL; ++i) rb[i] = p.b(bctx[i], key);
    } else {
#pragma unroll
      for (int i = 0; i < BL; ++i) rb[i] = p.b(bctx[i], p.bkey(g, k0 + b_k[i], ke));
    }
  };
  auto stash = [&](int buf) {
#pragma unroll
    for (int i = 0; i < AL; ++i) As[buf][a_k[i]][a_m[i]] = ra[i];
#pragma unroll
    for (int i = 0; i < BL; ++i) Bs[buf][b_k[i]][b_n[i]] = rb[i];
  };

  const int ty = tid / (BN / TN), tx = tid % (BN / TN);
  float acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.f;

  if (kb < ke) {
    load(kb);
    stash(0);
    __syncthreads();
    int buf = 0;
    for (int k0 = kb; k0 < ke; k0 += BK) {
      const bool more = k0 + BK < ke;
      if (more) load(k0 + BK);
#pragma unroll
      for (int kk = 0; kk < BK; ++kk) {
        float av[TM], bv[TN];
#pragma unroll
        for (int i = 0; i < TM; i += 4) {
          const float4 t = *reinterpret_cast<const float4*>(&As[buf][kk][ty * TM + i]);
          av[i] = t.x;
          av[i + 1] = t.y;
          av[i + 2] = t.z;
          av[i + 3] = t.w;
        }
#pragma unroll
        for (int j = 0; j < TN; j += 4) {
          const float4 t = *reinterpret_cast<const float4*>(&Bs[buf][kk][tx * TN + j]);
          bv[j] = t.x;
          bv[j + 1] = t.y;
          bv[j + 2] = t.z;
          bv[j + 3] = t.w;
        }
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
      }
      if (more) {
        stash(buf ^ 1);
        __syncthreads();
        buf ^= 1;
      }
    }
  }
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int m = m0 + ty * TM + i;
    if (m >= p.M) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int n = n0 + tx * TN + j;
      if (n < p.N) p.store(g, z, m, n, acc[i][j]);
    }
  }
}

// Fixed-order sum of the split partials into dW / db.
__global__ void wgrad_reduce(const float* __restrict__ ws, int splits, int G, int M, int N,
                             int Kf, int Kp, int Fg, float* __restrict__ dw,
                             float* __restrict__ db) {
  pdl_enter();
  const size_t total = static_cast<size_t>(G) * M * N;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int n = static_cast<int>(i % N);
    const size_t gm = i / N;
    const int m = static_cast<int>(gm % M), g = static_cast<int>(gm / M);
    float s = 0.f;
    for (int z = 0; z < splits; ++z) s += ws[static_cast<size_t>(z) * total + i];
    if (n < Kf)
      dw[static_cast<size_t>(g * Fg + m) * Kp + n] = s;
    else
      db[g * Fg + m] = s;
  }
}

// Fixed-order sum of fprop / dgrad split partials into the NHWC output:
//   out[m * ld + g * gstride + n] = (accumulate ? out : 0) + sum_z ws[z] (+ bias, relu)
__global__ void splitk_reduce(const float* __restrict__ ws, int splits, int G, int M, int N,
                              const float* __restrict__ bias, int relu, int accumulate, int ld,
                              int gstride, float* __restrict__ out) {
  pdl_enter();
  const size_t total = static_cast<size_t>(G) * M * N;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int n = static_cast<int>(i % N);
    const size_t gm = i / N;
    const int m = static_cast<int>(gm % M), g = static_cast<int>(gm / M);
    float s = 0.f;
    for (int z = 0; z < splits; ++z) s += ws[static_cast<size_t>(z) * total + i];
    float* o = out + static_cast<size_t>(m) * ld + g * gstride + n;
    if (bias) {
      s += bias[g * gstride + n];
      if (relu) s = s > 0.f ? s : 0.f;
      *o = s;
    } else {
      *o = accumulate ? *o + s : s;
    }
  }
}

struct TileCfg {
  int bm, bn;
};

// Smallest padded area, preferring bigger tiles on ties.
TileCfg pick_tiles(int M, int N) {
  static const TileCfg cfgs[] = {{128, 128}, {128, 64}, {64, 128}, {128, 32}, {64, 64}};
  TileCfg best = cfgs[0];
  double best_cost = 1e300;
  for (const TileCfg& c : cfgs) {
    const double tiles = static_cast<double>((M + c.bm - 1) / c.bm) * ((N + c.bn - 1) / c.bn);
    const double cost = tiles * c.bm * c.bn * (1.0 + 0.15 * (128.0 * 128.0 / (c.bm * c.bn) - 1.0));
    if (cost < best_cost) {
      best_cost = cost;
      best = c;
    }
  }
  return best;
}

template <class P>
void launch(const P& p, int splits, int kchunk, cudaStream_t s) {
  const TileCfg t = pick_tiles(p.M, p.N);
  const int tiles_m = (p.M + t.bm - 1) / t.bm, tiles_n = (p.N + t.bn - 1) / t.bn;
  const dim3 grid(tiles_m * tiles_n, 1, p.G * splits);
  if (t.bm == 128 && t.bn == 128)
    launch_k(igemm_simt<P, 128, 128, 8, 8>, grid, 256, 0, s, p, tiles_n, kchunk);
  else if (t.bm == 128 && t.bn == 64)
    launch_k(igemm_simt<P, 128, 64, 8, 4>, grid, 256, 0, s, p, tiles_n, kchunk);
  else if (t.bm == 64 && t.bn == 128)
    launch_k(igemm_simt<P, 64, 128, 4, 8>, grid, 256, 0, s, p, tiles_n, kchunk);
  else if (t.bm == 128 && t.bn == 32)
    launch_k(igemm_simt<P, 128, 32, 4, 4>, grid, 256, 0, s, p, tiles_n, kchunk);
  else
    launch_k(igemm_simt<P, 64, 64, 4, 4>, grid, 256, 0, s, p, tiles_n, kchunk);
  PSG_CUDA(cudaGetLastError());
}

template <class P>
void fill_geom(P& p, const ConvGeom& g) {
  p.H = g.H;
  p.W = g.W;
  p.cs_in = g.cs_in;
  p.OH = g.OH;
  p.OW = g.OW;
  p.F = g.F;
  p.kh = g.kh;
  p.kw = g.kw;
  p.sh = g.sh;
  p.sw = g.sw;
  p.ph = g.ph;
  p.pw = g.pw;
  p.Cgs = g.Cgs();
  p.Fg = g.Fg();
  p.G = g.G;
}

// Split-K plan: enough blocks to cover ~2 waves of 148 SMs, K chunks of at least
// `min_chunk` and at most `max_chunk` (bounded sequential fp32 sums).
struct Split {
  int splits, kchunk;
};

Split plan_split(int M, int N, int K, int G, int min_chunk, int max_chunk) {
  const TileCfg t = pick_tiles(M, N);
  const long tiles = static_cast<long>((M + t.bm - 1) / t.bm) * ((N + t.bn - 1) / t.bn) * G;
  long want = std::max<long>(1, (296 + tiles - 1) / tiles);
  want = std::max<long>(want, (K + max_chunk - 1) / max_chunk);
  want = std::min<long>(want, std::max(1, K / min_chunk));
  int kchunk = static_cast<int>((K + want - 1) / want);
  kchunk = (kchunk + BK - 1) / BK * BK;
  return Split{(K + kchunk - 1) / kchunk, kchunk};
}

Split fprop_split(const ConvGeom& g) {
  return plan_split(g.n * g.OH * g.OW, g.Fg(), g.Kf(), g.G, 64, 1 << 30);
}
Split dgrad_split(const ConvGeom& g) {
  return plan_split(g.n * g.H * g.W, g.Cgs(), g.kh * g.kw * g.Fg(), g.G, 64, 1 << 30);
}
// wgrad reduces over every output pixel: cap the sequential chunk at 4096.
Split wgrad_split(const ConvGeom& g) {
  return plan_split(g.Fg(), g.Kf() + 1, g.n * g.OH * g.OW, g.G, 128, 4096);
}

void reduce_into(const Workspace& ws, int splits, int G, int M, int N, const float* bias,
                 bool relu, bool accumulate, int ld, int gstride, float* out, cudaStream_t s) {
  const size_t total = static_cast<size_t>(G) * M * N;
  const int blocks = static_cast<int>(std::min<size_t>((total + 255) / 256, 148 * 8));
  launch_k(splitk_reduce, blocks, 256, 0, s, ws.ptr, splits, G, M, N, bias, relu, accumulate, ld,
                                       gstride, out);
  PSG_CUDA(cudaGetLastError());
}

float* split_ws(const Workspace& ws, const Split& sp, int G, int M, int N) {
  if (sp.splits == 1) return nullptr;
  if (ws.elems < static_cast<size_t>(sp.splits) * G * M * N)
    throw std::logic_error("conv: split-K workspace too small");
  return ws.ptr;
}

}  // namespace

// Small linear layers with few outputs (the logits layer, cifar10_quick ip2: 64 -> 10):
// fprop = one warp per output (lanes split the input features, fixed xor tree); dgrad = one
// thread per input feature (sum over the <= 32 outputs in order).  The tiled kernels run
// these on one or two blocks, bound by their K-loop latency.
bool linear_small(const ConvGeom& g) {
  const bool linear = g.H == 1 && g.W == 1 && g.OH == 1 && g.OW == 1 && g.kh == 1 && g.kw == 1;
  return linear && g.G == 1 && g.cs_in == g.Kf() && g.F <= 32 && g.n <= 65536;
}

__global__ void fprop_linear_small(const float* __restrict__ x, const float* __restrict__ w,
                                   const float* __restrict__ bias, int n, int D, int F, int Kp,
                                   int relu, float* __restrict__ y) {
  pdl_enter();
  const int o = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x % 32;
  if (o >= n * F) return;  // warp-uniform
  const int i = o / F, j = o - i * F;
  const float* xr = x + static_cast<size_t>(i) * D;
  const float* wr = w + static_cast<size_t>(j) * Kp;
  float acc = 0.f;
  for (int k = lane; k < D; k += 32) acc = fmaf(__ldg(xr + k), __ldg(wr + k), acc);
#pragma unroll
  for (int m = 16; m; m >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, m);
  if (lane == 0) {
    if (bias) acc += bias[j];
    y[o] = relu && !(acc > 0.f) ? 0.f : acc;
  }
}

__global__ void dgrad_linear_small(const float* __restrict__ dy, const float* __restrict__ w,
                                   int n, int D, int F, int Kp, int accumulate,
                                   float* __restrict__ dx) {
  pdl_enter();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * D) return;
  const int i = t / D, k = t - i * D;
  const float* dr = dy + static_cast<size_t>(i) * F;
  float acc = 0.f;
  for (int j = 0; j < F; ++j) acc = fmaf(__ldg(dr + j), __ldg(w + static_cast<size_t>(j) * Kp + k), acc);
  dx[t] = accumulate ? dx[t] + acc : acc;
}

void conv_fprop_simt(const ConvGeom& g, const float* x, const float* w, const float* bias,
                     float* y, bool relu, const Workspace& ws, cudaStream_t s) {
  if (linear_small(g)) {
    const long warps = static_cast<long>(g.n) * g.F;
    launch_k(fprop_linear_small, static_cast<unsigned>((warps + 7) / 8), 256, 0, s, x, w, bias,
             g.n, g.cs_in, g.F, g.Kp(), relu ? 1 : 0, y);
    PSG_CUDA(cudaGetLastError());
    return;
  }
  FpropProb p{};
  fill_geom(p, g);
  p.x = x;
  p.w = w;
  p.bias = bias;
  p.y = y;
  p.M = g.n * g.OH * g.OW;
  p.N = g.Fg();
  p.K = g.Kf();
  p.Kp = g.Kp();
  p.relu = relu;
  const Split sp = fprop_split(g);
  p.ws = split_ws(ws, sp, g.G, p.M, p.N);
  launch(p, sp.splits, sp.kchunk, s);
  if (p.ws) reduce_into(ws, sp.splits, g.G, p.M, p.N, bias, relu, false, g.F, g.Fg(), y, s);
}

void conv_dgrad_simt(const ConvGeom& g, const float* dy, const float* w, float* dx,
                     bool accumulate, const Workspace& ws, cudaStream_t s) {
  if (linear_small(g)) {
    const long total = static_cast<long>(g.n) * g.cs_in;
    launch_k(dgrad_linear_small, static_cast<unsigned>((total + 255) / 256), 256, 0, s, dy, w,
             g.n, g.cs_in, g.F, g.Kp(), accumulate ? 1 : 0, dx);
    PSG_CUDA(cudaGetLastError());
    return;
  }
  DgradProb p{};
  fill_geom(p, g);
  p.dy = dy;
  p.w = w;
  p.dx = dx;
  p.M = g.n * g.H * g.W;
  p.N = g.Cgs();
  p.K = g.kh * g.kw * g.Fg();
  p.Kp = g.Kp();
  p.accumulate = accumulate;
  const Split sp = dgrad_split(g);
  p.ws = split_ws(ws, sp, g.G, p.M, p.N);
  launch(p, sp.splits, sp.kchunk, s);
  if (p.ws)
    reduce_into(ws, sp.splits, g.G, p.M, p.N, nullptr, false, accumulate, g.cs_in, g.Cgs(), dx,
                s);
}

size_t conv_workspace_elems_simt(const ConvGeom& g) {
  const Split f = fprop_split(g), d = dgrad_split(g), w = wgrad_split(g);
  size_t e = 0;
  if (f.splits > 1) e = std::max(e, static_cast<size_t>(f.splits) * g.G * g.n * g.OH * g.OW * g.Fg());
  if (d.splits > 1) e = std::max(e, static_cast<size_t>(d.splits) * g.G * g.n * g.H * g.W * g.Cgs());
  if (w.splits > 1) e = std::max(e, static_cast<size_t>(w.splits) * g.G * g.Fg() * (g.Kf() + 1));
  return e;
}

bool wgrad_small(const ConvGeom& g);

bool linear_small(const ConvGeom& g);

int conv_launches_simt(const ConvGeom& g, int which) {
  if (which == 2 && wgrad_small(g)) return 1;
  if (which != 2 && linear_small(g)) return 1;
  const Split sp = which == 0 ? fprop_split(g) : which == 1 ? dgrad_split(g) : wgrad_split(g);
  return sp.splits == 1 ? 1 : 2;
}

// Linear wgrad with a small output (the logits layer, e.g. cifar10_quick ip2: 10 x 64 over
// a batch of 100): one warp per dW / db element, lane l summing batch rows l, l + 32, ...
// then a fixed xor-shuffle tree (deterministic).  The tiled kernel runs such a GEMM on one
// block, bound by its K-loop latency (30 us).
__global__ void wgrad_linear_small(const float* __restrict__ x, const float* __restrict__ dy,
                                   int n, int D, int F, int Kp, float* __restrict__ dw,
                                   float* __restrict__ db) {
  pdl_enter();
  const int idx = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x % 32;
  if (idx >= F * (Kp + 1)) return;  // warp-uniform
  const int f = idx / (Kp + 1), k = idx - f * (Kp + 1);
  if (k < Kp && k >= D) {
    if (lane == 0) dw[static_cast<size_t>(f) * Kp + k] = 0.f;  // row padding
    return;
  }
  float acc = 0.f;
  for (int i = lane; i < n; i += 32) {
    const float d = __ldg(dy + static_cast<size_t>(i) * F + f);
    acc = k == Kp ? acc + d : fmaf(d, __ldg(x + static_cast<size_t>(i) * D + k), acc);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) {
    if (k == Kp)
      db[f] = acc;  // bias column: sum over the batch of dY[:, f]
    else
      dw[static_cast<size_t>(f) * Kp + k] = acc;
  }
}

bool wgrad_small(const ConvGeom& g) {
  const bool linear = g.H == 1 && g.W == 1 && g.OH == 1 && g.OW == 1 && g.kh == 1 && g.kw == 1;
  return linear && g.G == 1 && g.cs_in == g.Kf() &&
         static_cast<long>(g.F) * (g.Kp() + 1) <= 16384 && g.n <= 4096;
}

void conv_wgrad_simt(const ConvGeom& g, const float* x, const float* dy, float* dw, float* db,
                     const Workspace& ws, cudaStream_t s) {
  if (wgrad_small(g)) {
    const int total = g.F * (g.Kp() + 1);  // one warp each
    launch_k(wgrad_linear_small, (total + 7) / 8, 256, 0, s, x, dy, g.n, g.cs_in, g.F, g.Kp(),
             dw, db);
    PSG_CUDA(cudaGetLastError());
    return;
  }
  WgradProb p{};
  fill_geom(p, g);
  p.x = x;
  p.dy = dy;
  p.dw = dw;
  p.db = db;
  p.Kf = g.Kf();
  p.Kp = g.Kp();
  p.M = g.Fg();
  p.N = p.Kf + 1;
  p.K = g.n * g.OH * g.OW;
  const Split sp = wgrad_split(g);
  p.direct = sp.splits == 1;
  p.ws = split_ws(ws, sp, g.G, p.M, p.N);
  launch(p, sp.splits, sp.kchunk, s);
  if (!p.direct) {
    const size_t total = static_cast<size_t>(g.G) * p.M * p.N;
    const int blocks = static_cast<int>(std::min<size_t>((total + 255) / 256, 148 * 8));
    launch_k(wgrad_reduce, blocks, 256, 0, s, ws.ptr, sp.splits, g.G, p.M, p.N, p.Kf, p.Kp, g.Fg(), dw,
                                        db);
    PSG_CUDA(cudaGetLastError());
  }
}

}  // namespace psg
