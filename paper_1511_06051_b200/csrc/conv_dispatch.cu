// Precision-mode dispatch for the GEMM-shaped layers (conv + linear):
//   Mode::Strict -> fp32 SIMT implicit GEMM (conv_simt.cu), the 1e-5 parity mode;
//   Mode::Tf32   -> tcgen05 kind::tf32 GEMMs (conv_tc.cu):
//     fprop / dgrad straight from the NHWC activations wherever the operands are
//       TMA-rectangle-describable (stride 1, channel blocks of 16/32);
//     otherwise (e.g. AlexNet conv1: 3 channels, stride 4) fprop goes through an explicit
//       im2col matrix (written once per step, reused by wgrad); such a layer's dgrad
//       (never needed for a first layer) stays on the SIMT kernel;
//     wgrad runs multi-tap implicit GEMM tiles from the activations; only layers whose
//       activations TMA cannot tile (stride > 1, C/G < 16) use the im2col matrix.
//   Strided convolutions (AlexNet conv1 11x11/4, GoogLeNet conv1 7x7/2) instead take the
//   space-to-depth route: x is rearranged once into s x s pixel blocks,
//   x'[b][hs][ws][(dy*s + dx)*C + c] = x[b][s*hs + dy - p][s*ws + dx - p][c], which turns
//   the layer into a stride-1 ceil(k/s) x ceil(k/s) convolution over s*s*C channels with
//   zero-extended weights W'.  fprop and wgrad then run as ordinary TMA-tiled tcgen05
//   convolutions (no im2col round trip through HBM); dW is folded back from dW'.
#include <algorithm>
#include <cstdlib>

#include "psg_internal.h"

namespace psg {

void conv_fprop_simt(const ConvGeom& g, const float* x, const float* w, const float* bias,
                     float* y, bool relu, const Workspace& ws, cudaStream_t s);
void conv_dgrad_simt(const ConvGeom& g, const float* dy, const float* w, float* dx,
                     bool accumulate, const Workspace& ws, cudaStream_t s);
bool linear_small(const ConvGeom& g);  // conv_simt.cu
void conv_wgrad_simt(const ConvGeom& g, const float* x, const float* dy, float* dw, float* db,
                     const Workspace& ws, cudaStream_t s);
size_t conv_workspace_elems_simt(const ConvGeom& g);
int conv_launches_simt(const ConvGeom& g, int which);

bool tc_supported(const ConvGeom& g, int which);
size_t tc_workspace_elems(const ConvGeom& g);
int tc_launches(const ConvGeom& g, int which);
void tc_fprop(const ConvGeom& g, const float* x, const float* w, const float* bias, float* y,
              bool relu, const Workspace& ws, cudaStream_t s);
void tc_dgrad(const ConvGeom& g, const float* dy, const float* w, float* dx, bool accumulate,
              const Workspace& ws, cudaStream_t s, const float* relu_mask, const float* wt);
bool tc_dgrad_wt(const ConvGeom& g);
void tc_dgrad_wt_transpose(const ConvGeom& g, const float* w, float* wt, cudaStream_t s);
void tc_wgrad(const ConvGeom& g, const float* x, const float* dy, float* dw, float* db,
              const Workspace& ws, cudaStream_t s);
bool tc_wgrad_col_supported(const ConvGeom& g);
size_t tc_wgrad_col_ws_elems(const ConvGeom& g);
int tc_wgrad_col_launches(const ConvGeom& g);
void tc_wgrad_col(const ConvGeom& g, const float* col, const float* dy, float* dw, float* db,
                  const Workspace& ws, cudaStream_t s);

void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess)
    throw CudaError(std::string(cudaGetErrorString(e)) + " in " + what + " (" + file + ":" +
                    std::to_string(line) + ")");
}

namespace {

bool is_linear(const ConvGeom& g) {
  return g.H == 1 && g.W == 1 && g.OH == 1 && g.OW == 1 && g.kh == 1 && g.kw == 1;
}

// The im2col matrix [n*OH*OW][Kp] seen as a linear layer's input (D = Kp), G = 1.
ConvGeom col_geom(const ConvGeom& g) {
  ConvGeom l;
  l.n = g.n * g.OH * g.OW;
  l.H = l.W = l.OH = l.OW = 1;
  l.cs_in = g.Kp();
  l.F = g.F;
  l.tc_pair = g.tc_pair;
  return l;
}

// ---- space-to-depth route ----
// x' channels: s*s*C rounded up to a multiple of 16 (16-float K blocks), or of 32 when that
// is more than one 32-block (AlexNet conv1: 48 -> 64, 128-byte rows / SWIZZLE_128B K
// blocks; PSG_S2D_C32=0 keeps 48)
int s2d_channels(const ConvGeom& g) {
  static const bool c32 = [] {
    const char* e = std::getenv("PSG_S2D_C32");
    return e ? std::atoi(e) != 0 : true;
  }();
  const int c = g.sh * g.sh * g.Cgs();
  return c32 && c > 32 ? (c + 31) / 32 * 32 : (c + 15) / 16 * 16;
}

ConvGeom s2d_geom(const ConvGeom& g) {
  const int s = g.sh, k = (g.kh + s - 1) / s;
  ConvGeom q;
  q.n = g.n;
  q.OH = g.OH;
  q.OW = g.OW;
  q.H = g.OH + k - 1;
  q.W = g.OW + k - 1;
  q.cs_in = s2d_channels(g);
  q.F = g.F;
  q.kh = q.kw = k;
  q.tc_pair = g.tc_pair;
  return q;
}

size_t s2d_x_elems(const ConvGeom& g) {
  const ConvGeom q = s2d_geom(g);
  return static_cast<size_t>(q.n) * q.H * q.W * q.cs_in;
}
size_t s2d_w_elems(const ConvGeom& g) {
  const ConvGeom q = s2d_geom(g);
  return (static_cast<size_t>(q.F) * q.Kf() + 31) / 32 * 32;  // keep the next buffer aligned
}

bool s2d_route(const ConvGeom& g) {
  static const bool enabled = [] {
    const char* e = std::getenv("PSG_S2D");
    return e ? std::atoi(e) != 0 : true;
  }();
  if (!enabled || is_linear(g) || g.G != 1 || g.sh < 2 || g.sh != g.sw || g.kh != g.kw ||
      g.ph != g.pw || tc_supported(g, 0))
    return false;
  const ConvGeom q = s2d_geom(g);
  // the s2d input must cover every output's receptive field
  if ((q.H - 1) * g.sh + g.sh - 1 - g.ph < (g.OH - 1) * g.sh + g.kh - 1 - g.ph) return false;
  return tc_supported(q, 0) && tc_supported(q, 2);
}

// x'[b][hs][ws][c'] for c' = (dy*s + dx)*C + c < s*s*C; 0 beyond (and outside x).
// Block = one x' row (b, hs).  Thread = one (ws, dy) pair: for fixed dy the s*C values
// c' = dy*s*C .. dy*s*C + s*C - 1 are one contiguous run of input row ih = s*hs + dy - ph
// (columns s*ws - pw .. s*ws - pw + s - 1, all channels), so the thread copies a run with
// one division per run instead of per element; the channel padding past s*s*C is written
// by the dy = s - 1 thread.  With `idx` the images come straight from the HBM-resident
// dataset (row idx[cursor * batch + b], channel stride src_cs) and the block of row hs = 0
// also copies the label: the batch gather and the space-to-depth rearrangement in one pass
// (data.hpp:292-304 gather_batch).
// RUN = s * C when it is 12 (AlexNet conv1: s = 4, C = 3): float4 stores; 6 (GoogLeNet
// conv1: s = 2, C = 3): float2 stores
template <int RUN>
__global__ void __launch_bounds__(256) s2d_x_k(const float* __restrict__ x, ConvGeom g,
                                               ConvGeom q, float* __restrict__ xs,
                                               const uint32_t* __restrict__ idx,
                                               const int* __restrict__ cursor, int batch,
                                               int src_cs, const int32_t* __restrict__ ds_labels,
                                               int32_t* __restrict__ labels) {
  pdl_enter();
  const int s = g.sh, C = g.Cgs(), run = s * C, row = blockIdx.x;
  const int hs = row % q.H, b = row / q.H;
  float* out = xs + static_cast<size_t>(row) * q.W * q.cs_in;
  size_t img = b;
  if (idx) {
    img = idx[static_cast<size_t>(cursor ? *cursor : 0) * batch + b];
    if (hs == 0 && threadIdx.x == 0) labels[b] = ds_labels[img];
  }
  // src_cs > 0: NHWC source with channel stride src_cs; src_cs < 0: NCHW with -src_cs
  // channels (a host-fed batch in the reference's layout)
  const bool nchw = src_cs < 0;
  const int cs = nchw ? -src_cs : src_cs;
  const int ps = nchw ? 1 : cs, cst = nchw ? g.H * g.W : 1, rs = nchw ? g.W : g.W * cs;
  const float* xb = x + img * g.H * g.W * cs;
  for (int j = threadIdx.x; j < q.W * s; j += blockDim.x) {
    const int ws = j / s, dy = j - ws * s;
    const int ih = s * hs + dy - g.ph, iw0 = s * ws - g.pw;
    float* o = out + ws * q.cs_in + dy * run;
    const bool row_ok = ih >= 0 && ih < g.H;
    const float* xr = xb + static_cast<size_t>(ih) * rs;
    if constexpr (RUN == 12) {
      float v[12];
#pragma unroll
      for (int dx = 0; dx < 4; ++dx) {
        const int iw = iw0 + dx;
        const bool ok = row_ok && iw >= 0 && iw < g.W;
#pragma unroll
        for (int c = 0; c < 3; ++c) v[dx * 3 + c] = ok ? __ldg(xr + iw * ps + c * cst) : 0.f;
      }
      float4* o4 = reinterpret_cast<float4*>(o);
      o4[0] = make_float4(v[0], v[1], v[2], v[3]);
      o4[1] = make_float4(v[4], v[5], v[6], v[7]);
      o4[2] = make_float4(v[8], v[9], v[10], v[11]);
    } else if constexpr (RUN == 6) {
      float v[6];
#pragma unroll
      for (int dx = 0; dx < 2; ++dx) {
        const int iw = iw0 + dx;
        const bool ok = row_ok && iw >= 0 && iw < g.W;
#pragma unroll
        for (int c = 0; c < 3; ++c) v[dx * 3 + c] = ok ? __ldg(xr + iw * ps + c * cst) : 0.f;
      }
      float2* o2 = reinterpret_cast<float2*>(o);
      o2[0] = make_float2(v[0], v[1]);
      o2[1] = make_float2(v[2], v[3]);
      o2[2] = make_float2(v[4], v[5]);
    } else {
      for (int dx = 0; dx < s; ++dx) {
        const int iw = iw0 + dx;
        const bool ok = row_ok && iw >= 0 && iw < g.W;
        for (int c = 0; c < C; ++c) o[dx * C + c] = ok ? __ldg(xr + iw * ps + c * cst) : 0.f;
      }
    }
    if (dy == s - 1) {
      float* z = out + ws * q.cs_in;
      int cp = s * run;
      if (RUN > 0)  // 16-byte aligned channel padding (s * run and cs_in multiples of 4)
        for (; cp + 4 <= q.cs_in; cp += 4)
          *reinterpret_cast<float4*>(z + cp) = make_float4(0.f, 0.f, 0.f, 0.f);
      for (; cp < q.cs_in; ++cp) z[cp] = 0.f;
    }
  }
}

using S2dKernel = void (*)(const float*, ConvGeom, ConvGeom, float*, const uint32_t*, const int*,
                          int, int, const int32_t*, int32_t*);
S2dKernel s2d_kernel(const ConvGeom& g, const ConvGeom& q) {
  // float4 runs: 12-float runs at 16-byte aligned offsets (cs_in % 4 == 0 by construction)
  // (6-float runs at 8-byte aligned offsets)
  if (q.cs_in % 4 == 0 && g.Cgs() == 3 && g.sh == 4) return s2d_x_k<12>;
  if (q.cs_in % 4 == 0 && g.Cgs() == 3 && g.sh == 2) return s2d_x_k<6>;
  return s2d_x_k<0>;
}

// W'[f][tu][tv][c'] = W[f][s*tu + dy][s*tv + dx][c] (0 past the kernel / past s*s*C)
__global__ void s2d_w_k(const float* __restrict__ w, ConvGeom g, ConvGeom q,
                        float* __restrict__ ws, int total) {
  pdl_enter();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  const int s = g.sh, C = g.Cgs(), Cp = q.cs_in, Kf = q.Kf();
  const int f = i / Kf, r = i % Kf;
  const int cp = r % Cp, tap = r / Cp, tu = tap / q.kw, tv = tap % q.kw;
  float v = 0.f;
  if (cp < s * s * C) {
    const int blk = cp / C, c = cp - blk * C;
    const int u = s * tu + blk / s, vv = s * tv + blk % s;
    if (u < g.kh && vv < g.kw) v = w[static_cast<size_t>(f) * g.Kp() + (u * g.kw + vv) * C + c];
  }
  ws[i] = v;
}

// dW[f][(u*kw + v)*C + c] = dW'[f][tu][tv][c'] (the inverse map; row padding stays 0)
__global__ void s2d_dw_k(const float* __restrict__ dws, ConvGeom g, ConvGeom q,
                         float* __restrict__ dw, int total) {
  pdl_enter();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  const int s = g.sh, C = g.Cgs(), Kp = g.Kp(), Kf = g.Kf();
  const int f = i / Kp, k = i % Kp;
  float v = 0.f;
  if (k < Kf) {
    const int c = k % C, t = k / C, u = t / g.kw, vv = t % g.kw;
    const int cp = ((u % s) * s + vv % s) * C + c, tap = (u / s) * q.kw + vv / s;
    v = dws[static_cast<size_t>(f) * q.Kf() + tap * q.cs_in + cp];
  }
  dw[i] = v;
}

void s2d_x(const ConvGeom& g, const float* x, float* xs, cudaStream_t st) {
  const ConvGeom q = s2d_geom(g);
  if (static_cast<size_t>(g.H) * g.W * g.cs_in >= (1ULL << 31))
    throw std::invalid_argument("s2d: image too large");
  launch_k(s2d_kernel(g, q), q.n * q.H, 256, 0, st, x, g, q, xs, nullptr, nullptr, 0, g.cs_in,
           nullptr, nullptr);
  PSG_CUDA(cudaGetLastError());
}

bool fprop_col_route(const ConvGeom& g) {
  return !is_linear(g) && g.G == 1 && !tc_supported(g, 0) && !s2d_route(g) &&
         tc_supported(col_geom(g), 0) && tc_wgrad_col_supported(g);
}

bool wgrad_col_route(const ConvGeom& g) {
  if (is_linear(g) || s2d_route(g) || !tc_wgrad_col_supported(g)) return false;
  return fprop_col_route(g) || !tc_supported(g, 2);
}

// col[g][pix][k] = x at (b, oh*sh - ph + u, ow*sw - pw + v, g*Cgs + c) for
// k = (u*kw + v)*Cgs + c < Kf; 0 for padding taps and for Kf <= k < Kp.  A block owns
// kPixPerBlock consecutive output pixels of one group (their origins decoded once into
// shared memory); thread t owns columns k = t, t + blockDim, ...: per column the
// kPixPerBlock loads are independent (unrolled) and every store row is contiguous.
constexpr int kPixPerBlock = 16;

__global__ void __launch_bounds__(128) im2col_k(const float* __restrict__ x, ConvGeom g,
                                                float* __restrict__ col, uint32_t pixels) {
  pdl_enter();
  __shared__ int s_ih[kPixPerBlock], s_iw[kPixPerBlock], s_base[kPixPerBlock];
  const int Kf = g.Kf(), Kp = g.Kp(), Cgs = g.Cgs(), grp = blockIdx.y;
  const uint32_t p0 = blockIdx.x * kPixPerBlock;
  if (threadIdx.x < kPixPerBlock) {
    const uint32_t p = min(p0 + threadIdx.x, pixels - 1);
    const int ow = static_cast<int>(p % g.OW), r = static_cast<int>(p / g.OW);
    const int oh = r % g.OH, b = r / g.OH;
    s_ih[threadIdx.x] = oh * g.sh - g.ph;
    s_iw[threadIdx.x] = ow * g.sw - g.pw;
    s_base[threadIdx.x] = b * g.H;
  }
  __syncthreads();
  const int np = static_cast<int>(min(static_cast<uint32_t>(kPixPerBlock), pixels - p0));
  float* colg = col + (static_cast<size_t>(grp) * pixels + p0) * Kp;
  const float* xg = x + grp * Cgs;
  for (int k = threadIdx.x; k < Kp; k += blockDim.x) {
    int ku = -(1 << 20), kv = 0, c = 0;  // padding column: every pixel out of range
    if (k < Kf) {
      c = k % Cgs;
      const int t = k / Cgs;
      kv = t % g.kw;
      ku = t / g.kw;
    }
    float v[kPixPerBlock];
#pragma unroll
    for (int i = 0; i < kPixPerBlock; ++i) {
      const int ih = s_ih[i] + ku, iw = s_iw[i] + kv;
      v[i] = (i < np && ih >= 0 && ih < g.H && iw >= 0 && iw < g.W)
                 ? __ldg(xg + (static_cast<size_t>(s_base[i] + ih) * g.W + iw) * g.cs_in + c)
                 : 0.f;
    }
#pragma unroll
    for (int i = 0; i < kPixPerBlock; ++i)
      if (i < np) colg[static_cast<size_t>(i) * Kp + k] = v[i];
  }
}

void im2col(const ConvGeom& g, const float* x, float* col, cudaStream_t s) {
  const size_t pixels = static_cast<size_t>(g.n) * g.OH * g.OW;
  if (pixels >= (1ULL << 31)) throw std::invalid_argument("im2col: too many pixels");
  const dim3 grid(static_cast<unsigned>((pixels + kPixPerBlock - 1) / kPixPerBlock), g.G);
  launch_k(im2col_k, grid, 128, 0, s, x, g, col, static_cast<uint32_t>(pixels));
  PSG_CUDA(cudaGetLastError());
}

bool use_tc(const ConvGeom& g, int which, Mode m) {
  return m == Mode::Tf32 && tc_supported(g, which);
}

// A 1x1 / stride-1 / unpadded conv (C % 4 == 0) is a linear layer over its
// pixels: its wgrad as the linear plan (dY^T X, the fprop-style epilogue with TMA stores, the
// bias as a separate pass) instead of the one-tap multi-tap plan.  PSG_TC_1X1_LINEAR=0: the
// multi-tap plan (A/B).
bool conv1x1_as_linear(const ConvGeom& g, Mode m, int cmod);
bool wgrad_1x1_linear(const ConvGeom& g, Mode m) {
  static const int env = [] {  // 1 = whole 32-channel blocks, 2 (default) = any C % 4 == 0
    const char* e = std::getenv("PSG_TC_1X1_LINEAR");
    return e ? std::atoi(e) : 2;
  }();
  return env && conv1x1_as_linear(g, m, env == 1 ? 32 : 4);
}
// ... and its fprop / dgrad (linear rows instead of pixel rectangles, the TMA-store epilogue);
// PSG_TC_1X1_LINEAR_FD=0: the rectangle plans (A/B)
bool fd_1x1_linear(const ConvGeom& g, Mode m) {
  static const bool env = [] {
    const char* e = std::getenv("PSG_TC_1X1_LINEAR_FD");
    return !e || std::atoi(e) != 0;
  }();
  return env && conv1x1_as_linear(g, m, 4) && tc_supported(col_geom(g), 0) &&
         tc_supported(col_geom(g), 1);
}
bool conv1x1_as_linear(const ConvGeom& g, Mode m, int cmod) {
  return m == Mode::Tf32 && !is_linear(g) && g.G == 1 && g.kh == 1 && g.kw == 1 &&
         g.sh == 1 && g.sw == 1 && g.ph == 0 && g.pw == 0 && g.H == g.OH && g.W == g.OW &&
         g.cs_in == g.Cgs() && g.Kp() == g.cs_in && g.cs_in % cmod == 0 &&
         tc_supported(col_geom(g), 2);
}

}  // namespace

bool conv_s2d_input(const ConvGeom& g, Mode m) { return m == Mode::Tf32 && s2d_route(g); }

void gather_s2d(const ConvGeom& g, const float* ds_images, const int32_t* ds_labels,
                const uint32_t* idx, const int* cursor, int src_cs, float* col, int32_t* labels,
                cudaStream_t st) {
  const ConvGeom q = s2d_geom(g);
  if (static_cast<size_t>(g.H) * g.W * src_cs >= (1ULL << 31))
    throw std::invalid_argument("s2d: image too large");
  launch_k(s2d_kernel(g, q), q.n * q.H, 256, 0, st, ds_images, g, q, col, idx, cursor, g.n,
           src_cs, ds_labels, labels);
  PSG_CUDA(cudaGetLastError());
}

void stage_s2d_nchw(const ConvGeom& g, const float* src, int C, float* col, cudaStream_t st) {
  const ConvGeom q = s2d_geom(g);
  if (static_cast<size_t>(g.H) * g.W * C >= (1ULL << 31))
    throw std::invalid_argument("s2d: image too large");
  launch_k(s2d_kernel(g, q), q.n * q.H, 256, 0, st, src, g, q, col, nullptr, nullptr, g.n, -C,
           nullptr, nullptr);
  PSG_CUDA(cudaGetLastError());
}

namespace {
size_t col_route_elems(const ConvGeom& g, Mode m) {
  // s2d route: x' (written by fprop, read by wgrad), W', dW'
  if (m == Mode::Tf32 && s2d_route(g)) return s2d_x_elems(g) + 2 * s2d_w_elems(g);
  if (m != Mode::Tf32 || !(fprop_col_route(g) || wgrad_col_route(g))) return 0;
  return static_cast<size_t>(g.G) * g.n * g.OH * g.OW * g.Kp();
}
bool dgrad_uses_wt(const ConvGeom& g, Mode m) { return use_tc(g, 1, m) && tc_dgrad_wt(g); }
}  // namespace

// col = [im2col / space-to-depth scratch][dgrad's transposed weights Wt (32-float aligned)]
size_t conv_col_elems(const ConvGeom& g, Mode m) {
  const size_t base = (col_route_elems(g, m) + 31) / 32 * 32;
  return base + (dgrad_uses_wt(g, m) ? static_cast<size_t>(g.F) * g.kh * g.kw * g.Cgs() : 0);
}

void conv_fprop(const ConvGeom& g, const float* x, const float* w, const float* bias, float* y,
                bool relu, const Workspace& ws, float* col, Mode m, cudaStream_t s, bool x_s2d) {
  if (m == Mode::Tf32 && col && s2d_route(g)) {
    const ConvGeom q = s2d_geom(g);
    float* wq = col + s2d_x_elems(g);
    if (!x_s2d) s2d_x(g, x, col, s);
    const int wt = q.F * q.Kf();
    launch_k(s2d_w_k, (wt + 255) / 256, 256, 0, s, w, g, q, wq, wt);
    PSG_CUDA(cudaGetLastError());
    tc_fprop(q, col, wq, bias, y, relu, ws, s);
  } else if (m == Mode::Tf32 && col && fprop_col_route(g)) {
    im2col(g, x, col, s);
    tc_fprop(col_geom(g), col, w, bias, y, relu, ws, s);
  } else if (linear_small(g)) {  // few-output linear layer: dedicated kernel (any mode)
    conv_fprop_simt(g, x, w, bias, y, relu, ws, s);
  } else if (fd_1x1_linear(g, m)) {
    tc_fprop(col_geom(g), x, w, bias, y, relu, ws, s);
  } else if (use_tc(g, 0, m)) {
    tc_fprop(g, x, w, bias, y, relu, ws, s);
  } else {
    conv_fprop_simt(g, x, w, bias, y, relu, ws, s);
  }
}

bool conv_dgrad_masks(const ConvGeom& g, Mode m) { return use_tc(g, 1, m) && !linear_small(g); }

void conv_dgrad(const ConvGeom& g, const float* dy, const float* w, float* dx, bool accumulate,
                const Workspace& ws, Mode m, cudaStream_t s, const float* relu_mask, float* col) {
  if (linear_small(g) && !relu_mask) {
    conv_dgrad_simt(g, dy, w, dx, accumulate, ws, s);
  } else if (fd_1x1_linear(g, m)) {
    tc_dgrad(col_geom(g), dy, w, dx, accumulate, ws, s, relu_mask, nullptr);
  } else if (use_tc(g, 1, m)) {
    float* wt = nullptr;
    if (tc_dgrad_wt(g)) {
      if (!col) throw std::logic_error("conv_dgrad: no scratch for the transposed weights");
      wt = col + (col_route_elems(g, m) + 31) / 32 * 32;
      tc_dgrad_wt_transpose(g, w, wt, s);
    }
    tc_dgrad(g, dy, w, dx, accumulate, ws, s, relu_mask, wt);
  }
  else if (relu_mask)
    throw std::logic_error("conv_dgrad: ReLU mask needs the tensor-core path");
  else
    conv_dgrad_simt(g, dy, w, dx, accumulate, ws, s);
}

void conv_wgrad(const ConvGeom& g, const float* x, const float* dy, float* dw, float* db,
                const Workspace& ws, float* col, Mode m, cudaStream_t s) {
  if (m == Mode::Tf32 && col && s2d_route(g)) {  // x' written by this step's fprop
    const ConvGeom q = s2d_geom(g);
    float* dwq = col + s2d_x_elems(g) + s2d_w_elems(g);
    tc_wgrad(q, col, dy, dwq, db, ws, s);
    const int total = g.F * g.Kp();
    launch_k(s2d_dw_k, (total + 255) / 256, 256, 0, s, dwq, g, q, dw, total);
    PSG_CUDA(cudaGetLastError());
  } else if (m == Mode::Tf32 && col && wgrad_col_route(g)) {
    if (!fprop_col_route(g)) im2col(g, x, col, s);  // else written by this step's fprop
    tc_wgrad_col(g, col, dy, dw, db, ws, s);
  } else if (wgrad_1x1_linear(g, m)) {
    tc_wgrad(col_geom(g), x, dy, dw, db, ws, s);
  } else if (use_tc(g, 2, m)) {
    tc_wgrad(g, x, dy, dw, db, ws, s);
  } else {
    conv_wgrad_simt(g, x, dy, dw, db, ws, s);
  }
}

size_t conv_workspace_elems(const ConvGeom& g, Mode m) {
  size_t e = conv_workspace_elems_simt(g);
  if (m == Mode::Tf32) {
    e = std::max(e, tc_workspace_elems(g));
    if (s2d_route(g)) e = std::max(e, tc_workspace_elems(s2d_geom(g)));
    if (fprop_col_route(g)) e = std::max(e, tc_workspace_elems(col_geom(g)));
    if (wgrad_col_route(g)) e = std::max(e, tc_wgrad_col_ws_elems(g));
    if (wgrad_1x1_linear(g, m) || fd_1x1_linear(g, m))
      e = std::max(e, tc_workspace_elems(col_geom(g)));
  }
  return e;
}

int conv_launches(const ConvGeom& g, int which, Mode m) {
  if (m == Mode::Tf32 && which == 0 && s2d_route(g)) return 2 + tc_launches(s2d_geom(g), 0);
  if (m == Mode::Tf32 && which == 2 && s2d_route(g)) return tc_launches(s2d_geom(g), 2) + 1;
  if (m == Mode::Tf32 && which == 0 && fprop_col_route(g))
    return 1 + tc_launches(col_geom(g), 0);
  if (m == Mode::Tf32 && which == 2 && wgrad_col_route(g))
    return (fprop_col_route(g) ? 0 : 1) + tc_wgrad_col_launches(g);
  if (which == 2 && wgrad_1x1_linear(g, m)) return tc_launches(col_geom(g), 2);
  if (which != 2 && fd_1x1_linear(g, m)) return tc_launches(col_geom(g), which);
  if (which != 2 && linear_small(g)) return 1;
  if (use_tc(g, which, m)) return tc_launches(g, which) + (which == 1 && tc_dgrad_wt(g) ? 1 : 0);
  return conv_launches_simt(g, which);
}

}  // namespace psg
